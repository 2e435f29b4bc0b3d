"""The QEF eigensolver on the device (odc_eigh3 through libodc's C-ABI, the
same inline code k_part_solve runs) against numpy.linalg.eigh -- the call
solve_qef_batch makes (dualize.py:358) -- bit for bit."""

import ctypes

import numpy as np
import pytest

from eigh3_cases import golden_qef_matrices, synthetic

pytestmark = pytest.mark.gpu


def device_eigh3(A):
    from paper_2409_13418_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = len(A)
    w = np.empty((n, 3))
    V = np.empty((n, 3, 3))
    info = np.empty(n, dtype=np.int32)
    _lib.check(L.odc_eigh3(ctx.handle, A.ctypes.data_as(ctypes.c_void_p), n, w.ctypes.data_as(ctypes.c_void_p),
                           V.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p)), ctx.handle)
    return w, V, info


@pytest.mark.parametrize("which", ["golden_qef", "synthetic"])
def test_device_eigh3_equals_numpy(which):
    A = golden_qef_matrices() if which == "golden_qef" else synthetic(20000, 7)
    w, V, info = device_eigh3(A)
    wn, Vn = np.linalg.eigh(A)
    assert (info == 0).all()
    bad = np.nonzero(~((w == wn).all(1) & (V == Vn).all((1, 2))))[0]
    assert bad.size == 0, f"{bad.size} of {len(A)} differ, first {A[bad[0]].tolist()}"
