"""The QEF eigensolver (odc_eigh3.cuh, the code k_part_solve inlines) run on
the host through libodc's C-ABI must equal numpy.linalg.eigh -- the call
solve_qef_batch makes (dualize.py:358) -- bit for bit, eigenvalues and
eigenvectors.  No device needed: the header is plain IEEE fp64 with explicit
fma(), compiled without contraction for both the host and the device."""

import ctypes

import numpy as np
import pytest

from eigh3_cases import golden_qef_matrices, synthetic


def host_eigh3(A):
    from paper_2409_13418_b200 import _lib

    L = _lib.load()
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = len(A)
    w = np.empty((n, 3))
    V = np.empty((n, 3, 3))
    info = np.empty(n, dtype=np.int32)
    rc = L.odc_eigh3_host(A.ctypes.data_as(ctypes.c_void_p), n, w.ctypes.data_as(ctypes.c_void_p),
                          V.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    return w, V, info


def _assert_same(A, w, V, info):
    wn, Vn = np.linalg.eigh(A)
    assert (info == 0).all()
    bad = np.nonzero(~((w == wn).all(1) & (V == Vn).all((1, 2))))[0]
    assert bad.size == 0, f"{bad.size} of {len(A)} differ, first {A[bad[0]].tolist()}"


def test_eigh3_golden_qef_matrices_bit_exact():
    A = golden_qef_matrices()
    assert len(A) > 20000
    _assert_same(A, *host_eigh3(A))


@pytest.mark.parametrize("seed", [0, 1])
def test_eigh3_synthetic_bit_exact(seed):
    A = synthetic(4000, seed)
    _assert_same(A, *host_eigh3(A))


def test_eigh3_empty():
    w, V, info = host_eigh3(np.zeros((0, 3, 3)))
    assert w.shape == (0, 3)
