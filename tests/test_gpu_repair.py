"""repair_nonmanifold on the device (odc_mesh_finish) for vertex fans larger
than the 64-triangle local-array fan (the global-scratch path; the reference
has no fan-size cap, polygonize.py:308-358), against golden outputs of the
unmodified reference (tests/golden/make_repair_golden.py)."""

import ctypes

import numpy as np
import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

CASES = ["bowtie_97", "book_4x20", "book_6x13", "bowtie_small"]


@pytest.mark.parametrize("name", CASES)
def test_gpu_repair_large_fans_match_reference(name):
    from paper_2409_13418_b200 import _lib
    from paper_2409_13418_b200.pipeline import _copy_mesh

    g = np.load(GOLDEN / "repair_golden.npz")
    v = np.ascontiguousarray(g[f"{name}__in_vertices"], dtype=np.float64)
    t = np.ascontiguousarray(g[f"{name}__in_triangles"], dtype=np.int32)
    n = len(v)
    kind = np.zeros(n, np.int64)
    ref = np.ascontiguousarray(np.stack([np.arange(n), np.zeros(n, np.int64)], 1))
    ctx = _lib.context(0)
    st = _lib.Stats()
    _lib.check(_lib.load().odc_mesh_finish(ctx.handle, v.ctypes.data, n, t.ctypes.data, len(t), n, kind.ctypes.data,
                                           ref.ctypes.data, 1, ctypes.byref(st)), ctx.handle)
    m = _copy_mesh(ctx, 0, st)
    assert np.array_equal(m.vertices, g[f"{name}__vertices"])
    assert np.array_equal(m.triangles, g[f"{name}__triangles"])
    assert np.array_equal(m.provenance_kind, g[f"{name}__kind"])
    assert np.array_equal(m.provenance_ref, g[f"{name}__ref"])
