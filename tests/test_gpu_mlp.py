"""tcgen05 MLP evaluator (K9) against the SIMT reference evaluator (same bf16
operands, fp32 accumulation on CUDA cores) and against numpy fp32."""

import ctypes

import numpy as np
import pytest

import oracle
from paper_2409_13418_b200 import MlpField, _lib
from paper_2409_13418_b200.pipeline import DeviceField

pytestmark = pytest.mark.gpu


def device_raw(field, pts, impl):
    ctx = _lib.Context(0)
    L = _lib.load()
    assert L.odc_set_param(ctx.handle, b"mlp_impl", impl) == 0
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.empty(len(pts))
    with DeviceField(ctx, field) as f:
        rc = L.odc_eval_raw(ctx.handle, f.handle, pts.ctypes.data, len(pts), out.ctypes.data)
        assert rc == 0, L.odc_last_error(ctx.handle)
    return out


def logit(raw):
    raw = np.clip(raw, 1e-300, 1 - 1e-16)
    return np.log(raw / (1 - raw))


@pytest.mark.parametrize("impl", [0, 2, 3])
@pytest.mark.parametrize("n", [1, 255, 256, 1000, 70001])
def test_tc_matches_simt(n, impl):
    """impl 0: CTA-pair tcgen05 (TMEM A operand); impl 2: single-CTA tcgen05; impl 3: CTA-pair N=256 ping-pong."""
    field = MlpField(seed=0, amplitude=1.0)
    rng = np.random.default_rng(n)
    pts = rng.uniform(0, 1, size=(n, 3))
    a = device_raw(field, pts, impl)
    b = device_raw(field, pts, 1)
    la, lb = logit(a), logit(b)
    ok = np.isfinite(la) & np.isfinite(lb)
    # only the fp32 summation order differs
    assert np.abs(la - lb)[ok].max() < 2e-2
    sure = np.abs(lb) > 0.05
    assert np.array_equal(a[sure] > 0.5, b[sure] > 0.5)


def test_tc_vs_numpy_fp32_label_agreement():
    field = MlpField(seed=0, amplitude=1.0)
    rng = np.random.default_rng(7)
    pts = rng.uniform(0.1, 0.9, size=(20000, 3))
    a = device_raw(field, pts, 0) > 0.5
    c = oracle.mlp_raw_numpy(field, pts) > 0.5
    assert np.mean(a == c) > 0.995


@pytest.mark.parametrize("impl", [0, 3])
def test_tc_batch_invariance(impl):
    """A point's value does not depend on its batch or position in it (the
    shared-field oracle evaluates other batches than the pipeline)."""
    field = MlpField(seed=3, amplitude=2.0)
    rng = np.random.default_rng(1)
    pts = rng.uniform(0, 1, size=(5000, 3))
    full = device_raw(field, pts, impl)
    part = np.concatenate([device_raw(field, pts[:1234], impl), device_raw(field, pts[1234:], impl)])
    assert np.array_equal(full, part)
    rev = device_raw(field, pts[::-1].copy(), impl)[::-1]
    assert np.array_equal(full, rev)


@pytest.mark.parametrize("impl", [2, 3])
def test_labels_fast_path_equals_fp64(impl):
    """Labels-only evaluation decides most labels in fp32 within a margin
    derived from the fp32 rounding bound, and finishes the rest in fp64
    (deferred to a fix-up kernel on the CTA-pair evaluator).  Every label
    must equal the fp64 expression's (raw > 1/2), on random points and on
    points at the surface, where the fp32 test is most often undecided."""
    from paper_2409_13418_b200 import GridSpec, contour, eval_labels

    field = MlpField(seed=0, amplitude=1.0)
    mesh = contour(field, GridSpec((0, 0, 0), (1, 1, 1), 64)).mesh
    rng = np.random.default_rng(11)
    near = mesh.vertices[rng.integers(0, mesh.n_vertices, 400_000)]
    near = near + rng.normal(scale=1e-7, size=near.shape)
    pts = np.concatenate([near, rng.uniform(0, 1, size=(400_000, 3))])
    ctx = _lib.Context(0)
    L = _lib.load()
    assert L.odc_set_param(ctx.handle, b"mlp_impl", impl) == 0
    lab = np.empty(len(pts), dtype=np.uint8)
    raw = np.empty(len(pts))
    pts = np.ascontiguousarray(pts)
    with DeviceField(ctx, field) as f:
        assert L.odc_eval_labels(ctx.handle, f.handle, pts.ctypes.data, len(pts), lab.ctypes.data) == 0
        assert L.odc_eval_raw(ctx.handle, f.handle, pts.ctypes.data, len(pts), raw.ctypes.data) == 0
    assert np.array_equal(lab, (raw > 0.5).astype(np.uint8))
    assert 0.1 < lab[:400_000].mean() < 0.9  # the near set straddles the surface
