"""CPU-side checks of the C-ABI library (no device calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import gpu_available

REPO = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (REPO / "include" / "odc.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(odc_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2409_13418_b200 import _lib

    L = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_struct_layouts_match_header():
    from paper_2409_13418_b200 import _lib

    assert ctypes.sizeof(_lib.Node) == 136
    assert ctypes.sizeof(_lib.Options) == 4 * 11 + 4 + 8 * 4  # 11 int32 (+4 padding), 4 doubles
    L = _lib.load()
    o = _lib.Options()
    L.odc_default_options(ctypes.byref(o))
    assert (o.iters_1d, o.s1_lin, o.s1_bin, o.s2_lin, o.s2_bin) == (15, 4, 11, 3, 12)
    assert o.s2_range == np.sqrt(2.0) / 2.0 and o.s1_range == 0.8


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_device():
    from paper_2409_13418_b200 import GridSpec, SphereField, contour
    from paper_2409_13418_b200._lib import OdcFailure

    with pytest.raises(OdcFailure):
        contour(SphereField((0.5, 0.5, 0.5), 0.3), GridSpec((0, 0, 0), (1, 1, 1), 8))


def test_lowering_matches_oracle_interpreter_semantics():
    """Scene programs evaluated by the oracle interpreter reproduce the
    reference's labels (pinned by the golden grids of every scene)."""
    import oracle
    from golden_util import cases, field_of, load

    for tag in cases():
        if tag.startswith("mlp"):
            continue
        field, lo, hi, R = field_of(tag)
        g = load(tag)
        S = R + 1
        rng = np.random.default_rng(0)
        vid = rng.integers(0, S**3, 4000)
        c = np.stack([vid % S, (vid // S) % S, vid // (S * S)], axis=1)
        h = (np.asarray(hi) - np.asarray(lo)) / R
        pts = np.asarray(lo) + c * h
        lab = (oracle.eval_raw_program(field, pts) > 0.5).astype(np.uint8)
        assert np.array_equal(lab, g["labels"][vid]), tag


def test_rotation_matches_reference_blas_order():
    from paper_2409_13418_b200.fields import rotation_from_euler

    R = rotation_from_euler(30, 30, 0)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-15)
    # recorded from occmesh.fields.rotation_from_euler(30, 30, 0) on the reference host
    expect = np.array([[0.8660254037844387, 0.24999999999999994, 0.4330127018922193],
                       [0.0, 0.8660254037844387, -0.49999999999999994],
                       [-0.49999999999999994, 0.4330127018922193, 0.7500000000000001]])
    assert np.array_equal(R, expect)
