"""The drop-in boundary takes the reference's own objects (INTEGRATION.md
section 1): occmesh field instances, GridSpec, ContourOptions and
EvalCounter.  Checked without a device: every reference field of every
scene lowers to exactly the device program our own field classes produce,
and that program -- run by the oracle's interpreter, the same postfix
semantics the device interprets -- labels 10^5 points exactly as the
reference field's own eval_raw does; options, grid and counter objects
marshal to the same C structs / snapshots.  Needs /root/reference (the
build container); skipped elsewhere."""

import ctypes
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference sources not present")


@pytest.fixture(scope="module")
def occmesh():
    sys.path.insert(0, str(REF))
    import occmesh as m

    return m


def _scenes():
    from paper_2409_13418_b200 import scenes

    out = [(k, v) for k, v in scenes.SCENES.items() if k not in ("mlp",)]
    out += [("thin_shell_256", scenes.thin_shell(256))]
    out += [(f"batch_{s}", scenes.batch_shape(s)) for s in (0, 1, 2, 3, 17, 40, 63)]
    return out


@pytest.mark.parametrize("name,scene", _scenes())
def test_reference_fields_lower_to_the_same_program(occmesh, name, scene):
    import oracle
    from occmesh.fields import Scene as RefScene
    from occmesh.fields import field_from_dict as ref_from_dict
    from paper_2409_13418_b200.fields import field_continuous, lower_program
    from paper_2409_13418_b200.fields import Scene, field_from_dict

    R = 64
    h = np.full(3, 1.0 / R)
    dom = scene.get("domain", {})
    ref = RefScene(ref_from_dict(scene["field"]), smooth_k=scene.get("smooth_k"),
                   domain_lo=dom.get("lo", (0, 0, 0)), domain_hi=dom.get("hi", (1, 1, 1))).resolve_field(h)
    ours = Scene(field_from_dict(scene["field"]), smooth_k=scene.get("smooth_k"),
                 domain_lo=dom.get("lo", (0, 0, 0)), domain_hi=dom.get("hi", (1, 1, 1))).resolve_field(h)
    assert type(ref).__module__.startswith("occmesh")
    pr, po = lower_program(ref), lower_program(ours)
    assert pr.tobytes() == po.tobytes()
    assert field_continuous(ref) == field_continuous(ours)
    pts = np.random.default_rng(len(name)).uniform(-0.05, 1.05, size=(100_000, 3))
    lab_ref = (np.asarray(ref.eval_raw(pts)) > ref.iso_level)
    lab_prog = oracle.eval_raw_program(ref, pts) > ref.iso_level
    assert np.array_equal(lab_ref, lab_prog)


def test_reference_options_grid_counter_marshal(occmesh):
    from occmesh import pipeline as RP
    from occmesh import search as RS
    from paper_2409_13418_b200 import GridSpec
    from paper_2409_13418_b200.pipeline import (ContourOptions, EvalCounter, LineBudget, SearchBudget,
                                                _grid_args, make_options, record_counts)
    from paper_2409_13418_b200 import _lib

    for kw in ({}, {"one_d": "midpoint", "split": "mdc", "repair": False},
               {"one_d": "linear-interp", "normals": "fd-gradient", "qef_truncation": 0.2, "fd_step_factor": 0.02}):
        ro = RP.ContourOptions(**kw)
        oo = ContourOptions(**kw)
        ro.budget = RS.SearchBudget(iters_1d=12, step1=RS.LineBudget(3, 9, 0.7), step2=RS.LineBudget(2, 10, 0.6))
        oo.budget = SearchBudget(iters_1d=12, step1=LineBudget(3, 9, 0.7), step2=LineBudget(2, 10, 0.6))
        a, b = make_options(ro), make_options(oo)
        assert bytes(a) == bytes(b)
    lo, hi, R = _grid_args(occmesh.GridSpec((0.1, 0.2, 0.3), (0.9, 1.0, 1.1), 77))
    lo2, hi2, R2 = _grid_args(GridSpec((0.1, 0.2, 0.3), (0.9, 1.0, 1.1), 77))
    assert list(lo) == list(lo2) and list(hi) == list(hi2) and R == R2
    st = _lib.Stats()
    st.cat_order[0], st.cat_order[1], st.cat_order[2] = 0, 1, -1
    st.eval_batches[0], st.eval_evals[0] = 1, 1000
    st.eval_batches[1], st.eval_evals[1] = 15, 300
    rc, oc = RP.EvalCounter(None), EvalCounter(None)
    record_counts(rc, st)
    record_counts(oc, st)
    assert rc.snapshot() == oc.snapshot() and rc.total_evals == 1300
