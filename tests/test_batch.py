"""Config 5 throughput mode: concurrent extractions equal sequential ones."""

import numpy as np
import pytest

from paper_2409_13418_b200 import GridSpec, contour, scenes
from paper_2409_13418_b200.batch import contour_batch


def test_batch_shapes_are_valid_scenes():
    shapes = scenes.batch_shapes(64)
    assert len(shapes) == 64
    kinds = {s["field"]["type"] for s in shapes}
    assert kinds == {"sphere", "torus", "box", "csg"}
    for s in shapes[:8]:
        f, lo, hi = scenes.resolve(s, 32)  # lowers without error
        from paper_2409_13418_b200.fields import lower_program

        assert len(lower_program(f)) > 0


@pytest.mark.gpu
def test_gpu_batch_equals_sequential():
    jobs = []
    for s in scenes.batch_shapes(12):
        f, lo, hi = scenes.resolve(s, 48)
        jobs.append((f, GridSpec(lo, hi, 48)))
    seq = [contour(f, g) for f, g in jobs]
    par = contour_batch(jobs, workers=4)
    for a, b in zip(seq, par):
        assert np.array_equal(a.mesh.triangles, b.mesh.triangles)
        assert np.array_equal(a.mesh.vertices, b.mesh.vertices)
        assert a.stats["eval_counts"] == b.stats["eval_counts"]


@pytest.mark.gpu
def test_gpu_batch_shapes_match_oracle():
    import oracle

    for s in scenes.batch_shapes(8):
        f, lo, hi = scenes.resolve(s, 40)
        r = contour(f, GridSpec(lo, hi, 40))
        o = oracle.contour_oracle(f, lo, hi, 40)
        assert np.array_equal(r.mesh.triangles, o["triangles"])
        assert np.abs(r.mesh.vertices - o["vertices"]).max(initial=0) <= 1e-4 / 40
