"""Any occupancy function (the reference's field duck type: an object with
``eval_raw``, fields.py:51-61) runs through the device pipeline as a callback
field: every batch of query points the reference would pass to eval_raw is
handed to the field (``eval_raw_torch`` on the device when present, else
``eval_raw`` on a host copy).  The result must equal the oracle pipeline
driven by the same function, and the field's own exceptions must surface
unchanged (pipeline.py:154-240, fields.py:35-48)."""

import numpy as np
import pytest

import oracle
from paper_2409_13418_b200 import ContourOptions, GridSpec, contour
from paper_2409_13418_b200.pipeline import stage_arrays

pytestmark = pytest.mark.gpu


class Gyroid:
    """A user-defined field with no device program: a gyroid slab."""

    iso_level = 0.5
    continuous = False

    def __init__(self, scale=9.0, thick=0.6):
        self.scale, self.thick = scale, thick

    def eval_raw(self, p):
        p = np.asarray(p, dtype=np.float64) * self.scale
        g = np.sin(p[:, 0]) * np.cos(p[:, 1]) + np.sin(p[:, 1]) * np.cos(p[:, 2]) + np.sin(p[:, 2]) * np.cos(p[:, 0])
        r = np.linalg.norm(np.asarray(p) / self.scale - 0.5, axis=1)
        return ((np.abs(g) < self.thick) & (r < 0.42)).astype(np.float64)


class SoftBlob:
    """Continuous user field (raw values used by linear-interp / fd normals)."""

    iso_level = 0.5
    continuous = True

    def eval_raw(self, p):
        p = np.asarray(p, dtype=np.float64)
        d = np.linalg.norm(p - (0.5, 0.5, 0.5), axis=1) - 0.3 - 0.05 * np.sin(7 * p[:, 0])
        return 1.0 / (1.0 + np.exp(np.clip(25.0 * d, -500, 500)))


class TorchBox:
    """A field evaluated on the device by the user's own torch code; its
    numpy twin computes the same bits (comparisons of exact differences)."""

    iso_level = 0.5
    continuous = False
    c = (0.47, 0.52, 0.5)
    h = (0.21, 0.17, 0.26)

    def eval_raw_torch(self, p):
        import torch

        c = torch.tensor(self.c, dtype=torch.float64, device=p.device)
        h = torch.tensor(self.h, dtype=torch.float64, device=p.device)
        return ((p - c).abs() < h).all(dim=1).to(torch.float64)

    def eval_raw(self, p):
        p = np.asarray(p, dtype=np.float64)
        return (np.abs(p - np.asarray(self.c)) < np.asarray(self.h)).all(axis=1).astype(np.float64)


def _check(field, R, options=None):
    res, ctx, st = contour(field, GridSpec((0, 0, 0), (1, 1, 1), R), options, keep_intermediates=True,
                           return_context=True)
    arrs = stage_arrays(ctx, ["labels", "edge_key", "cells"])
    o = oracle.contour_oracle(field, (0, 0, 0), (1, 1, 1), R, options=options,
                              raw_fn=lambda p, cat: field.eval_raw(p), continuous=field.continuous)
    assert np.array_equal(arrs["labels"], o["labels"])
    assert np.array_equal(arrs["edge_key"], o["edge_key"])
    assert np.array_equal(arrs["cells"], o["cells"])
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    assert np.array_equal(res.mesh.vertices, o["vertices"])
    assert res.stats["eval_counts"] == o["eval_counts"]
    return res


def test_user_numpy_field_matches_oracle():
    res = _check(Gyroid(), 40)
    assert res.mesh.n_triangles > 1000


@pytest.mark.parametrize("opts", [dict(), dict(one_d="linear-interp"), dict(normals="fd-gradient")])
def test_user_continuous_field_modes(opts):
    _check(SoftBlob(), 33, ContourOptions(**opts))


def test_user_torch_field_stays_on_device():
    _check(TorchBox(), 37)


def test_user_field_exception_propagates():
    class Boom(Gyroid):
        calls = 0

        def eval_raw(self, p):
            Boom.calls += 1
            if Boom.calls == 3:
                raise KeyError("user field failed")
            return super().eval_raw(p)

    with pytest.raises(KeyError, match="user field failed"):
        contour(Boom(), GridSpec((0, 0, 0), (1, 1, 1), 24))


def test_user_field_wrong_length_raises():
    class Short(Gyroid):
        def eval_raw(self, p):
            return super().eval_raw(p)[:-1]

    with pytest.raises(ValueError, match="values for"):
        contour(Short(), GridSpec((0, 0, 0), (1, 1, 1), 16))


def test_reference_field_types_never_become_callbacks():
    """A CsgField with a child the device cannot lower raises LoweringError
    rather than silently evaluating on the host."""
    from paper_2409_13418_b200 import CsgField, SphereField
    from paper_2409_13418_b200.fields import LoweringError

    f = CsgField("union", [SphereField((0.5, 0.5, 0.5), 0.2), Gyroid()])
    with pytest.raises(LoweringError):
        contour(f, GridSpec((0, 0, 0), (1, 1, 1), 16))
