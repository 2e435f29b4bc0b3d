"""Benchmark and parity scenes in the reference's JSON scene schema
(/root/reference/pkg/src/occmesh/fields.py:401-477).

* The six analytic scenes of the reference's scene directory
  (sphere, smooth_sphere, torus, rotated_box, csg_union, csg_difference),
  restated as dicts so the package carries no files from the reference.
* ``thin_shell(R)`` -- BASELINE config 4: a rotated hollow box whose wall is
  ``cells`` grid cells thick.
* ``mlp`` -- BASELINE config 3: the positionally encoded MLP occupancy.
* ``batch_shapes(n)`` -- BASELINE config 5: n random analytic shapes inside
  [0.15, 0.85]^3, shape s drawn from numpy.random.default_rng(s).
"""

from __future__ import annotations

import numpy as np

_BOX_C = [0.5033, 0.4987, 0.4942]

SCENES = {
    "sphere": {"field": {"type": "sphere", "center": [0.5, 0.5, 0.5], "radius": 0.3}},
    "smooth_sphere": {
        "field": {"type": "sphere", "center": [0.5, 0.5, 0.5], "radius": 0.3},
        "smooth_k": "auto",
    },
    "torus": {"field": {"type": "torus", "center": [0.5, 0.5, 0.5], "major_radius": 0.27, "minor_radius": 0.12}},
    "rotated_box": {
        "field": {"type": "box", "center": _BOX_C, "half_extents": [0.2452, 0.1976, 0.1469],
                  "rotation_euler_deg": [30, 30, 0]}
    },
    "csg_union": {
        "field": {"type": "csg", "op": "union", "children": [
            {"type": "sphere", "center": [0.42, 0.5, 0.5], "radius": 0.22},
            {"type": "box", "center": [0.58, 0.5, 0.5], "half_extents": [0.18, 0.14, 0.14]},
        ]}
    },
    "csg_difference": {
        "field": {"type": "csg", "op": "difference", "children": [
            {"type": "box", "center": [0.5, 0.5, 0.46], "half_extents": [0.22, 0.18, 0.18]},
            {"type": "sphere", "center": [0.5, 0.5, 0.72], "radius": 0.16},
        ]}
    },
    "mlp": {"field": {"type": "mlp", "seed": 0, "amplitude": 1.0}},
}


def thin_shell(R, cells=2.5):
    """Hollow rotated box with a wall ``cells`` grid cells thick at resolution R."""
    outer = np.array([0.30, 0.24, 0.18])
    w = cells / float(R)
    inner = outer - w
    return {
        "field": {"type": "csg", "op": "difference", "children": [
            {"type": "box", "center": _BOX_C, "half_extents": outer.tolist(), "rotation_euler_deg": [30, 30, 0]},
            {"type": "box", "center": _BOX_C, "half_extents": inner.tolist(), "rotation_euler_deg": [30, 30, 0]},
        ]}
    }


SCENES["thin_shell"] = thin_shell(64)

# Thin rotated walls (thickness < one cell at the resolutions used with
# them): the 2D searches' step-2 arms come out parallel on some faces, so
# these exercise the midpoint-fallback status (search.py:280-313), and the
# second also range-exhausted searches.
SCENES["thin_wall"] = {"field": {"type": "box", "center": [0.543211, 0.511308, 0.484636],
                                 "half_extents": [0.209059, 0.170578, 0.009314],
                                 "rotation_euler_deg": [50.038, 51.628, 11.843]}}
SCENES["thin_wall_b"] = {"field": {"type": "box", "center": [0.573464, 0.526427, 0.562055],
                                   "half_extents": [0.244974, 0.207064, 0.005822],
                                   "rotation_euler_deg": [65.276, 58.848, 38.81]}}


def batch_shape(s):
    """Shape s of the config-5 batch: a random sphere, torus, box or CSG pair."""
    rng = np.random.default_rng(s)
    kind = ["sphere", "torus", "box", "csg"][s % 4]

    def center(margin):
        return rng.uniform(0.15 + margin, 0.85 - margin, size=3).round(6).tolist()

    def prim(k):
        if k == "sphere":
            r = round(float(rng.uniform(0.12, 0.3)), 6)
            return {"type": "sphere", "center": center(r), "radius": r}
        if k == "torus":
            R_ = round(float(rng.uniform(0.14, 0.22)), 6)
            r_ = round(float(rng.uniform(0.04, 0.1)), 6)
            return {"type": "torus", "center": center(R_ + r_), "major_radius": R_, "minor_radius": r_}
        half = rng.uniform(0.08, 0.2, size=3).round(6)
        ang = rng.uniform(0, 60, size=3).round(3).tolist()
        return {"type": "box", "center": center(float(np.linalg.norm(half))), "half_extents": half.tolist(),
                "rotation_euler_deg": ang}

    if kind != "csg":
        return {"field": prim(kind)}
    op = ["union", "intersection", "difference"][int(rng.integers(3))]
    return {"field": {"type": "csg", "op": op, "children": [prim("sphere"), prim("box")]}}


def batch_shapes(n=64):
    return [batch_shape(s) for s in range(n)]


def resolve(scene, R):
    """(field, lo, hi) for a scene dict at resolution R (Scene.resolve_field semantics)."""
    from .fields import field_from_dict, Scene

    doc = scene
    f = field_from_dict(doc["field"])
    dom = doc.get("domain", {})
    sc = Scene(f, smooth_k=doc.get("smooth_k"), domain_lo=dom.get("lo", (0, 0, 0)), domain_hi=dom.get("hi", (1, 1, 1)))
    lo, hi = tuple(sc.domain_lo.tolist()), tuple(sc.domain_hi.tolist())
    h = (np.asarray(hi) - np.asarray(lo)) / R
    return sc.resolve_field(h), lo, hi
