"""Occupancy field descriptions and their lowering to device field programs.

Mirrors the reference's field API (/root/reference/pkg/src/occmesh/fields.py)
for the classes the extraction path uses -- constructor signatures, the
``iso_level`` / ``continuous`` attributes and the JSON scene schema
(fields.py:401-477) -- but the objects here are *descriptions*: they are
lowered to a postfix program (analytic / CSG / smoothed) or to packed bf16
weights (``MlpField``) and evaluated only on the GPU by libodc.  There is no
CPU evaluation path in this package.

Lowering is duck-typed on the class name and attributes, so reference
``occmesh`` field objects lower identically (that is how the parity tests
feed the same inputs to both sides).
"""

from __future__ import annotations

import json
import math
from fractions import Fraction
from pathlib import Path

import numpy as np

# opcodes: keep in sync with include/odc.h (ODC_OP_*)
OP_END = 0
OP_SPHERE_SD = 1
OP_BOX_SD = 2
OP_TORUS_SD = 3
OP_PLANE_SD = 4
OP_SD2RAW = 5
OP_RAW_MAX = 6
OP_RAW_MIN = 7
OP_RAW_DIFF = 8
OP_RAW_COMPL = 9
OP_SD_MIN = 10
OP_SD_MAX = 11
OP_SD_DIFF = 12
OP_SD_NEG = 13
OP_XFORM_BEGIN = 14
OP_XFORM_END = 15
OP_SMOOTH = 16

NODE_DTYPE = np.dtype([("op", "<i4"), ("pad", "<i4"), ("p", "<f8", (16,))])
MAX_NODES = 256
MAX_VALUE_STACK = 32
MAX_POINT_STACK = 8

_CSG_OPS = ("union", "intersection", "difference", "complement", "transform")


class OccupancyField:
    """Base class (fields.py:51-61): a pure point -> value description."""

    iso_level: float = 0.5
    continuous: bool = False


class AnalyticField(OccupancyField):
    """Exact signed distance, negative inside (fields.py:64-72)."""


class SphereField(AnalyticField):
    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.radius = float(radius)


class BoxField(AnalyticField):
    def __init__(self, center, half_extents, rotation=None):
        self.center = np.asarray(center, dtype=np.float64)
        self.half_extents = np.asarray(half_extents, dtype=np.float64)
        self.rotation = None if rotation is None else np.asarray(rotation, dtype=np.float64)


class TorusField(AnalyticField):
    def __init__(self, center, major_radius, minor_radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.major_radius = float(major_radius)
        self.minor_radius = float(minor_radius)


class PlaneField(AnalyticField):
    def __init__(self, point, normal):
        self.point = np.asarray(point, dtype=np.float64)
        n = np.asarray(normal, dtype=np.float64)
        self.normal = n / np.linalg.norm(n)


class CsgField(OccupancyField):
    """Boolean combination (fields.py:145-218)."""

    def __init__(self, op, children, rotation=None, translation=None):
        if op not in _CSG_OPS:
            raise ValueError(f"unknown CSG op {op!r}")
        children = tuple(children)
        if op == "complement" and len(children) != 1:
            raise ValueError("complement takes exactly one child")
        if op == "difference" and len(children) != 2:
            raise ValueError("difference takes exactly two children")
        if op == "transform" and len(children) != 1:
            raise ValueError("transform takes exactly one child")
        if op in ("union", "intersection") and len(children) < 2:
            raise ValueError(f"{op} takes at least two children")
        self.op = op
        self.children = children
        self.rotation = None if rotation is None else np.asarray(rotation, dtype=np.float64)
        self.translation = (
            np.zeros(3) if translation is None else np.asarray(translation, dtype=np.float64)
        )

    @property
    def continuous(self):
        return all(c.continuous for c in self.children)


class SmoothedOccupancy(OccupancyField):
    """raw = 1 / (1 + exp(k * sd)) (fields.py:221-242)."""

    continuous = True

    def __init__(self, base, sharpness):
        if not _has_signed_distance(base):
            raise TypeError("SmoothedOccupancy requires a base with signed_distance")
        self.base = base
        self.sharpness = float(sharpness)


def _fma(a, b, c):
    """Correctly rounded fused multiply-add (exact rational arithmetic)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _matmul3(a, b):
    """3x3 @ 3x3 with OpenBLAS dgemm's accumulation order on the reference
    host: c_ij = fma(a_i2, b_2j, fma(a_i1, b_1j, a_i0 * b_0j)).  Written out so
    the rotation matrix does not depend on the BLAS build of the host."""
    out = np.empty((3, 3))
    for i in range(3):
        for j in range(3):
            out[i, j] = _fma(a[i, 2], b[2, j], _fma(a[i, 1], b[1, j], a[i, 0] * b[0, j]))
    return out


def rotation_from_euler(rx_deg, ry_deg, rz_deg):
    """R = Rz @ Ry @ Rx from extrinsic xyz Euler angles (fields.py:389-398)."""
    rx, ry, rz = np.radians([rx_deg, ry_deg, rz_deg])
    cx, sx = math.cos(rx), math.sin(rx)
    cy, sy = math.cos(ry), math.sin(ry)
    cz, sz = math.cos(rz), math.sin(rz)
    mx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]], dtype=np.float64)
    my = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]], dtype=np.float64)
    mz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]], dtype=np.float64)
    return _matmul3(_matmul3(mz, my), mx)


class MlpField(OccupancyField):
    """Positionally encoded MLP occupancy (NEW: BASELINE config 3).

    Not in the reference; it subclasses the reference's ``OccupancyField``
    contract (fields.py:51-61) so ``contour`` accepts it unchanged.

      gamma(p) = [x, sin(2^k pi x), cos(2^k pi x)]_{k<n_freq},  x = p - 0.5
                 laid out as [x(3), sin_k0(3), cos_k0(3), sin_k1(3), ...] (39)
      h_0 = relu(gamma W_0 + b_0), h_i = relu(h_{i-1} W_i + b_i), i < depth
      mlp = h_{depth-1} w_head + b_head
      logit = amplitude * mlp - prior_scale * (|p - prior_center| - prior_radius)
      label = logit > 0, raw = sigmoid(logit) (continuous).

    Weights are He-normal from ``numpy.random.default_rng(seed)``, drawn in
    layer order as (fan_in, fan_out) arrays, then rounded to bf16 so the GPU
    (bf16 tensor cores) and any CPU evaluation see identical weight values.
    Biases are zero.
    """

    continuous = True

    def __init__(self, seed=0, n_freq=6, width=256, depth=8, amplitude=1.0,
                 prior_center=(0.5, 0.5, 0.5), prior_radius=0.3, prior_scale=40.0):
        if width != 256 or depth != 8 or n_freq != 6:
            raise ValueError("the device MLP is specialised to 8 x 256, n_freq = 6")
        self.seed = int(seed)
        self.n_freq = int(n_freq)
        self.width = int(width)
        self.depth = int(depth)
        self.amplitude = float(amplitude)
        self.prior_center = np.asarray(prior_center, dtype=np.float64)
        self.prior_radius = float(prior_radius)
        self.prior_scale = float(prior_scale)
        rng = np.random.default_rng(self.seed)
        d_in = 3 + 6 * self.n_freq
        dims = [d_in] + [width] * depth
        self.weights = []
        for i in range(depth):
            w = rng.standard_normal((dims[i], dims[i + 1])) * math.sqrt(2.0 / dims[i])
            self.weights.append(bf16_round(w))
        self.biases = [np.zeros(width, dtype=np.float32) for _ in range(depth)]
        self.w_head = bf16_round(rng.standard_normal((width, 1)) * math.sqrt(2.0 / width))[:, 0]
        self.b_head = 0.0

    @property
    def d_in(self):
        return 3 + 6 * self.n_freq

    @property
    def flops_per_eval(self):
        """Algorithmic FLOP per evaluation: 2*(39*256 + 7*256^2 + 256)."""
        w = self.width
        return 2 * (self.d_in * w + (self.depth - 1) * w * w + w)


def bf16_round(x):
    """Round float64/float32 values to the nearest bf16 (RNE), returned as float32."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    u = ((u + rounding) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


def _has_signed_distance(obj):
    return hasattr(obj, "signed_distance") or _kind(obj) in (
        "SphereField", "BoxField", "TorusField", "PlaneField", "CsgField", "SmoothedOccupancy",
    )


def _kind(field):
    return type(field).__name__


def field_continuous(field):
    if _kind(field) == "CsgField":
        return all(field_continuous(c) for c in field.children)
    return bool(getattr(field, "continuous", False))


class LoweringError(TypeError):
    pass


class SurfaceCoincidenceError(ValueError):
    """A winding-number query could not be moved off the surface (fields.py:21-22)."""


class MeshWindingField(OccupancyField):
    """Occupancy from a triangle mesh (fields.py:370-386): raw = generalized
    winding number, inside where raw > 1/2; queries exactly on the surface are
    perturbed deterministically.  Evaluated on the GPU (csrc/odc_winding.cu)."""

    continuous = True

    def __init__(self, vertices, triangles):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.triangles = np.asarray(triangles, dtype=np.int64)
        if len(self.triangles) == 0:
            raise ValueError("mesh field needs at least one triangle")


def is_mesh_winding(field):
    return _kind(field) == "MeshWindingField"


class VoxelField(OccupancyField):
    """Trilinear interpolation of a dense value grid, zero outside
    (fields.py:245-278).  Evaluated on the GPU (csrc/odc_voxel.cu)."""

    continuous = True

    def __init__(self, origin, spacing, values):
        self.origin = np.asarray(origin, dtype=np.float64)
        self.spacing = np.asarray(spacing, dtype=np.float64)
        self.values = np.asarray(values, dtype=np.float64)
        if self.values.ndim != 3:
            raise ValueError("voxel values must be a 3D array")


def is_voxels(field):
    return _kind(field) == "VoxelField"


def _node(op, params=()):
    n = np.zeros((), dtype=NODE_DTYPE)
    n["op"] = op
    p = np.zeros(16)
    p[: len(params)] = params
    n["p"] = p
    return n


def _rot_params(rot):
    if rot is None:
        return [0.0] + [0.0] * 9
    return [1.0] + list(np.asarray(rot, dtype=np.float64).reshape(9))


def _emit_sd(field, out):
    k = _kind(field)
    if k == "SphereField":
        out.append(_node(OP_SPHERE_SD, list(field.center) + [field.radius]))
    elif k == "BoxField":
        out.append(_node(OP_BOX_SD, list(field.center) + list(field.half_extents) + _rot_params(field.rotation)))
    elif k == "TorusField":
        out.append(_node(OP_TORUS_SD, list(field.center) + [field.major_radius, field.minor_radius]))
    elif k == "PlaneField":
        out.append(_node(OP_PLANE_SD, list(field.point) + list(field.normal)))
    elif k == "CsgField":
        op = field.op
        if op == "transform":
            out.append(_node(OP_XFORM_BEGIN, list(field.translation) + [0.0, 0.0, 0.0] + _rot_params(field.rotation)))
            _emit_sd(field.children[0], out)
            out.append(_node(OP_XFORM_END))
        elif op in ("union", "intersection"):
            _emit_sd(field.children[0], out)
            for c in field.children[1:]:
                _emit_sd(c, out)
                out.append(_node(OP_SD_MIN if op == "union" else OP_SD_MAX))
        elif op == "difference":
            _emit_sd(field.children[0], out)
            _emit_sd(field.children[1], out)
            out.append(_node(OP_SD_DIFF))
        else:
            _emit_sd(field.children[0], out)
            out.append(_node(OP_SD_NEG))
    elif k == "SmoothedOccupancy":
        _emit_sd(field.base, out)
    else:
        raise LoweringError(f"field {k} has no device signed distance")


def _emit_raw(field, out):
    k = _kind(field)
    if k in ("SphereField", "BoxField", "TorusField", "PlaneField"):
        _emit_sd(field, out)
        out.append(_node(OP_SD2RAW))
    elif k == "CsgField":
        op = field.op
        if op == "transform":
            out.append(_node(OP_XFORM_BEGIN, list(field.translation) + [0.0, 0.0, 0.0] + _rot_params(field.rotation)))
            _emit_raw(field.children[0], out)
            out.append(_node(OP_XFORM_END))
        elif op in ("union", "intersection"):
            _emit_raw(field.children[0], out)
            for c in field.children[1:]:
                _emit_raw(c, out)
                out.append(_node(OP_RAW_MAX if op == "union" else OP_RAW_MIN))
        elif op == "difference":
            _emit_raw(field.children[0], out)
            _emit_raw(field.children[1], out)
            out.append(_node(OP_RAW_DIFF))
        else:
            _emit_raw(field.children[0], out)
            out.append(_node(OP_RAW_COMPL))
    elif k == "SmoothedOccupancy":
        _emit_sd(field.base, out)
        out.append(_node(OP_SMOOTH, [field.sharpness]))
    else:
        raise LoweringError(
            f"cannot lower field type {k!r} to a device program; supported: sphere, box, "
            "torus, plane, csg, smoothed, MlpField (no CPU fallback exists)"
        )


def _check_stacks(prog):
    vs = ps = vmax = pmax = 0
    for n in prog:
        op = int(n["op"])
        if op in (OP_SPHERE_SD, OP_BOX_SD, OP_TORUS_SD, OP_PLANE_SD):
            vs += 1
        elif op in (OP_RAW_MAX, OP_RAW_MIN, OP_RAW_DIFF, OP_SD_MIN, OP_SD_MAX, OP_SD_DIFF):
            vs -= 1
        elif op == OP_XFORM_BEGIN:
            ps += 1
        elif op == OP_XFORM_END:
            ps -= 1
        vmax, pmax = max(vmax, vs), max(pmax, ps)
    if vmax > MAX_VALUE_STACK or pmax > MAX_POINT_STACK or len(prog) > MAX_NODES:
        raise LoweringError("field program too deep for the device interpreter")


def lower_program(field):
    """Postfix program (structured array of NODE_DTYPE) computing eval_raw."""
    out = []
    _emit_raw(field, out)
    prog = np.array(out, dtype=NODE_DTYPE)
    _check_stacks(prog)
    return prog


def is_mlp(field):
    return _kind(field) == "MlpField"


# ---------------------------------------------------------------------------
# scene files (fields.py:401-477)
# ---------------------------------------------------------------------------
def field_from_dict(spec, base_dir=None):
    if not isinstance(spec, dict) or "type" not in spec:
        raise ValueError("field spec must be a dict with a 'type' key")
    kind = spec["type"]
    if kind == "sphere":
        return SphereField(spec["center"], spec["radius"])
    if kind == "box":
        rot = None
        if "rotation_euler_deg" in spec:
            rot = rotation_from_euler(*spec["rotation_euler_deg"])
        return BoxField(spec["center"], spec["half_extents"], rotation=rot)
    if kind == "torus":
        return TorusField(spec["center"], spec["major_radius"], spec["minor_radius"])
    if kind == "plane":
        return PlaneField(spec["point"], spec["normal"])
    if kind == "csg":
        rot = None
        if "rotation_euler_deg" in spec:
            rot = rotation_from_euler(*spec["rotation_euler_deg"])
        children = [field_from_dict(c, base_dir) for c in spec["children"]]
        return CsgField(spec["op"], children, rotation=rot, translation=spec.get("translation"))
    if kind == "mlp":
        return MlpField(**{k: v for k, v in spec.items() if k != "type"})
    if kind == "mesh":  # fields.py:424-431
        from pathlib import Path

        from .meshio import import_obj

        path = Path(spec["path"])
        if base_dir is not None and not path.is_absolute():
            path = Path(base_dir) / path
        mesh = import_obj(path)
        return MeshWindingField(mesh.vertices, mesh.triangles)
    if kind == "voxels":  # fields.py:432-440
        from pathlib import Path

        if "path" in spec:
            path = Path(spec["path"])
            if base_dir is not None and not path.is_absolute():
                path = Path(base_dir) / path
            values = np.load(path)
        else:
            values = np.asarray(spec["values"], dtype=np.float64)
        return VoxelField(spec.get("origin", (0, 0, 0)), spec.get("spacing", (1, 1, 1)), values)
    raise ValueError(f"unknown field type {kind!r}")


class Scene:
    """Parsed scene: a field plus optional smoothing and domain box (fields.py:432-461)."""

    def __init__(self, field, smooth_k=None, domain_lo=(0, 0, 0), domain_hi=(1, 1, 1)):
        self.field = field
        self.smooth_k = smooth_k
        self.domain_lo = np.asarray(domain_lo, dtype=np.float64)
        self.domain_hi = np.asarray(domain_hi, dtype=np.float64)

    def resolve_field(self, cell_size):
        if self.smooth_k is None:
            return self.field
        k = self.smooth_k
        if k == "auto":
            k = 2.0 / float(np.min(cell_size))
        return SmoothedOccupancy(self.field, k)


def load_scene(path):
    path = Path(path)
    with open(path) as fh:
        doc = json.load(fh)
    if "field" not in doc:
        raise ValueError(f"{path}: scene file lacks a 'field' entry")
    field = field_from_dict(doc["field"], base_dir=path.parent)
    domain = doc.get("domain", {})
    return Scene(
        field,
        smooth_k=doc.get("smooth_k"),
        domain_lo=domain.get("lo", (0, 0, 0)),
        domain_hi=domain.get("hi", (1, 1, 1)),
    )
