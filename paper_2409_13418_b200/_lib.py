"""ctypes binding of libodc (include/odc.h).  Fails loudly when the CUDA
library or a CUDA device is missing: there is no CPU fallback."""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libodc.so"

ODC_OK, ODC_E_ASSERT, ODC_E_CONTRACT, ODC_E_CONFIG, ODC_E_VALUE, ODC_E_CUDA, ODC_E_NOMEM, ODC_E_ARG, ODC_E_CALLBACK = range(9)
# int fn(void* user, const double* points, int64_t n, uint8_t* labels, double* raw, void* stream)
EVAL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p)
ODC_N_CAT = 6
CATEGORIES = ("labels", "search_1d", "probe_face_center", "probe_face_midpoint", "search_2d", "fd_gradient")

ARR = dict(
    labels=(0, np.uint8), edge_key=(1, np.int64), face_key=(2, np.int64), face_n_crossing=(3, np.int64),
    cells=(4, np.int64), instance_edges=(5, np.int64), t1d=(6, np.float64), pos1d=(7, np.float64),
    pos2=(8, np.float64), status=(9, np.uint8), part_cell=(10, np.int64), part_index=(11, np.int64),
    cyc_len=(12, np.int64), cyc_edges=(13, np.int64), cyc_insts=(14, np.int64), normals=(15, np.float64),
    qef_pos=(16, np.float64), qef_rank=(17, np.int64), qef_resid=(18, np.float64), split_cases=(19, np.int64),
    v_in=(20, np.int64), mid_label=(21, np.uint8), pos3=(22, np.float64), dup_source=(23, np.int64),
)


class Node(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("pad", ctypes.c_int32), ("p", ctypes.c_double * 16)]


class MlpDesc(ctypes.Structure):
    _fields_ = [
        ("d_in", ctypes.c_int32), ("width", ctypes.c_int32), ("depth", ctypes.c_int32), ("n_freq", ctypes.c_int32),
        ("w0", ctypes.c_void_p), ("w_hidden", ctypes.c_void_p), ("biases", ctypes.c_void_p), ("w_head", ctypes.c_void_p),
        ("b_head", ctypes.c_double), ("amplitude", ctypes.c_double), ("prior_scale", ctypes.c_double),
        ("prior_radius", ctypes.c_double), ("prior_center", ctypes.c_double * 3),
    ]


class Options(ctypes.Structure):
    _fields_ = [
        ("one_d", ctypes.c_int32), ("normals", ctypes.c_int32), ("split", ctypes.c_int32), ("repair", ctypes.c_int32),
        ("iters_1d", ctypes.c_int32), ("s1_lin", ctypes.c_int32), ("s1_bin", ctypes.c_int32),
        ("s2_lin", ctypes.c_int32), ("s2_bin", ctypes.c_int32), ("keep_intermediates", ctypes.c_int32),
        ("method", ctypes.c_int32), ("s1_range", ctypes.c_double), ("s2_range", ctypes.c_double), ("qef_truncation", ctypes.c_double),
        ("fd_step_factor", ctypes.c_double),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n_grid_vertices", ctypes.c_int64), ("boundary_inside_vertices", ctypes.c_int64),
        ("n_crossing_edges", ctypes.c_int64), ("n_crossing_faces", ctypes.c_int64),
        ("n_face_center_probes", ctypes.c_int64), ("n_crossing_cells", ctypes.c_int64),
        ("n_2d_points", ctypes.c_int64), ("n_partitions", ctypes.c_int64), ("n_plane_samples", ctypes.c_int64),
        ("point2d_status_counts", ctypes.c_int64 * 4), ("qef_rank_counts", ctypes.c_int64 * 4),
        ("split_case_counts", ctypes.c_int64 * 4), ("qef_max_residual", ctypes.c_double),
        ("normal_fallbacks", ctypes.c_int64), ("skipped_boundary_edges", ctypes.c_int64),
        ("raw_n_vertices", ctypes.c_int64), ("raw_n_triangles", ctypes.c_int64),
        ("n_vertices", ctypes.c_int64), ("n_triangles", ctypes.c_int64),
        ("repair_added_vertices", ctypes.c_int64), ("repair_passes", ctypes.c_int64),
        ("eval_batches", ctypes.c_int64 * ODC_N_CAT), ("eval_evals", ctypes.c_int64 * ODC_N_CAT),
        ("cat_order", ctypes.c_int32 * ODC_N_CAT), ("n_kernel_launches", ctypes.c_int32),
        ("device_ms", ctypes.c_float), ("stage_ms", ctypes.c_float * 8),
    ]


class SlabInfo(ctypes.Structure):
    _fields_ = [
        ("n_halo_partitions", ctypes.c_int64), ("n_partitions", ctypes.c_int64),
        ("n_window_partitions", ctypes.c_int64), ("n_fans", ctypes.c_int64), ("n_triangles", ctypes.c_int64),
        ("partition_vertices", ctypes.c_void_p), ("fan_vertices", ctypes.c_void_p), ("triangles", ctypes.c_void_p),
        ("partition_cell", ctypes.c_void_p), ("partition_index", ctypes.c_void_p), ("fan_edge", ctypes.c_void_p),
    ]


class ManifoldReport(ctypes.Structure):
    _fields_ = [("manifold", ctypes.c_int32), ("pad", ctypes.c_int32), ("n_nonmanifold_edges", ctypes.c_int64),
                ("n_pinched_vertices", ctypes.c_int64), ("n_boundary_edges", ctypes.c_int64),
                ("n_isolated_vertices", ctypes.c_int64)]


EXPORTS = (
    "odc_version", "odc_create", "odc_destroy", "odc_last_error", "odc_set_stream", "odc_field_analytic",
    "odc_field_mlp", "odc_field_free", "odc_default_options", "odc_extract", "odc_copy_mesh", "odc_copy_mesh_pair", "odc_mesh_device",
    "odc_copy_array", "odc_eval_raw", "odc_eval_labels", "odc_surface_probe", "odc_set_param", "odc_extract_slab",
    "odc_slab_globalize", "odc_mesh_finish", "odc_profile_mlp", "odc_export_obj", "odc_export_ply",
    "odc_validate_manifold", "odc_validate_copy", "odc_count_self_intersections", "odc_self_intersection_pairs",
    "odc_mesh_distance", "odc_triangle_areas", "odc_field_mesh", "odc_field_voxels", "odc_eigh3",
    "odc_eigh3_host", "odc_eval_mlp_dot", "odc_extract_batch", "odc_batch_layout", "odc_copy_batch_meshes",
    "odc_slab_seam", "odc_slab_local_finish", "odc_slab_top_ids", "odc_slab_final", "odc_field_callback",
)

_lib = None
_lock = threading.Lock()


def load():
    """Load libodc.so (build it with ``__graft_entry__.build()``)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(f"libodc.so not built at {LIB_PATH}; run __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        L.odc_version.restype = ctypes.c_int
        L.odc_create.argtypes = [ctypes.c_int, P(vp)]
        L.odc_destroy.argtypes = [vp]
        L.odc_destroy.restype = None
        L.odc_last_error.argtypes = [vp]
        L.odc_last_error.restype = ctypes.c_char_p
        L.odc_set_stream.argtypes = [vp, vp]
        L.odc_set_param.argtypes = [vp, ctypes.c_char_p, i64]
        L.odc_field_analytic.argtypes = [vp, P(Node), i32, i32, dbl, P(vp)]
        L.odc_field_mlp.argtypes = [vp, P(MlpDesc), P(vp)]
        L.odc_field_mesh.argtypes = [vp, vp, i64, vp, i64, P(vp)]
        L.odc_field_voxels.argtypes = [vp, P(dbl), P(dbl), vp, i64, i64, i64, P(vp)]
        L.odc_field_free.argtypes = [vp, vp]
        L.odc_field_callback.argtypes = [vp, EVAL_FN, vp, i32, dbl, P(vp)]
        L.odc_field_free.restype = None
        L.odc_default_options.argtypes = [P(Options)]
        L.odc_default_options.restype = None
        L.odc_extract.argtypes = [vp, vp, P(dbl), P(dbl), i64, P(Options), P(Stats)]
        L.odc_copy_mesh.argtypes = [vp, i32, vp, vp, vp, vp]
        L.odc_copy_mesh_pair.argtypes = [vp, vp, vp, vp, vp, vp]
        L.odc_mesh_device.argtypes = [vp, i32, P(vp), P(vp), P(i64), P(i64)]
        L.odc_copy_array.argtypes = [vp, i32, vp, i64, P(i64)]
        L.odc_eval_raw.argtypes = [vp, vp, vp, i64, vp]
        L.odc_eval_labels.argtypes = [vp, vp, vp, i64, vp]
        L.odc_surface_probe.argtypes = [vp, vp, vp, vp, i64, i64, vp]
        L.odc_eigh3.argtypes = [vp, vp, i64, vp, vp, vp]
        L.odc_eval_mlp_dot.argtypes = [vp, vp, vp, i64, vp]
        L.odc_eigh3_host.argtypes = [vp, i64, vp, vp, vp]
        L.odc_extract_slab.argtypes = [vp, vp, P(dbl), P(dbl), i64, P(Options), i64, i64, P(Stats), P(SlabInfo)]
        L.odc_extract_batch.argtypes = [vp, vp, i32, vp, vp, i64, P(Options), vp]
        L.odc_slab_seam.argtypes = [vp, vp, P(i64)]
        L.odc_slab_local_finish.argtypes = [vp, vp, i64, i64, P(i64), P(i64)]
        L.odc_slab_top_ids.argtypes = [vp, i64, i64, vp]
        L.odc_slab_final.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp]
        L.odc_batch_layout.argtypes = [vp, vp, vp, vp]
        L.odc_copy_batch_meshes.argtypes = [vp, vp, vp, vp, vp, vp]
        L.odc_slab_globalize.argtypes = [vp, i64, i64, i64, vp]
        L.odc_mesh_finish.argtypes = [vp, vp, i64, vp, i64, i64, vp, vp, i32, P(Stats)]
        L.odc_profile_mlp.argtypes = [vp, vp, i64, vp, i64]
        L.odc_validate_manifold.argtypes = [vp, vp, i64, i64, P(ManifoldReport)]
        L.odc_validate_copy.argtypes = [vp, vp, vp, vp]
        L.odc_count_self_intersections.argtypes = [vp, vp, i64, vp, i64, dbl, P(i64)]
        L.odc_self_intersection_pairs.argtypes = [vp, vp]
        L.odc_mesh_distance.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, vp, vp]
        L.odc_triangle_areas.argtypes = [vp, vp, i64, vp, i64, vp]
        L.odc_export_obj.argtypes = [ctypes.c_char_p, vp, i64, vp, i64]
        L.odc_export_ply.argtypes = [ctypes.c_char_p, vp, i64, vp, i64]
        _lib = L
        return L


class OdcFailure(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc, ctx=None):
    if rc == ODC_OK:
        return
    msg = load().odc_last_error(ctx).decode() if ctx else f"libodc error {rc}"
    raise OdcFailure(rc, msg)


_local = threading.local()  # per host thread: {device: Context}; freed with the thread


class Context:
    """One libodc context (device workspace + stream) per device and thread."""

    def __init__(self, device=0):
        L = load()
        self._L = L
        h = ctypes.c_void_p()
        rc = L.odc_create(int(device), ctypes.byref(h))
        if rc != ODC_OK:
            raise OdcFailure(rc, f"odc_create(device={device}) failed: no usable CUDA device (no CPU fallback)")
        self.handle = h
        self.device = device

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._L.odc_destroy(self.handle)
        except Exception:
            pass


def context(device=0):
    """This host thread's context on ``device`` (created on first use; it is
    destroyed when the thread's locals are, so short-lived threads do not
    accumulate device workspaces)."""
    ctxs = getattr(_local, "ctxs", None)
    if ctxs is None:
        ctxs = _local.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    return ctx
