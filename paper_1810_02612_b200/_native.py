"""ctypes binding of include/ltlgrid_gpu.h (libltlgrid_gpu.so) -- no torch types.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no CPU fallback: if the library is missing, importing the
engine raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "_lib")
# the A/B build: the product library plus the variants reached only through
# dev knobs (csrc/Makefile); tests and dev tools load it with LTLG_DEV_SO
AB_SO = os.path.join(LIB_DIR, "libltlgrid_gpu_ab.so")
GPU_SO = os.environ.get("LTLG_DEV_SO") or os.path.join(LIB_DIR, "libltlgrid_gpu.so")

LTLG_OK, LTLG_EINVAL, LTLG_EFORMAT, LTLG_EIO, LTLG_ECUDA, LTLG_ENCCL, LTLG_ENOMEM, LTLG_ESTATE, LTLG_EDOMAIN = range(9)

# Every symbol include/ltlgrid_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "ltlg_create", "ltlg_create_ex", "ltlg_destroy", "ltlg_last_error", "ltlg_abi_version",
    "ltlg_load_abstraction", "ltlg_load_abstraction_file", "ltlg_load_abstraction_words",
    "ltlg_submit_grid", "ltlg_submit_grid_device", "ltlg_submit_world_grid", "ltlg_wait",
    "ltlg_get_labels", "ltlg_get_labels_packed", "ltlg_device_labels", "ltlg_get_info",
    "ltlg_stream", "ltlg_stage_times", "ltlg_validate_csr", "ltlg_label_all",
    "ltlg_submit_grid_files", "ltlg_save_labels", "ltlg_read_csb1_words", "ltlg_read_zobv",
    "ltlg_rasterize_boxes", "ltlg_submit_boxes", "ltlg_set_guards", "ltlg_get_admitted", "ltlg_device_admitted",
    "ltlg_submit_grid_device_ex",
    "ltlg_swept_volume", "ltlg_csr_rows", "ltlg_csr_cols", "ltlg_csr_nnz", "ltlg_csr_build_ms", "ltlg_csr_copy",
    "ltlg_load_csr", "ltlg_csr_free", "ltlg_set_profiling", "ltlg_generate_scenario", "ltlg_submit_scenario",
    "ltlg_csr_save", "ltlg_apply_labels", "ltlg_edge_counting", "ltlg_submit_grid_device_async",
]


class Options(C.Structure):
    _fields_ = [("sort_rows", C.c_int), ("stream_task_pairs", C.c_int), ("batch_task_pairs", C.c_int),
                ("profile", C.c_int), ("readback_chunks", C.c_int), ("task_rows", C.c_int), ("reserved", C.c_int * 5)]


class GridK(C.Structure):
    _fields_ = [("dims", C.c_int), ("depth", C.c_int), ("lo", C.c_double * 4), ("hi", C.c_double * 4)]


class Scenario(C.Structure):
    _fields_ = [("loop_cx", C.c_double), ("loop_cy", C.c_double), ("loop_radius", C.c_double),
                ("lane_width", C.c_double), ("agent_count", C.c_int), ("agent_speed_min", C.c_double),
                ("agent_speed_max", C.c_double), ("agent_length", C.c_double), ("agent_width", C.c_double),
                ("lateral_spread", C.c_double), ("horizon", C.c_double), ("seed", C.c_uint64)]


class Footprint(C.Structure):
    _fields_ = [("length", C.c_double), ("width", C.c_double), ("ref_offset", C.c_double)]


class Info(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64), ("words", C.c_uint64),
                ("pairs", C.c_uint64), ("t_bytes", C.c_uint64), ("n_devices", C.c_int), ("props", C.c_int),
                ("frames", C.c_int), ("label_bytes", C.c_int), ("label_words", C.c_int),
                ("reserved", C.c_int * 7)]


class Grid2(C.Structure):
    _fields_ = [("depth", C.c_int), ("lo0", C.c_double), ("hi0", C.c_double), ("lo1", C.c_double),
                ("hi1", C.c_double)]


class Pose2(C.Structure):
    _fields_ = [("dx", C.c_double), ("dy", C.c_double), ("cos_t", C.c_double), ("sin_t", C.c_double)]


class NativeMissing(ImportError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(GPU_SO):
        raise NativeMissing(
            f"{GPU_SO} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the labeling path has no CPU fallback)")
    L = C.CDLL(GPU_SO, mode=C.RTLD_GLOBAL)
    u64, i32, vp = C.c_uint64, C.c_int, C.c_void_p
    P64, P32 = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
    ctxp = C.c_void_p
    sig = {
        "ltlg_create": ([C.POINTER(i32), i32, C.POINTER(ctxp)], i32),
        "ltlg_create_ex": ([C.POINTER(i32), i32, C.POINTER(Options), C.POINTER(ctxp)], i32),
        "ltlg_destroy": ([ctxp], None),
        "ltlg_last_error": ([ctxp], C.c_char_p),
        "ltlg_abi_version": ([], i32),
        "ltlg_load_abstraction": ([ctxp, u64, u64, vp, vp], i32),
        "ltlg_load_abstraction_file": ([ctxp, C.c_char_p], i32),
        "ltlg_load_abstraction_words": ([ctxp, u64, u64, vp, vp, vp], i32),
        "ltlg_submit_grid": ([ctxp, u64, i32, vp, i32], i32),
        "ltlg_submit_grid_device": ([ctxp, u64, i32, vp, i32], i32),
        "ltlg_submit_grid_device_ex": ([ctxp, u64, i32, vp, i32, i32], i32),
        "ltlg_submit_grid_device_async": ([ctxp, u64, i32, vp, i32, i32, vp], i32),
        "ltlg_submit_world_grid": ([ctxp, C.POINTER(Grid2), C.POINTER(Grid2), i32, vp, i32, vp, i32, i32], i32),
        "ltlg_wait": ([ctxp], i32),
        "ltlg_get_labels": ([ctxp, i32, vp], i32),
        "ltlg_apply_labels": ([ctxp, i32, u64, i32, vp], i32),
        "ltlg_edge_counting": ([ctxp, i32, i32, vp, vp], i32),
        "ltlg_get_labels_packed": ([ctxp, vp, C.c_size_t], i32),
        "ltlg_device_labels": ([ctxp, i32, C.POINTER(vp), P64, P64, C.POINTER(i32)], i32),
        "ltlg_get_info": ([ctxp, C.POINTER(Info)], i32),
        "ltlg_stream": ([ctxp, i32, C.POINTER(vp)], i32),
        "ltlg_stage_times": ([ctxp, i32, i32, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float)], i32),
        "ltlg_validate_csr": ([u64, u64, vp, u64, vp, u64, C.c_char_p, C.c_size_t], i32),
        "ltlg_label_all": ([u64, u64, vp, vp, u64, i32, vp, i32, vp], i32),
        "ltlg_submit_grid_files": ([ctxp, C.POINTER(C.c_char_p), i32, i32], i32),
        "ltlg_save_labels": ([ctxp, i32, C.c_char_p], i32),
        "ltlg_read_csb1_words": ([C.c_char_p, P64, P64, P64, P64], i32),
        "ltlg_read_zobv": ([C.c_char_p, u64, vp], i32),
        "ltlg_rasterize_boxes": ([C.POINTER(GridK), i32, vp, vp, vp, i32, vp], i32),
        "ltlg_submit_boxes": ([ctxp, C.POINTER(GridK), i32, i32, vp, vp, vp], i32),
        "ltlg_set_guards": ([ctxp, i32, vp, vp], i32),
        "ltlg_get_admitted": ([ctxp, i32, vp], i32),
        "ltlg_device_admitted": ([ctxp, i32, C.POINTER(vp)], i32),
        "ltlg_swept_volume": ([C.POINTER(GridK), C.POINTER(Footprint), u64, vp, vp, i32, C.POINTER(vp)], i32),
        "ltlg_csr_rows": ([vp], u64),
        "ltlg_csr_cols": ([vp], u64),
        "ltlg_csr_nnz": ([vp], u64),
        "ltlg_csr_build_ms": ([vp], C.c_double),
        "ltlg_csr_copy": ([vp, vp, vp], i32),
        "ltlg_load_csr": ([ctxp, vp], i32),
        "ltlg_csr_free": ([vp], None),
        "ltlg_csr_save": ([vp, C.c_char_p], i32),
        "ltlg_set_profiling": ([ctxp, i32], i32),
        "ltlg_generate_scenario": ([C.POINTER(Scenario), C.POINTER(GridK), u64, i32, vp], i32),
        "ltlg_submit_scenario": ([ctxp, C.POINTER(Scenario), C.POINTER(GridK), u64, i32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    del P32
    _lib = L
    return L
