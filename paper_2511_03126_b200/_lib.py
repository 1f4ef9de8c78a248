"""ctypes binding of the C ABI in include/propfield_b200.h.

This is the "reference-side binding" for a Python caller: the reference is a Python package, so a
ctypes stub over the extern "C" symbols is the natural FFI. Device buffers are
torch CUDA tensors (PyTorch is the allocator and stream provider only); no torch type crosses the
ABI. The library must load: there is no CPU fallback, and a missing/unbuildable .so or a missing
GPU raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import BundleLoadError, BundleStructureError, CudaError, MaterialError

_LIB_NAME = "libpropfield_b200.so"
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", _LIB_NAME)

PF_OK, PF_ERR_VALUE, PF_ERR_STRUCTURE, PF_ERR_MATERIAL, PF_ERR_CUDA, PF_ERR_LOAD = 0, 1, 2, 3, 4, 5
PF_F32, PF_BF16, PF_F64 = 0, 1, 2

PF_FUSE_WRITE_FEATURES = 1
PF_FUSE_WRITE_SIMS = 2
PF_FUSE_WRITE_WEIGHTS = 4
PF_FUSE_SKIP_VOXELS = 8
PF_FUSE_FORCE_SIMT = 16
PF_FUSE_PREPARED = 32
PF_FUSE_FEATURE_KERNEL = 64
PF_FUSE_DETERMINISTIC = 128

# pf_view_t (160 bytes)
VIEW_DTYPE = np.dtype(
    [
        ("R", "<f8", (9,)),
        ("t", "<f8", (3,)),
        ("fx", "<f8"),
        ("fy", "<f8"),
        ("cx", "<f8"),
        ("cy", "<f8"),
        ("depth_offset", "<i8"),
        ("fmap_offset", "<i8"),
        ("H", "<i4"),
        ("W", "<i4"),
        ("Hf", "<i4"),
        ("Wf", "<i4"),
    ],
    align=True,
)
assert VIEW_DTYPE.itemsize == 160


class FuseArgs(C.Structure):
    """pf_fuse_args_t — field order must match include/propfield_b200.h."""

    _fields_ = [
        ("points", C.c_void_p),
        ("n", C.c_int64),
        ("views", C.c_void_p),
        ("views_host", C.c_void_p),
        ("nviews", C.c_int32),
        ("depth", C.c_void_p),
        ("fmap", C.c_void_p),
        ("fmap_dtype", C.c_int32),
        ("d", C.c_int32),
        ("text", C.c_void_p),
        ("k", C.c_int32),
        ("values", C.c_void_p),
        ("p", C.c_int32),
        ("density_col", C.c_int32),
        ("mid_theta", C.c_void_p),
        ("temperature", C.c_double),
        ("eps", C.c_double),
        ("grid", C.c_int32),
        ("lo_hi", C.c_void_p),
        ("flags", C.c_uint32),
        ("counts", C.c_void_p),
        ("mask_bits", C.c_void_p),
        ("props", C.c_void_p),
        ("codes", C.c_void_p),
        ("grid_partials", C.c_void_p),
        ("partials", C.c_void_p),
        ("status", C.c_void_p),
        ("features", C.c_void_p),
        ("sims", C.c_void_p),
        ("weights", C.c_void_p),
        ("workspace", C.c_void_p),
        ("vox_list", C.c_void_p),
        ("vox_count", C.c_void_p),
        ("depth_ready", C.c_void_p),
        ("fmap_ready", C.c_void_p),
    ]


_P, _I32, _I64, _D, _U32 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint32

# symbol -> argtypes (every symbol declared in include/propfield_b200.h)
SIGNATURES = {
    "pf_last_error": ([], C.c_char_p),
    "pf_abi_version": ([], C.c_int),
    "pf_launch_count": ([], C.c_uint64),
    "pf_visible_in_view": ([_P, _P, _P, _I64, _P, _I32, _I32, _D, _P, _P], C.c_int),
    "pf_bilinear_gather": ([_P, _I32, _I32, _I32, _I32, _P, _P, _I64, _P, _P], C.c_int),
    "pf_accumulate_features": ([_P, _I32, _I32, _I32, _I32, _P, _P, _P, _I64, _P, _P, _P], C.c_int),
    "pf_project_points": ([_P, _I64, _P, _P, _P, _P], C.c_int),
    "pf_visibility_mask": ([_P, _I32, _I64, _P, _I32, _P, _D, _P, _P], C.c_int),
    "pf_aggregate_features": ([_P, _I32, _I64, _P, _I32, _P, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "pf_material_similarity": ([_P, _I64, _I32, _P, _I32, _P, _P], C.c_int),
    "pf_softmax_weights": ([_P, _I64, _I32, _D, _P, _P, _P, _P], C.c_int),
    "pf_regress_with_weights": ([_P, _I64, _I32, _P, _I32, _P, _P], C.c_int),
    "pf_bbox": ([_P, _I64, _P, _P], C.c_int),
    "pf_voxel_codes": ([_P, _I64, _P, _I32, _P, _P], C.c_int),
    "pf_voxel_accumulate": ([_P, _P, _I64, _I32, _P, _P], C.c_int),
    "pf_voxel_mass": ([_P, _I32, _P, _P, _P], C.c_int),
    "pf_fuse_workspace_bytes": ([C.POINTER(FuseArgs)], C.c_uint64),
    "pf_fuse_prepare": ([C.POINTER(FuseArgs), _P], C.c_int),
    "pf_fuse_query": ([C.POINTER(FuseArgs), _P], C.c_int),
    "pf_stage_timing": ([_I32], C.c_int),
    "pf_voxel_mass_sparse": ([_P, _I32, _P, _P, _I64, _P, _P, _P], C.c_int),
    "pf_knn_workspace_bytes": ([_I64], C.c_uint64),
    "pf_knn_kth_distance": ([_P, _I64, _I32, _P, _P, _P, _P], C.c_int),
    "pf_integrate_partials": ([_P, _I64, _I32, _P, _P, _P, _P, _P, _P], C.c_int),
    "pf_normals_workspace_bytes": ([_I64], C.c_uint64),
    "pf_estimate_normals": ([_P, _I64, _I32, _D, _D, _D, _P, _P, _P, _P], C.c_int),
    "pf_score_views": ([_P, _P, _I64, _P, _I32, _P, _P, _P, _P, _P, _I32, _P, _P], C.c_int),
    "pf_tb32_info": ([C.c_char_p, _P, _P], C.c_int),
    "pf_tb32_read": ([C.c_char_p, _P, _I64], C.c_int),
    "pf_ply_info": ([C.c_char_p, _P, _P], C.c_int),
    "pf_ply_read_points": ([C.c_char_p, _P, _P, _I64], C.c_int),
    "pf_dino_knn_workspace_bytes": ([_I64, _I64, _I32], C.c_uint64),
    "pf_dino_knn_interpolate": ([_P, _I64, _P, _I64, _I32, _P, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "pf_nearest_index": ([_P, _I64, _P, _I64, _P, _P], C.c_int),
    "pf_nearest_workspace_bytes": ([_I64], C.c_uint64),
    "pf_nearest_index_grid": ([_P, _I64, _P, _I64, _P, _P, _P], C.c_int),
    "pf_shard_bins": ([], C.c_int32),
    "pf_shard_keys": ([_P, _I64, _P, _I32, _P, _P, _P], C.c_int),
    "pf_shard_cuts": ([_P, _I32, _P, _P], C.c_int),
    "pf_shard_pack": ([_P, _I64, _P, _P, _I32, _P, _P, _P, _P], C.c_int),
    "pf_shard_xyz": ([_P, _I64, _P, _P], C.c_int),
    "pf_shard_pack_results": ([_I64, _I32, _I32, _P, _P, _P, _P, _P, _P], C.c_int),
    "pf_shard_unpack_results": ([_I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "pf_shard_pack_padded": ([_P, _I64, _P, _P, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "pf_shard_unpad": ([_P, _I32, _I32, _P, _P], C.c_int),
    "pf_shard_unpack_results_padded": ([_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "pf_allreduce_partials": ([_P, _I64, _P, _I64, _P, _P], C.c_int),
    "pf_nccl_comm_init_single": ([C.POINTER(C.c_void_p)], C.c_int),
    "pf_nccl_comm_destroy": ([_P], C.c_int),
    "pf_bench_umma": ([_I32, _I32, _I32, _I32, _P, _P], C.c_int),
    "pf_bench_gather": ([_P, _I32, _I32, _I32, _P, _P], C.c_int),
    "pf_stage_times": ([_P, _I32], C.c_int),
    "pf_tile_executed_flops": ([C.POINTER(FuseArgs), _P, _P], C.c_int),
    "pf_hilbert_table": ([_P, _I32], C.c_int),
    "pf_hilbert_keys": ([_P, _I64, _P, _I32, _P, _P], C.c_int),
    "pf_selftest_umma": ([_P, _P, _P, _I32, _I32, _I32, _P], C.c_int),
}

_lock = threading.Lock()
_lib = None


def load(path: str | None = None):
    """Load (once) and return the native library; raise loudly when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise CudaError(
                f"native library {p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)"
            )
        lib = C.CDLL(p)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.pf_abi_version() != 1:
            raise CudaError(f"ABI mismatch: {p} reports {lib.pf_abi_version()}")
        _lib = lib
        return lib


def check(status: int) -> None:
    """Map a pf_status to the reference's exception classes (errors.py:4-37)."""
    if status == PF_OK:
        return
    msg = load().pf_last_error().decode(errors="replace")
    if status == PF_ERR_VALUE:
        raise ValueError(msg)
    if status == PF_ERR_STRUCTURE:
        raise BundleStructureError(msg)
    if status == PF_ERR_MATERIAL:
        raise MaterialError(msg)
    if status == PF_ERR_LOAD:
        raise BundleLoadError(msg)
    raise CudaError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().pf_launch_count())


STAGES = ("sort", "prep", "tile_kernel", "unsort", "overflow_simt")


def stage_timing(enable: bool) -> None:
    """Start (True) / stop recording CUDA-event stage marks in every following pf_fuse_query."""
    check(load().pf_stage_timing(1 if enable else 0))


def stage_times() -> tuple[int, dict]:
    """(calls, {stage: summed device ms}) over the calls recorded since stage_timing(True)."""
    buf = (C.c_float * len(STAGES))()
    n = int(load().pf_stage_times(buf, len(STAGES)))
    if n < 0:
        check(-n)
    return n, {k: float(buf[i]) for i, k in enumerate(STAGES)}
