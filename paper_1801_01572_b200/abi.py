"""ctypes binding of the C ABI in include/loopkit_b200.h.

The shared libraries are built in-tree (``make -C paper_1801_01572_b200``)
into ``paper_1801_01572_b200/_lib/``. Loading fails loudly when they are
missing: there is no Python or CPU fallback for the device path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.environ.get("LK_LIB_OVERRIDE") or os.path.join(LIB_DIR, "libloopkit_b200.so")  # override: A/B experiments
SYNTH_PATH = os.path.join(LIB_DIR, "libloopkit_synth.so")

# lk_status (include/loopkit_b200.h), mirroring proj/include/loopkit/errors.hpp
LK_OK = 0
LK_NO_ALIGNMENT = 1
LK_EMPTY_CLOUD = 2
LK_TOO_FEW_POINTS = 3
LK_MISSING_DATA = 4
LK_MISSING_NORMALS = 5
LK_NO_CORRESPONDENCES = 6
LK_DEGENERATE = 7
LK_INVALID_ARGUMENT = 8
LK_CUDA_ERROR = 9
LK_NCCL_ERROR = 10
LK_ROTATION_TOO_LARGE = 11
LK_INTERNAL_ERROR = 99

dptr = C.POINTER(C.c_double)
fptr = C.POINTER(C.c_float)
i32ptr = C.POINTER(C.c_int32)
i64ptr = C.POINTER(C.c_int64)
u8ptr = C.POINTER(C.c_uint8)


class lk_cloud(C.Structure):
    _fields_ = [("xyz", dptr), ("nxyz", dptr), ("n", C.c_int64)]


class lk_reg_params(C.Structure):
    _fields_ = [
        ("leaf", C.c_double),
        ("normal_radius", C.c_double),
        ("feature_radius", C.c_double),
        ("hypothesis_count", C.c_int64),
        ("similarity_tau", C.c_double),
        ("d_max", C.c_double),
        ("min_inlier_ratio", C.c_double),
        ("max_fitness", C.c_double),
        ("normal_angle_max", C.c_double),
        ("seed", C.c_uint64),
        ("threads", C.c_int32),
        ("device", C.c_int32),
        ("device_count", C.c_int32),
        ("_reserved", C.c_int32),
    ]


class lk_reg_result(C.Structure):
    _fields_ = [
        ("R", C.c_double * 9),
        ("t", C.c_double * 3),
        ("inlier_ratio", C.c_double),
        ("fitness", C.c_double),
        ("inliers", C.c_int64),
        ("hypothesis_index", C.c_int64),
        ("found", C.c_int32),
        ("_pad", C.c_int32),
    ]


class lk_icp_params(C.Structure):
    _fields_ = [
        ("max_correspondence_distance", C.c_double),
        ("max_iterations", C.c_int32),
        ("device", C.c_int32),
        ("convergence_eps", C.c_double),
    ]


class lk_icp_result(C.Structure):
    _fields_ = [
        ("R", C.c_double * 9),
        ("t", C.c_double * 3),
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("correspondences", C.c_int64),
        ("rmse", C.c_double),
        ("fitness", C.c_double),
    ]


class lk_verify_params(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("overlap_radius", C.c_double),
        ("d_max", C.c_double),
        ("grid_cell", C.c_double),
        ("normal_angle_max", C.c_double),
        ("device", C.c_int32),
        ("device_count", C.c_int32),
    ]


class lk_loop_params(C.Structure):
    _fields_ = [("overlap_radius", C.c_double), ("min_overlap", C.c_double), ("device", C.c_int32),
                ("_pad", C.c_int32)]


class lk_loop_proposal(C.Structure):
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("overlap", C.c_double)]


class lk_verify_result(C.Structure):
    _fields_ = [
        ("info", C.c_double * 36),
        ("pair_count", C.c_int64),
        ("overlap_hits", C.c_int64),
        ("overlap", C.c_double),
        ("inliers", C.c_int64),
        ("inlier_ratio", C.c_double),
        ("fitness", C.c_double),
    ]


class lk_hyp_stats(C.Structure):
    _fields_ = [
        ("sampled", C.c_int64),
        ("prerejected", C.c_int64),
        ("degenerate", C.c_int64),
        ("evaluated", C.c_int64),
        ("qualified", C.c_int64),
        ("w_ref", C.c_int64),
        ("evals_executed", C.c_int64),
        ("prepare_seconds", C.c_double),
        ("hypothesis_seconds", C.c_double),
    ]


class lk_reg_record(C.Structure):
    _fields_ = [
        ("valid", C.c_int64),
        ("inliers", C.c_int64),
        ("fitness", C.c_double),
        ("index", C.c_int64),
        ("R", C.c_double * 9),
        ("t", C.c_double * 3),
        ("sampled", C.c_int64),
        ("prerejected", C.c_int64),
        ("degenerate", C.c_int64),
        ("evaluated", C.c_int64),
        ("qualified", C.c_int64),
        ("w_ref", C.c_int64),
        ("evals_executed", C.c_int64),
        ("_reserved", C.c_int64),
    ]


assert C.sizeof(lk_reg_record) == 192


class lk_cand_score(C.Structure):
    _fields_ = [("inlier_ratio", C.c_double), ("fitness", C.c_double), ("inliers", C.c_int64)]


# name -> (restype, argtypes); every symbol declared in include/loopkit_b200.h
SIGNATURES = {
    "lk_abi_version": (C.c_int, []),
    "lk_last_error": (C.c_char_p, []),
    "lk_device_count": (C.c_int, []),
    "lk_reg_prepare": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), C.POINTER(lk_reg_params),
                                 C.POINTER(C.c_void_p)]),
    "lk_reg_ctx_create": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), i32ptr, C.POINTER(lk_reg_params),
                                    C.POINTER(C.c_void_p)]),
    "lk_reg_ctx_destroy": (None, [C.c_void_p]),
    "lk_reg_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "lk_reg_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "lk_reg_ctx_kernel_times": (C.c_int, [C.c_void_p, dptr, i64ptr, C.c_int32]),
    "lk_reg_ctx_phase_times": (C.c_int, [C.c_void_p, dptr, C.c_int32, i64ptr, C.c_int32]),
    "lk_reg_ctx_sizes": (C.c_int, [C.c_void_p, i64ptr, i64ptr]),
    "lk_reg_ctx_download": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, i32ptr, fptr, fptr]),
    "lk_reg_run_hypotheses": (C.c_int, [C.c_void_p, C.POINTER(lk_reg_params), C.POINTER(lk_reg_result),
                                        C.POINTER(lk_hyp_stats)]),
    "lk_reg_run_range": (C.c_int, [C.c_void_p, C.POINTER(lk_reg_params), C.c_int64, C.c_int64, C.c_void_p,
                                   C.c_int32]),
    "lk_reg_merge_records": (C.c_int, [C.POINTER(lk_reg_record), C.c_int32, C.c_int64, C.POINTER(lk_reg_result),
                                       C.POINTER(lk_hyp_stats)]),
    "lk_register_global": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), C.POINTER(lk_reg_params),
                                     C.POINTER(lk_reg_result), C.POINTER(lk_hyp_stats)]),
    "lk_grid_build": (C.c_int, [C.POINTER(lk_cloud), C.c_int32, C.c_double, C.c_double, C.c_int32,
                                C.POINTER(C.c_void_p)]),
    "lk_grid_destroy": (None, [C.c_void_p]),
    "lk_grid_dims": (C.c_int, [C.c_void_p, dptr, dptr, i32ptr, i64ptr, i64ptr]),
    "lk_grid_download": (C.c_int, [C.c_void_p, i32ptr, i32ptr, dptr, dptr, u8ptr]),
    "lk_score_candidates": (C.c_int, [C.c_void_p, C.POINTER(lk_cloud), dptr, C.c_int64, C.POINTER(lk_reg_params),
                                      C.c_int32, C.POINTER(lk_cand_score), C.POINTER(lk_reg_result), i64ptr]),
    "lk_edge_info_batched": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), dptr, dptr, C.c_int64, C.c_double,
                                       C.c_int32, dptr, i64ptr]),
    "lk_feature_nn_cache": (C.c_int, [fptr, C.c_int64, fptr, C.c_int64, C.c_int32, i32ptr]),
    "lk_edge_residual": (C.c_int, [dptr, dptr, dptr, dptr, dptr]),
    "lk_update_weight": (C.c_double, [C.c_double, C.c_double]),
    "lk_loop_weights": (C.c_int, [C.c_int64, dptr, dptr, dptr, dptr, C.POINTER(C.c_int64), C.c_double, C.c_double,
                                  dptr, C.POINTER(C.c_int32)]),
    "lk_verify_batch": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), dptr, dptr, dptr, C.c_int64,
                                  C.POINTER(lk_verify_params), C.POINTER(lk_verify_result)]),
    "lk_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "lk_reg_ctx_attach_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32]),
    "lk_reg_run_exchange": (C.c_int, [C.c_void_p, C.POINTER(lk_reg_params), C.c_void_p]),
    "lk_reg_ctx_topology": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "lk_propose_loops": (C.c_int, [C.POINTER(lk_cloud), dptr, C.c_int32, i32ptr, C.c_int32, C.POINTER(lk_loop_params),
                                   C.POINTER(lk_loop_proposal), C.c_int64, i64ptr]),
    "lk_icp_point_to_plane": (C.c_int, [C.POINTER(lk_cloud), C.POINTER(lk_cloud), dptr, C.POINTER(lk_icp_params),
                                        C.POINTER(lk_icp_result), dptr]),
    "lk_estimate_normals": (C.c_int, [C.POINTER(lk_cloud), C.c_double, dptr, C.c_int32, dptr]),
    "lk_voxel_downsample": (C.c_int, [C.POINTER(lk_cloud), C.c_double, dptr, dptr, i64ptr]),
    "lk_compute_fpfh": (C.c_int, [C.POINTER(lk_cloud), C.c_double, C.c_int32, fptr]),
}

SYNTH_SIGNATURES = {
    "lks_last_error": (C.c_char_p, []),
    "lks_registration_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.POINTER(C.c_int)]),
    "lks_negative_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.POINTER(C.c_int)]),
    "lks_frame_pair": (C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "lks_surface_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_int)]),
    "lks_submap_pair": (C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                     C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "lks_random_cloud": (C.c_void_p, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int,
                                      C.POINTER(C.c_int)]),
    "lks_count": (C.c_int64, [C.c_void_p, C.c_int]),
    "lks_has_normals": (C.c_int, [C.c_void_p, C.c_int]),
    "lks_get": (None, [C.c_void_p, C.c_int, dptr, dptr]),
    "lks_truth": (None, [C.c_void_p, dptr, dptr, dptr]),
    "lks_free": (None, [C.c_void_p]),
    "lks_transform_from_twist": (None, [dptr, dptr, dptr]),
    "lks_compose": (None, [dptr, dptr, dptr, dptr, dptr, dptr]),
    "lks_inverse": (None, [dptr, dptr, dptr, dptr]),
    "lks_apply": (None, [dptr, dptr, dptr, C.c_int64, dptr]),
    "lks_rotate": (None, [dptr, dptr, C.c_int64, dptr]),
    "lks_random_transform": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double, dptr, dptr]),
    "lks_angle_axis": (None, [C.c_double, dptr, dptr]),
}

_lib = None
_synth = None


def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)  # AttributeError -> a declared symbol is missing
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The device library. Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                "(the B200 path has no CPU fallback)")
        _lib = _bind(C.CDLL(LIB_PATH), SIGNATURES)
    return _lib


def synth_lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing: build it with `make -C {_HERE}`")
        _synth = _bind(C.CDLL(SYNTH_PATH), SYNTH_SIGNATURES)
    return _synth


def last_error() -> str:
    msg = lib().lk_last_error()
    return msg.decode() if msg else ""


def prefer_process_nccl() -> None:
    """The library opens libnccl.so.2 on first NCCL use and reuses one already
    in the process (lk_abi.cu nccl()). If PyTorch is installed but not yet
    imported, import it first so that its bundled NCCL is the one loaded:
    otherwise a later `import torch` would bind to the system NCCL already in
    the process and fail on missing symbols."""
    import sys
    if "torch" not in sys.modules:
        try:
            import torch  # noqa: F401
        except Exception:
            pass
