"""Loader for libedgealign_b200.so (the C-ABI of include/edgealign_b200.h).

The library is built in-tree (paper_2112_05576_b200/build.py); there is no
fallback: importing the compute API without the built library, or calling it
without a CUDA device, raises.
"""
import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EAB_LIB_PATH") or os.path.join(HERE, "libedgealign_b200.so")

_lib = None

_P = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

# name -> (restype, argtypes); every ea_status function returns c_int
_SIGS = {
    "ea_last_error": (C.c_char_p, []),
    "ea_last_error_value": (C.c_double, []),
    "ea_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "ea_ctx_destroy": (None, [_P]),
    "ea_ctx_set_stream": (C.c_int, [_P, _P]),
    "ea_ctx_stream": (_P, [_P]),
    "ea_ctx_synchronize": (C.c_int, [_P]),
    "ea_ctx_last_stats": (C.c_int, [_P, C.POINTER(abi.SearchStats)]),
    "ea_ctx_kernel_launches": (C.c_uint64, [_P]),
    "ea_ctx_set_timing": (C.c_int, [_P, C.c_int]),
    "ea_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_P)]),
    "ea_host_free": (None, [_P]),
    "ea_compute_grid_counts": (C.c_int, [C.POINTER(abi.PoseGrid), C.POINTER(abi.GridCounts)]),
    "ea_pose_at": (C.c_int, [C.POINTER(abi.PoseGrid), C.c_uint64, C.POINTER(abi.Pose)]),
    "ea_max_pyramid_levels": (C.c_int, [C.c_int, C.c_int]),
    "ea_pyramid_dims": (C.c_int, [C.c_int, C.c_int, C.c_int, _ip]),
    "ea_downsample": (C.c_int, [_P, _dp, C.c_int, C.c_int, _dp]),
    "ea_build_pyramid": (C.c_int, [_P, _dp, C.c_int, C.c_int, C.c_int, _dp]),
    "ea_compute_gradients": (C.c_int, [_P, _dp, C.c_int, C.c_int, _dp, _dp, _dp]),
    "ea_field_upload": (C.c_int, [_P, _dp, _dp, _dp, C.c_int, C.c_int, C.POINTER(_P)]),
    "ea_field_from_image": (C.c_int, [_P, _dp, C.c_int, C.c_int, C.POINTER(_P)]),
    "ea_field_download": (C.c_int, [_P, _P, _dp, _dp, _dp]),
    "ea_field_dims": (C.c_int, [_P, _ip, _ip]),
    "ea_field_free": (None, [_P]),
    "ea_default_thresholds": (C.c_int, [_dp, C.c_int, C.c_int, C.POINTER(abi.EdgeThresholds)]),
    "ea_extract_edge_model": (C.c_int, [_dp, _dp, _dp, C.c_int, C.c_int,
                                        C.POINTER(abi.EdgeThresholds), C.c_int,
                                        C.POINTER(abi.EdgePoint), C.c_int, _ip, _dp, _dp]),
    "ea_model_create": (C.c_int, [_P, C.POINTER(abi.EdgePoint), C.c_int, C.c_double,
                                  C.c_double, C.c_int, C.POINTER(_P)]),
    "ea_model_size": (C.c_int, [_P]),
    "ea_field_extract_model": (C.c_int, [_P, _P, C.POINTER(abi.EdgeThresholds), C.c_int,
                                         C.POINTER(_P)]),
    "ea_model_points": (C.c_int, [_P, C.POINTER(abi.EdgePoint), C.c_int, _ip, _dp, _dp]),
    "ea_model_free": (None, [_P]),
    "ea_validate_params": (C.c_int, [C.POINTER(abi.ScoreParams)]),
    "ea_point_vote": (C.c_int, [_P, C.c_double, C.c_double, _P, C.c_int, C.c_int,
                                C.POINTER(abi.ScoreParams), _dp]),
    "ea_rotate_model": (C.c_int, [_P, _P, C.c_double, _dp, _dp, _dp, _dp]),
    "ea_pose_score": (C.c_int, [_P, _P, C.POINTER(abi.Pose), _P, C.POINTER(abi.ScoreParams),
                                _dp, _ip]),
    "ea_exhaustive_search": (C.c_int, [_P, _P, _P, C.POINTER(abi.PoseGrid),
                                       C.POINTER(abi.ScoreParams), C.c_int,
                                       C.POINTER(abi.ScoredPose)]),
    "ea_search_topk": (C.c_int, [_P, _P, _P, C.POINTER(abi.PoseGrid),
                                 C.POINTER(abi.ScoreParams), C.c_int, C.c_int,
                                 C.POINTER(abi.ScoredPose), _ip]),
    "ea_search_topk_slab": (C.c_int, [_P, _P, _P, C.POINTER(abi.PoseGrid),
                                      C.POINTER(abi.ScoreParams), C.c_int, C.c_uint64,
                                      C.c_uint64, C.POINTER(abi.ScoredPose), _ip]),
    "ea_merge_topk": (C.c_int, [C.POINTER(abi.ScoredPose), C.c_int, C.c_int,
                                C.POINTER(abi.ScoredPose), _ip]),
    "ea_score_map": (C.c_int, [_P, _P, _P, C.POINTER(abi.PoseGrid), C.POINTER(abi.ScoreParams),
                               C.c_uint64, _dp]),
    "ea_screen_map": (C.c_int, [_P, _P, _P, C.POINTER(abi.PoseGrid),
                                C.POINTER(abi.ScoreParams), C.c_uint64,
                                C.POINTER(C.c_float), _dp]),
    "ea_prepare_levels": (C.c_int, [_P, C.POINTER(_dp), _ip, C.c_int, C.POINTER(_dp), _ip,
                                    C.c_int, C.POINTER(abi.SearchConfig), C.POINTER(_P)]),
    "ea_prepare_models": (C.c_int, [_P, _dp, C.c_int, C.c_int, C.POINTER(abi.SearchConfig),
                                    C.POINTER(_P)]),
    "ea_levels_set_image": (C.c_int, [_P, _P, _dp, C.c_int, C.c_int]),
    "ea_levels_count": (C.c_int, [_P]),
    "ea_levels_model": (C.c_int, [_P, C.c_int, C.POINTER(abi.EdgePoint), C.c_int, _ip, _dp,
                                  _dp]),
    "ea_levels_field": (_P, [_P, C.c_int]),
    "ea_levels_get_model": (_P, [_P, C.c_int]),
    "ea_levels_free": (None, [_P]),
    "ea_search_levels": (C.c_int, [_P, _P, C.POINTER(abi.SearchConfig), C.POINTER(abi.Outcome)]),
    "ea_search_top_slab": (C.c_int, [_P, _P, C.POINTER(abi.SearchConfig), C.c_uint64,
                                     C.c_uint64, C.POINTER(abi.ScoredPose), _ip]),
    "ea_search_top_slab_async": (C.c_int, [_P, _P, C.POINTER(abi.SearchConfig), C.c_uint64,
                                           C.c_uint64, C.c_void_p]),
    "ea_merge_rows_async": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ea_ctx_async_status": (C.c_int, [_P, _ip, C.POINTER(C.c_float), C.c_int, _ip]),
    "ea_refine": (C.c_int, [_P, _P, C.POINTER(abi.SearchConfig), C.POINTER(abi.ScoredPose),
                            C.c_int, C.POINTER(abi.Outcome)]),
    "ea_coarse_to_fine": (C.c_int, [_P, C.POINTER(_dp), _ip, C.c_int, C.POINTER(_dp), _ip,
                                    C.c_int, C.POINTER(abi.SearchConfig),
                                    C.POINTER(abi.Outcome)]),
    "ea_detect": (C.c_int, [_P, _P, _dp, C.c_int, C.c_int, C.POINTER(abi.SearchConfig),
                            C.POINTER(abi.Outcome)]),
    "ea_detect_batch": (C.c_int, [_P, _P, C.POINTER(_dp), C.c_int, C.c_int, C.c_int,
                                  C.POINTER(abi.SearchConfig), C.POINTER(abi.Outcome)]),
    "ea_detect_multi": (C.c_int, [_P, C.POINTER(_P), C.c_int, _dp, C.c_int, C.c_int,
                                  C.POINTER(abi.SearchConfig), C.POINTER(abi.Outcome)]),
    "ea_theta_slab": (None, [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                             C.POINTER(C.c_uint64)]),
    "ea_comm_unique_id": (C.c_int, [C.POINTER(abi.CommId)]),
    "ea_comm_init": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(abi.CommId)]),
    "ea_comm_info": (C.c_int, [_P, _ip, _ip]),
    "ea_comm_destroy": (C.c_int, [_P]),
    "ea_gather_rows_async": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_void_p]),
    "ea_search_levels_sharded": (C.c_int, [_P, _P, C.POINTER(abi.SearchConfig),
                                           C.POINTER(abi.Outcome)]),
    "ea_detect_sharded": (C.c_int, [_P, _P, _dp, C.c_int, C.c_int,
                                    C.POINTER(abi.SearchConfig), C.POINTER(abi.Outcome)]),
    "ea_plan_multi": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _ip, C.c_int,
                                C.c_int, C.c_double, C.POINTER(abi.WorkItem), C.c_int, _ip]),
    "ea_gather_rows_multi_async": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ea_detect_multi_sharded": (C.c_int, [_P, C.POINTER(_P), C.c_int, _dp, C.c_int, C.c_int,
                                          C.POINTER(abi.SearchConfig), C.POINTER(abi.Outcome)]),
    "ea_render_template": (C.c_int, [C.c_int, C.c_int, _dp]),
    "ea_luminance_to_byte": (C.c_uint8, [C.c_double]),
    "ea_load_pgm": (C.c_int, [C.c_char_p, C.c_size_t, C.c_void_p, C.c_size_t, _ip, _ip]),
    "ea_save_pgm": (C.c_int, [_dp, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                              C.POINTER(C.c_size_t)]),
    "ea_save_ppm": (C.c_int, [_dp, C.c_int, C.c_int, _ip, C.c_int, C.c_uint8, C.c_uint8,
                              C.c_uint8, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ea_overlay_points": (C.c_int, [C.POINTER(abi.EdgePoint), C.c_int, C.POINTER(abi.Pose),
                                    _ip]),
    "ea_compose_multi": (C.c_int, [C.POINTER(abi.SceneSpec), C.POINTER(abi.Stamp), C.c_int,
                                   _dp]),
    "ea_compose_scene": (C.c_int, [C.POINTER(abi.SceneSpec), _dp, _dp, C.POINTER(abi.Pose),
                                   _dp]),
}


def _prefer_torch_nccl():
    """Point the library's run-time NCCL load (csrc/nccl_dl.cpp) at the copy
    torch links (the nvidia-nccl wheel), unless the caller chose one: a
    process that loads the system libnccl.so.2 first and imports torch later
    would hand torch that older copy (same soname) and break it."""
    if os.environ.get("EAB_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["EAB_NCCL_LIB"] = cand
            return


def lib():
    """The loaded C-ABI library (raises if it was never built)."""
    global _lib
    if _lib is None:
        _prefer_torch_nccl()
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2112_05576_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)
