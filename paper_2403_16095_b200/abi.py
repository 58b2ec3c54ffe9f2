"""ctypes view of the C-ABI declared in include/gsf_cuda.h.

The product library is ``paper_2403_16095_b200/libgsf_cuda.so`` (built by
``__graft_entry__.build()``).  There is no CPU fallback: if the library is missing, or no
CUDA device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GSF_LIB: an alternative in-tree build of the same library (kernel-variant A/B measurements)
LIB_PATH = os.environ.get("GSF_LIB") or os.path.join(HERE, "libgsf_cuda.so")

GSF_OK, GSF_EINVAL, GSF_ENONFINITE, GSF_EDIVERGED, GSF_ECUDA, GSF_EUNSUPPORTED, GSF_ENOMEM, GSF_ERUNTIME = range(8)

dp = C.POINTER(C.c_double)
fp = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_scale", C.c_double),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class RasterCfg(C.Structure):
    _fields_ = [("alpha_clamp", C.c_double), ("alpha_skip", C.c_double),
                ("termination_threshold", C.c_double), ("footprint_sigma", C.c_double),
                ("dilation", C.c_double), ("tile_size", C.c_int32),
                ("uncertainty_full_gradient", C.c_int32), ("threads", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("rotation_tangent", C.c_double * 3), ("translation", C.c_double * 3)]


class LossWeights(C.Structure):
    _fields_ = [("w_color", C.c_double), ("w_ssim", C.c_double), ("w_geo", C.c_double),
                ("w_align", C.c_double), ("w_iso", C.c_double), ("w_var", C.c_double),
                ("t_color", C.c_double), ("t_geo", C.c_double), ("iso_epsilon", C.c_double),
                ("opacity_floor", C.c_double), ("normalize_by_valid", C.c_int32)]


class TrackerCfg(C.Structure):
    _fields_ = [("lr_rotation", C.c_double), ("lr_translation", C.c_double),
                ("iterations", C.c_int32), ("ba_window", C.c_int32), ("ba_iterations", C.c_int32),
                ("keyframe_interval", C.c_int32), ("recent_keyframes", C.c_int32),
                ("freeze_oldest_pose", C.c_int32), ("degraded_loss_ratio", C.c_double)]


class MapperCfg(C.Structure):
    _fields_ = [("sh_coeffs", C.c_int32), ("scene_extent", C.c_double), ("lr_mean", C.c_double),
                ("lr_sh", C.c_double), ("lr_opacity", C.c_double), ("lr_scale", C.c_double),
                ("lr_rotation", C.c_double), ("densify_interval", C.c_int32),
                ("densify_grad_threshold", C.c_double), ("densify_split_factor", C.c_double),
                ("densify_size_fraction", C.c_double), ("densify_cull_opacity", C.c_double),
                ("uncertainty_tau", C.c_double), ("uncertainty_reduced_opacity", C.c_double),
                ("seed", C.c_uint64), ("raster", RasterCfg), ("weights", LossWeights),
                ("init_stride", C.c_int32), ("spawn_stride", C.c_int32),
                ("spawn_opacity_threshold", C.c_double), ("init_opacity", C.c_double)]


class StructuralChange(C.Structure):
    _fields_ = [("split", C.c_int32), ("cloned", C.c_int32), ("removed", C.c_int32)]


class SlamCfg(C.Structure):
    _fields_ = [("intrinsics", Intrinsics), ("tracker", TrackerCfg), ("mapper", MapperCfg),
                ("map_iterations", C.c_int32), ("init_iterations", C.c_int32), ("seed", C.c_uint64)]


class FrameLog(C.Structure):
    _fields_ = [("frame", C.c_int32), ("timestamp", C.c_double), ("track_loss", C.c_double),
                ("track_iterations", C.c_int32), ("track_degraded", C.c_int32), ("keyframe", C.c_int32),
                ("primitives", C.c_int64), ("track_ms", C.c_double), ("map_ms", C.c_double), ("ba_ms", C.c_double),
                ("uncertainty_ms", C.c_double), ("spawn_ms", C.c_double), ("kf_psnr_db", C.c_double),
                ("kf_depth_l1_cm", C.c_double), ("pose", Pose)]


class MapHost(C.Structure):
    _fields_ = [("count", C.c_int64), ("sh_coeffs", C.c_int32), ("mean", dp), ("log_scale", dp),
                ("quat", dp), ("opacity_logit", dp), ("sh", dp), ("uncertainty", dp),
                ("observed", u8p)]


class RenderOut(C.Structure):
    _fields_ = [("color", fp), ("alpha_depth", fp), ("median_depth", fp), ("median_valid", u8p),
                ("opacity", fp), ("uncertainty", fp), ("final_transmittance", fp),
                ("per_pixel_count", i32p), ("dominant", i32p), ("median_prim", i32p),
                ("dominant_weight", fp), ("visible", u8p), ("has_uncertainty", C.c_int32),
                ("num_visible", C.c_int64), ("num_pairs", C.c_int64)]


class Upstream(C.Structure):
    _fields_ = [("d_color", fp), ("d_alpha_depth", fp), ("d_median_depth", fp),
                ("d_opacity", fp), ("d_uncertainty", fp)]


class GradsOut(C.Structure):
    _fields_ = [("d_mean", fp), ("d_log_scale", fp), ("d_quat", fp), ("d_opacity_logit", fp),
                ("d_sh", fp), ("d_mean2d", fp), ("d_pose", C.c_double * 6)]


class TrackResult(C.Structure):
    _fields_ = [("pose", Pose), ("final_loss", C.c_double), ("degraded", C.c_int32),
                ("iterations_run", C.c_int32), ("initial_loss", C.c_double)]


class LossTerms(C.Structure):
    _fields_ = [("color", C.c_double), ("ssim", C.c_double), ("geo", C.c_double),
                ("align", C.c_double), ("iso", C.c_double), ("var", C.c_double),
                ("total", C.c_double), ("valid_color", C.c_int32), ("valid_geo", C.c_int32),
                ("any_empty_mask", C.c_int32)]


# name -> (restype, argtypes); every symbol declared in include/gsf_cuda.h
SIGNATURES = {
    "gsf_abi_version": (C.c_int, []),
    "gsf_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "gsf_ctx_destroy": (C.c_int, [C.c_void_p]),
    "gsf_last_error": (C.c_char_p, [C.c_void_p]),
    "gsf_last_error_index": (C.c_int64, [C.c_void_p]),
    "gsf_kernel_launches": (C.c_int64, [C.c_void_p]),
    "gsf_track_candidates": (C.c_int64, [C.c_void_p]),
    "gsf_reserve": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
    "gsf_capacity": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "gsf_synchronize": (C.c_int, [C.c_void_p]),
    "gsf_profile_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "gsf_profile_read": (C.c_int, [C.c_void_p, C.c_int32, dp, i64p]),
    "gsf_event_record": (C.c_int, [C.c_void_p, C.c_int32]),
    "gsf_event_elapsed": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, dp]),
    "gsf_map_upload": (C.c_int, [C.c_void_p, C.POINTER(MapHost)]),
    "gsf_map_download": (C.c_int, [C.c_void_p, C.POINTER(MapHost)]),
    "gsf_map_count": (C.c_int64, [C.c_void_p]),
    "gsf_map_sh_coeffs": (C.c_int32, [C.c_void_p]),
    "gsf_optimizer_reset": (C.c_int, [C.c_void_p]),
    "gsf_render": (C.c_int, [C.c_void_p, C.POINTER(Pose), C.POINTER(Intrinsics), fp,
                             C.POINTER(RasterCfg), C.POINTER(RenderOut)]),
    "gsf_render_backward": (C.c_int, [C.c_void_p, C.POINTER(Upstream), fp, C.POINTER(GradsOut)]),
    "gsf_render_record": (C.c_int, [C.c_void_p, u32p, i32p, fp, fp, i64p]),
    "gsf_render_tiles": (C.c_int, [C.c_void_p, i32p, C.c_int64, i32p, C.c_int64]),
    "gsf_tracking_loss": (C.c_int, [C.c_void_p, fp, fp, C.POINTER(LossWeights),
                                    C.POINTER(LossTerms), fp, fp]),
    "gsf_mapping_loss": (C.c_int, [C.c_void_p, fp, fp, C.POINTER(LossWeights),
                                   C.POINTER(LossTerms), fp, fp, fp, fp, fp]),
    "gsf_ssim": (C.c_int, [C.c_void_p, fp, fp, C.c_int32, C.c_int32, dp, fp]),
    "gsf_frame_upload": (C.c_int, [C.c_void_p, C.c_int32, fp, fp, C.c_int32, C.c_int32]),
    "gsf_track_frame": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Pose), C.POINTER(Intrinsics),
                                  C.POINTER(TrackerCfg), C.POINTER(LossWeights),
                                  C.POINTER(RasterCfg), C.POINTER(TrackResult)]),
    "gsf_tracking_gradient": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Pose), C.POINTER(Intrinsics),
                                        C.POINTER(LossWeights), C.POINTER(RasterCfg), C.POINTER(LossTerms),
                                        C.POINTER(C.c_double * 6)]),
    "gsf_track_frame_host": (C.c_int, [C.c_void_p, fp, fp, C.POINTER(Pose), C.POINTER(Intrinsics),
                                       C.POINTER(TrackerCfg), C.POINTER(LossWeights),
                                       C.POINTER(RasterCfg), C.POINTER(TrackResult)]),
    "gsf_map_step": (C.c_int, [C.c_void_p, i32p, C.POINTER(Pose), C.c_int32, C.POINTER(Intrinsics),
                               C.POINTER(MapperCfg), C.c_int32, dp]),
    "gsf_sliding_ba": (C.c_int, [C.c_void_p, i32p, C.POINTER(Pose), i32p, C.c_int32,
                                 C.POINTER(Intrinsics), C.POINTER(TrackerCfg), C.POINTER(MapperCfg),
                                 C.c_int32, dp]),
    "gsf_initialize_map": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Pose), C.POINTER(Intrinsics),
                                     C.POINTER(MapperCfg), C.POINTER(C.c_int64)]),
    "gsf_spawn_gaussians": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Pose), C.POINTER(Intrinsics),
                                      C.POINTER(MapperCfg), C.POINTER(C.c_int32)]),
    "gsf_render_reference": (C.c_int, [C.c_void_p, C.POINTER(Pose), C.POINTER(Intrinsics), fp, C.POINTER(RasterCfg),
                                       C.POINTER(RenderOut)]),
    "gsf_checkpoint_save": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(Intrinsics)]),
    "gsf_checkpoint_load": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(Intrinsics)]),
    "gsf_slam_create": (C.c_int, [C.c_void_p, C.POINTER(SlamCfg), C.POINTER(C.c_void_p)]),
    "gsf_slam_destroy": (C.c_int, [C.c_void_p]),
    "gsf_slam_process": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, fp, fp, C.POINTER(FrameLog)]),
    "gsf_slam_keyframes": (C.c_int32, [C.c_void_p]),
    "gsf_slam_degraded_frames": (C.c_int32, [C.c_void_p]),
    "gsf_densify_and_cull": (C.c_int, [C.c_void_p, C.POINTER(MapperCfg), C.POINTER(StructuralChange)]),
    "gsf_map_stats_upload": (C.c_int, [C.c_void_p, dp, i32p]),
    "gsf_map_stats_download": (C.c_int, [C.c_void_p, dp, i32p]),
    "gsf_accumulate_uncertainty": (C.c_int, [C.c_void_p, i32p, C.POINTER(Pose), C.c_int32,
                                             C.POINTER(Intrinsics), C.POINTER(RasterCfg), i32p]),
    "gsf_prune_unreliable": (C.c_int, [C.c_void_p, C.c_double, C.c_double, i32p]),
    "gsf_ba_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, u8p]),
    "gsf_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8 * 128)]),
    "gsf_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_uint8 * 128)]),
    "gsf_comm_init_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
}

# gsf_host_allreduce_fn: int (*)(void* buf, size_t count, int32_t dtype, void* user)
HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
GSF_DT_U32, GSF_DT_F32, GSF_DT_F64 = 3, 7, 8

_lib = None


class GsfError(RuntimeError):
    """Raised for a non-OK status; .status carries the gsf_status code."""

    def __init__(self, status: int, message: str, index: int = -1):
        super().__init__(message)
        self.status = status
        self.index = index


def load() -> C.CDLL:
    """Load libgsf_cuda.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def defaults_raster() -> RasterCfg:
    """RasterConfig defaults (raster/config.hpp:5-16)."""
    return RasterCfg(0.99, 1.0 / 255.0, 1e-8, 3.0, 0.3, 16, 1, 0)


def defaults_weights(handheld_real: bool = False) -> LossWeights:
    """LossWeights::indoor_synthetic / handheld_real (losses.cpp:33-46)."""
    w = LossWeights(0.7, 0.1, 0.25, 0.25, 0.1, 0.15, 0.2, 1.0, 1.0, 0.1, 1)
    if handheld_real:
        w.w_color, w.w_ssim, w.w_geo, w.w_align, w.w_iso, w.w_var = 1.0, 0.1, 0.8, 0.5, 0.1, 0.5
        w.t_color, w.t_geo = 1.0, 0.6
    return w


def defaults_tracker() -> TrackerCfg:
    """TrackerConfig defaults (track/tracker.hpp:11-22)."""
    return TrackerCfg(0.0015, 0.00215, 15, 4, 10, 30, 2, 1, 2.0)


def defaults_slam(K: Intrinsics) -> SlamCfg:
    """RunConfig defaults (io/config.hpp:16-35) with intrinsics K: tracker, mapper, 60 / 120 mapping iterations."""
    return SlamCfg(K, defaults_tracker(), defaults_mapper(), 60, 120, 0)


def defaults_mapper() -> MapperCfg:
    """MapperConfig defaults (map/mapper.hpp:21-41)."""
    return MapperCfg(1, 4.0, 1.6e-4, 2.5e-3, 5e-2, 5e-3, 1e-3, 100, 2e-4, 1.6, 0.01, 0.005, 0.025,
                     0.005, 0, defaults_raster(), defaults_weights(), 2, 2, 0.5, 0.5)
