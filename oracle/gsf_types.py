"""TEST INFRASTRUCTURE ONLY — ctypes views of the plain-C types of include/gsf_cuda.h for the CPU
checker (oracle/).  They restate the header's struct layouts so that oracle/ never imports the
product package; the product's own ctypes views (paper_2403_16095_b200/abi.py) have the same
layouts, so either can be passed by reference to the oracle's entry points."""
import ctypes as C

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


class MapHost(C.Structure):
    _fields_ = [("count", C.c_int64), ("sh_coeffs", C.c_int32), ("mean", dp), ("log_scale", dp),
                ("quat", dp), ("opacity_logit", dp), ("sh", dp), ("uncertainty", dp),
                ("observed", u8p)]


class TrackResult(C.Structure):
    _fields_ = [("pose", Pose), ("final_loss", C.c_double), ("degraded", C.c_int32),
                ("iterations_run", C.c_int32), ("initial_loss", C.c_double)]


class LossTerms(C.Structure):
    _fields_ = [("color", C.c_double), ("ssim", C.c_double), ("geo", C.c_double),
                ("align", C.c_double), ("iso", C.c_double), ("var", C.c_double),
                ("total", C.c_double), ("valid_color", C.c_int32), ("valid_geo", C.c_int32),
                ("any_empty_mask", C.c_int32)]
