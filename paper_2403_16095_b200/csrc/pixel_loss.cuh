// pixel_loss.cuh — per-pixel loss contributions and adjoint seeds shared by the fused blend
// epilogue, the backward kernel and the stand-alone loss API kernels.
//   tracking: evaluate_tracking_loss (losses.cpp:284-339)
//   mapping:  evaluate_mapping_loss  (losses.cpp:156-282)
#pragma once

#include "common.cuh"

namespace gsfk {

__device__ __forceinline__ bool px_depth_valid(float d, double near_plane, double far_plane) {
  const double v = d;
  return isfinite(v) && v > near_plane && v < far_plane;
}

__device__ __forceinline__ float px_sgn(float v) { return v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : 0.0f); }

// Residual sums and mask counts of one pixel into v[LS_NUM].
// LMODE 1 = tracking, 2 = mapping.  depth may be NULL (no sensor depth -> no geo terms);
// has_unc says whether the render carried an uncertainty map (mapping var term).
template <int LMODE>
__device__ __forceinline__ void loss_pixel(double* v, float cr, float cg, float cb, float ad, float md, bool mvalid,
                                           float op, float unc, const float* I, const float* depth, int64_t pi,
                                           bool has_unc, double near_plane, double far_plane, float floor) {
  const bool opm = op >= floor;
  const float D = depth ? depth[pi] : 0.0f;
  const bool geo = opm && depth && px_depth_valid(D, near_plane, far_plane);
  const double cabs = static_cast<double>(fabsf(cr - I[0])) + static_cast<double>(fabsf(cg - I[1])) +
                      static_cast<double>(fabsf(cb - I[2]));
  if (LMODE == 1) {
    if (opm) { v[LS_COLOR_SUM] = cabs; v[LS_COLOR_CNT] = 1.0; }
  } else {
    v[LS_COLOR_SUM] = cabs;
    v[LS_COLOR_CNT] = opm ? 1.0 : 0.0;
    if (opm && mvalid) { v[LS_ALIGN_SUM] = fabsf(ad - md); v[LS_ALIGN_CNT] = 1.0; }
    if (has_unc && geo) { v[LS_VAR_SUM] = fabsf(unc); v[LS_VAR_CNT] = 1.0; }
  }
  if (geo) { v[LS_GEO_SUM] = fabsf(ad - D); v[LS_GEO_CNT] = 1.0; }
}

// Tracking seeds (losses.cpp:330-337) are a global scale times a per-pixel sign: the fused tracking
// forward stores the signs (2 bits each: colour 0..2, alpha depth; 1 = +, 2 = -, masks folded in)
// so the pose backward reads one byte instead of the maps, the target and the sensor depth.
__device__ __forceinline__ uint32_t sgn_code(float v) { return v > 0.0f ? 1u : (v < 0.0f ? 2u : 0u); }
__device__ __forceinline__ float code_sgn(uint32_t c) { return c == 1u ? 1.0f : (c == 2u ? -1.0f : 0.0f); }
__device__ __forceinline__ uint8_t pixel_seed_code(float cr, float cg, float cb, float ad, float op, const float* I,
                                                   const float* depth, int64_t pi, double near_plane, double far_plane,
                                                   float floor) {
  const bool opm = op >= floor;
  const float D = depth ? depth[pi] : 0.0f;
  const bool geo = opm && depth && px_depth_valid(D, near_plane, far_plane);
  uint32_t code = 0u;
  if (opm) code = sgn_code(cr - I[0]) | (sgn_code(cg - I[1]) << 2) | (sgn_code(cb - I[2]) << 4);
  if (geo) code |= sgn_code(ad - D) << 6;
  return static_cast<uint8_t>(code);
}

struct PixSeeds {
  float gc0, gc1, gc2, gad, gmd, gu;
};

// Adjoint seeds of one pixel from the finalised normalisers in DevState.
// SEED 1 = tracking (losses.cpp:330-337), 2 = mapping (losses.cpp:241-270).
// dssim (mapping) is d(mean ssim)/d colour, 3 per pixel, or NULL.
template <int SEED>
__device__ __forceinline__ PixSeeds seeds_pixel(int64_t pi, const float* color, float ad, float md, bool mvalid, float op,
                                                const float* target, const float* depth, const float* dssim,
                                                const DevState* ds, const LossParams& lp, double near_plane,
                                                double far_plane) {
  PixSeeds s;
  s.gc0 = s.gc1 = s.gc2 = s.gad = s.gmd = s.gu = 0.0f;
  const bool opm = op >= lp.opacity_floor;
  const float D = depth ? depth[pi] : 0.0f;
  const bool geo = opm && depth && px_depth_valid(D, near_plane, far_plane);
  const float* I = target + 3 * pi;
  const float* c = color + 3 * pi;
  if (SEED == 1) {
    if (opm) {
      const float sc = static_cast<float>(ds->seed_color);
      s.gc0 = sc * px_sgn(c[0] - I[0]);
      s.gc1 = sc * px_sgn(c[1] - I[1]);
      s.gc2 = sc * px_sgn(c[2] - I[2]);
    }
    if (geo) s.gad = static_cast<float>(ds->seed_geo) * px_sgn(ad - D);
  } else {
    const float sc = static_cast<float>(ds->seed_color);
    s.gc0 = sc * px_sgn(c[0] - I[0]);
    s.gc1 = sc * px_sgn(c[1] - I[1]);
    s.gc2 = sc * px_sgn(c[2] - I[2]);
    if (dssim && lp.w_ssim > 0.0) {
      const float ws = static_cast<float>(lp.w_ssim);
      s.gc0 -= ws * dssim[3 * pi];
      s.gc1 -= ws * dssim[3 * pi + 1];
      s.gc2 -= ws * dssim[3 * pi + 2];
    }
    if (geo) s.gad += static_cast<float>(ds->seed_geo) * px_sgn(ad - D);
    if (opm && mvalid) {
      const float sa = static_cast<float>(ds->seed_align) * px_sgn(ad - md);
      s.gad += sa;
      s.gmd = -sa;
    }
    if (geo && ds->has_obs) s.gu = static_cast<float>(ds->seed_var);
  }
  return s;
}

}  // namespace gsfk
