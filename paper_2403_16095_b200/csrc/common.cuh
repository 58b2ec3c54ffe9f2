// common.cuh — device state, workspace layout and launch helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gsf_shared.cuh"

namespace gsfk {

constexpr int kTile = 16;             // tile edge (RasterConfig::tile_size, config.hpp:10)
constexpr int kTilePixels = kTile * kTile;
constexpr int kFieldsBase = 11;       // mean 3, log_scale 3, quat 4, opacity 1; then 3*K SH

// Pixel of thread `tid` inside a 16x16 tile: each warp owns an 8x4 block (warp w -> block
// column w & 1, block row w >> 1), which keeps a warp's pixels compact so that footprint
// edges split fewer warps than 16x2 rows would.
__host__ __device__ __forceinline__ int tile_lx(int tid) { return ((tid >> 5) & 1) * 8 + (tid & 7); }
__host__ __device__ __forceinline__ int tile_ly(int tid) { return (tid >> 6) * 4 + ((tid >> 3) & 3); }

// Loss partial slots written per tile by the fused blend epilogue (fixed order reduction).
enum LossSlot {
  LS_COLOR_SUM = 0,   // sum |c - I| over the colour mask (tracking: opacity mask, mapping: all)
  LS_GEO_SUM,         // sum |ad - D| over geo mask
  LS_ALIGN_SUM,       // sum |ad - md| over align mask
  LS_VAR_SUM,         // sum |U| over var mask
  LS_COLOR_CNT,       // counts (stored as double, exact below 2^53)
  LS_GEO_CNT,
  LS_ALIGN_CNT,
  LS_VAR_CNT,
  LS_NUM
};

// Scalars living on the device so that whole track/map loops run without host round trips.
struct DevState {
  uint32_t V;              // visible primitives of the current render
  uint32_t M;              // (tile, primitive) pairs of the current render
  uint32_t overflow;       // pair capacity exceeded (host grows and re-runs)
  int32_t bad_index;       // smallest non-finite primitive index, INT32_MAX if none
  int32_t halt;            // 0 run, 1 nothing to track at it 0, 2 diverged, 3 non-finite map
  int32_t halt_iter;
  int32_t iteration;       // loop iteration counter
  int32_t has_obs;         // current render has an observed depth map
  // loss (finalised by k_loss_finalize)
  double loss[LS_NUM];
  double term_color, term_geo, term_align, term_var, term_ssim, term_iso, loss_total;
  double seed_color, seed_geo, seed_align, seed_var;   // per-pixel seed magnitudes w/m
  int32_t any_empty;
  int32_t pad0;
  double ssim_sum;         // sum of per-pixel ssim (finalised into term_ssim)
  double iso_sum; double iso_count;
  // pose optimisation (tracking): current pose, Adam state, gradient
  double pose_rot[3], pose_trans[3];
  double adam_m[6], adam_v[6];
  double adam_t;
  double d_pose[6];
  double initial_loss, final_loss;
  int32_t iterations_run, degraded;
  double lr_rot, lr_trans, degraded_ratio;
  Cam cam;                 // camera of the current render
};

struct LossParams {       // what the fused epilogues need (constant per loop)
  int32_t mode;           // 0 none, 1 tracking, 2 mapping
  float opacity_floor;
  int32_t normalize_by_valid;
  double w_color, w_ssim, w_geo, w_align, w_iso, w_var, t_color, t_geo, iso_epsilon;
  int32_t uncertainty_full_gradient;
};

#define GSF_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) throw gsfk::CudaError(_e, #expr, __FILE__, __LINE__);    \
  } while (0)

struct CudaError {
  cudaError_t code;
  const char* expr;
  const char* file;
  int line;
  CudaError(cudaError_t c, const char* e, const char* f, int l) : code(c), expr(e), file(f), line(l) {}
};

inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace gsfk
