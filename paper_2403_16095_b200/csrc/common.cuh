// common.cuh — device state, workspace layout and launch helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gsf_shared.cuh"

namespace gsfk {

constexpr int kTile = 16;
// Binning: one fill counter per 32-byte L2 sector (the L2 serialises atomics per sector:
// measured 35 us for the 563k pair increments of configs[1] packed vs 12 us one per sector),
// primitives with more than kBigPairs tiles go to the one-CTA-per-primitive scatter, and the
// slots of Workspace::bin_counters.
#ifndef GSF_BIN_STRIDE
#define GSF_BIN_STRIDE 8
#endif
constexpr int kBinStride = GSF_BIN_STRIDE;
static_assert(kBinStride >= 4, "the tile-list scan word shares the fill counter's sector");
constexpr int kPjFloats = 56;   // per-primitive pose matrix: 9 columns x 6 rows + 2 pad (k_posejac)
constexpr int kBigPairs = 128;
enum BinCounter { kCntVisible = 0, kCntBlendTicket = 1, kCntBwdTicket = 2, kCntBig = 3, kCntPairAlloc = 4, kCntSortTicket = 5, kCntFixup = 6, kCntTileAlloc = 7, kCntNum = 8 };             // tile edge (RasterConfig::tile_size, config.hpp:10)
constexpr int kTilePixels = kTile * kTile;
constexpr int kFieldsBase = 11;       // mean 3, log_scale 3, quat 4, opacity 1; then 3*K SH

// Pixel of thread `tid` inside a 16x16 tile: each warp owns an 8x4 block (warp w -> block
// column w & 1, block row w >> 1), which keeps a warp's pixels compact so that footprint
// edges split fewer warps than 16x2 rows would.
__host__ __device__ __forceinline__ int tile_lx(int tid) { return ((tid >> 5) & 1) * 8 + (tid & 7); }
__host__ __device__ __forceinline__ int tile_ly(int tid) { return (tid >> 6) * 4 + ((tid >> 3) & 3); }

// Conservative footprint test of one staged tile-list entry against the eight 8x4 warp blocks
// of its tile.  Bit w is set unless every pixel centre of warp block w is certainly rejected by
// the per-pair test (rho > cutoff + band, or sigma*exp(-rho/2) below the alpha skip); the
// margins dwarf fp32 rounding, so the mask only removes work that would produce nothing and
// never changes a result.  min over a rectangle of a x^2 + 2 b x y + c y^2 is attained at the
// origin (if inside) or on an edge at the clamped stationary point.
__device__ __forceinline__ float quad_min_rect(float a, float b, float c, float x0, float x1, float y0, float y1) {
  if (x0 <= 0.0f && x1 >= 0.0f && y0 <= 0.0f && y1 >= 0.0f) return 0.0f;
  float m = 3.0e38f;
  const float ia = 1.0f / a, ic = 1.0f / c;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float X = e ? x1 : x0;
    const float y = fminf(fmaxf(-b * X * ic, y0), y1);
    m = fminf(m, a * X * X + 2.0f * b * X * y + c * y * y);
    const float Y = e ? y1 : y0;
    const float x = fminf(fmaxf(-b * Y * ia, x0), x1);
    m = fminf(m, a * x * x + 2.0f * b * x * Y + c * Y * Y);
  }
  return m;
}

__device__ __forceinline__ uint32_t warp_block_mask(const BlendG& g, float tile_x0, float tile_y0, const BlendConsts& kc) {
  const float a = g.c00, b = 0.5f * g.c01x2, c = g.c11;
  if (!(a > 0.0f) || !(c > 0.0f) || !(a * c > b * b)) return 0xffu;
  if (g.sigma < kc.skip_lo) return 0u;   // sigma * g <= sigma < skip: nothing can contribute
  float thr = kc.rho_hi;
  const float ra = 2.0f * __logf(g.sigma / kc.skip_lo);   // rho beyond which alpha < skip
  thr = fminf(thr, ra);
  thr = thr * 1.002f + 2e-3f;
  uint32_t mask = 0u;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const float bx0 = tile_x0 + static_cast<float>(8 * (w & 1)) + 0.5f - g.mx;
    const float by0 = tile_y0 + static_cast<float>(4 * (w >> 1)) + 0.5f - g.my;
    if (quad_min_rect(a, b, c, bx0, bx0 + 7.0f, by0, by0 + 3.0f) <= thr) mask |= 1u << w;
  }
  return mask;
}

// 8x8 variant for the two-pixels-per-lane tracking kernels: bit w (w < 4) says whether the
// primitive can reach the 8x8 block (8 (w & 1), 8 (w >> 1)) of the tile.
__device__ __forceinline__ uint32_t warp_block_mask8(const BlendG& g, float tile_x0, float tile_y0, const BlendConsts& kc) {
  const float a = g.c00, b = 0.5f * g.c01x2, c = g.c11;
  if (!(a > 0.0f) || !(c > 0.0f) || !(a * c > b * b)) return 0xfu;
  if (g.sigma < kc.skip_lo) return 0u;
  float thr = kc.rho_hi;
  const float ra = 2.0f * __logf(g.sigma / kc.skip_lo);
  thr = fminf(thr, ra);
  thr = thr * 1.002f + 2e-3f;
  uint32_t mask = 0u;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const float bx0 = tile_x0 + static_cast<float>(8 * (w & 1)) + 0.5f - g.mx;
    const float by0 = tile_y0 + static_cast<float>(8 * (w >> 1)) + 0.5f - g.my;
    if (quad_min_rect(a, b, c, bx0, bx0 + 7.0f, by0, by0 + 7.0f) <= thr) mask |= 1u << w;
  }
  return mask;
}

// One 8x8 block at pixel origin (bx0, by0): warp_block_mask8's test for a single block.
__device__ __forceinline__ bool block_hit8(const BlendG& g, float bx0, float by0, const BlendConsts& kc) {
  const float a = g.c00, b = 0.5f * g.c01x2, c = g.c11;
  if (!(a > 0.0f) || !(c > 0.0f) || !(a * c > b * b)) return true;
  if (g.sigma < kc.skip_lo) return false;
  float thr = kc.rho_hi;
  const float ra = 2.0f * __logf(g.sigma / kc.skip_lo);
  thr = fminf(thr, ra);
  thr = thr * 1.002f + 2e-3f;
  const float x0 = bx0 + 0.5f - g.mx, y0 = by0 + 0.5f - g.my;
  return quad_min_rect(a, b, c, x0, x0 + 7.0f, y0, y0 + 7.0f) <= thr;
}

// Shared-memory loads from an explicit 32-bit address.  opaque_smem_base() returns the address of a
// __shared__ object through a warp shuffle, which ptxas cannot re-derive: the hot loops then keep
// one base register instead of re-forming (SR_CgaCtaId << 24) + offset with an S2R per access.
__device__ __forceinline__ uint32_t opaque_smem_base(const void* p) {
  return __shfl_sync(0xffffffffu, static_cast<uint32_t>(__cvta_generic_to_shared(p)), 0);
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ BlendG lds_blend(uint32_t a) {
  const float4 a0 = lds_f4(a), a1 = lds_f4(a + 16), a2 = lds_f4(a + 32);
  BlendG g;
  g.mx = a0.x; g.my = a0.y; g.sigma = a0.z; g.rho_hi = a0.w;
  g.c00 = a1.x; g.c01x2 = a1.y; g.c11 = a1.z; g.rho_fast = a1.w;
  g.r = a2.x; g.g = a2.y; g.b = a2.z; g.depth = a2.w;
  return g;
}

__device__ __forceinline__ void sts_s32(uint32_t a, int32_t v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// 16-byte asynchronous global -> shared copy to an explicit shared address (L2 only: read once)
__device__ __forceinline__ void cp_async16_to(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Ampere-style asynchronous global -> shared copies (cp.async, 16 bytes, L1-allocating).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
// 4-byte cp.async with zero fill (src_bytes 0: the destination word is zeroed, nothing is read)
__device__ __forceinline__ void cp_async4_zfill(void* smem_dst, const void* gmem_src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem_src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Guard-band entries (rare) of the two-pixel kernels: eval_pair_full out of line.  Takes the
// record's geometry by value (the caller's registers; nothing is materialised on the hot path) and
// kc through a pointer.  alpha < 0: no contribution.
struct GuardOut {
  float alpha, gval;
  int clamped;
};
static __device__ __noinline__ GuardOut guard_full(float px, float py, float mx, float my, float c00, float c01x2,
                                                   float c11, float sigma, const GuardG* gp, const BlendConsts* kc) {
  BlendG g;
  g.mx = mx; g.my = my; g.c00 = c00; g.c01x2 = c01x2; g.c11 = c11; g.sigma = sigma;
  const PairEval e = eval_pair_full(px, py, g, gp, *kc);
  return GuardOut{e.code ? e.alpha : -1.0f, e.gval, e.clamped};
}
__device__ __forceinline__ GuardOut guard_decide(float px, float py, const BlendG& g, const GuardG* gp, const BlendConsts* kc) {
  return guard_full(px, py, g.mx, g.my, g.c00, g.c01x2, g.c11, g.sigma, gp, kc);
}

// pair_rho for two pixels in one column (same dx, dy = (dy_a, dy_b)) on packed FP32x2: each lane
// performs pair_rho's operations in pair_rho's order, so rho.x / rho.y equal the scalar values.
__device__ __forceinline__ float2 pair_rho2(float dx, float2 dy, const BlendG& g) {
  const float a1 = __fmul_rn(g.c00, dx), b1 = __fmul_rn(g.c01x2, dx);
  float2 t = __fmul2_rn(make_float2(g.c11, g.c11), dy);
  t = __fmul2_rn(t, dy);
  t = __ffma2_rn(make_float2(b1, b1), dy, t);
  return __ffma2_rn(make_float2(a1, a1), make_float2(dx, dx), t);
}

// exp_neg_half_inrange (gsf_shared.cuh) of two values on packed FP32x2, bit-identical per lane.
__device__ __forceinline__ float2 exp_neg_half_inrange2(float2 rho) {
  const float2 y = __fmul2_rn(rho, make_float2(-0.72134752044448170368f, -0.72134752044448170368f));
  const float nx = rintf(y.x), ny = rintf(y.y);
  const float2 f = __fadd2_rn(y, make_float2(-nx, -ny));   // y - n, exactly fsub's result
  // 2^n without F2I (XU pipe): n + 1.5 * 2^23 is exact for the integer n, and the low 9 bits of its
  // pattern are n's, so (bits(t) << 23) + (127 << 23) is 2^n's pattern.  (y itself must not meet
  // the magic constant: ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2.)
  const float2 t = __fadd2_rn(make_float2(nx, ny), make_float2(12582912.0f, 12582912.0f));
  float2 p = make_float2(1.5403530393381606e-4f, 1.5403530393381606e-4f);
  p = __ffma2_rn(p, f, make_float2(1.3333558146428443e-3f, 1.3333558146428443e-3f));
  p = __ffma2_rn(p, f, make_float2(9.6181291076284772e-3f, 9.6181291076284772e-3f));
  p = __ffma2_rn(p, f, make_float2(5.5504108664821580e-2f, 5.5504108664821580e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022650695910071e-1f, 2.4022650695910071e-1f));
  p = __ffma2_rn(p, f, make_float2(6.9314718055994531e-1f, 6.9314718055994531e-1f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return __fmul2_rn(p, make_float2(__uint_as_float((__float_as_uint(t.x) << 23) + 0x3f800000u),
                                   __uint_as_float((__float_as_uint(t.y) << 23) + 0x3f800000u)));
}

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
  uint32_t overflow;       // pair / tile-bucket capacity exceeded (host grows and re-runs)
  uint32_t max_tile;       // longest tile list over the renders since the last reset (atomicMax)
  uint32_t M_max;          // largest pair total over the renders since the last reset (sizes the growth)
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
  // tracking trust region (k_candidates / track_update): the candidate list holds every primitive
  // that can be visible while the camera stays within (theta, dist) of the frame's first camera
  double cand_W0[9], cand_t0[3];
  double cand_cos_min, cand_dist_max;
  uint32_t ncand;
  int32_t cand_ok;         // 1 while the current camera is inside the trust region
};

struct LossParams {       // what the fused epilogues need (constant per loop)
  int32_t mode;           // 0 none, 1 tracking, 2 mapping
  float opacity_floor;
  int32_t normalize_by_valid;
  double w_color, w_ssim, w_geo, w_align, w_iso, w_var, t_color, t_geo, iso_epsilon;
  int32_t uncertainty_full_gradient;
};

// Warp-wide exclusive prefix sum of one int per lane.
__device__ __forceinline__ int warp_excl_scan(int v) {
  const int lane = threadIdx.x & 31;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// Largest lane j with excl_j <= k (excl non-decreasing over the lanes, excl_0 == 0).
__device__ __forceinline__ int warp_owner(int excl, int k) {
  int lo = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int e = __shfl_sync(0xffffffffu, excl, lo + step);
    if (e <= k) lo += step;
  }
  return lo;
}

// Tile-list sort key: (fp32 bits of the depth) << 32 | id (binning.cu).
__device__ __forceinline__ unsigned long long pair_key(double depth, uint32_t id) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(__float_as_int(static_cast<float>(depth)))) << 32) | id;
}

// One (tile, primitive) pair into its tile's bucket (binning.cu).
__device__ __forceinline__ void bucket_put(uint32_t* fill, unsigned long long* bucket, uint32_t bucket_cap, int64_t t,
                                           unsigned long long key) {
  const uint32_t slot = atomicAdd(&fill[t * kBinStride], 1u);
  if (slot < bucket_cap) bucket[t * bucket_cap + slot] = key;
}

// Programmatic dependent launch inside the tracking loop: each kernel lets its successor launch as
// soon as all of its own CTAs are running (launch_dependents) and waits for its predecessor's
// completion and memory (wait) before touching anything the predecessor writes.  Both are no-ops
// without a programmatic edge.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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

#ifndef GSF_NO_PDL
// Launch with a programmatic (PDL) edge to the previous kernel on the stream.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GSF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
#else
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  kern<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
  GSF_CUDA_CHECK(cudaGetLastError());
}
#endif


inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace gsfk
