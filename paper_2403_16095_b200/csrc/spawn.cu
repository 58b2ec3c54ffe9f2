// spawn.cu — map growth on the device: initialize_map and spawn_gaussians (map/mapper.cpp:12-26,
// 125-170).  One candidate per stride-sampled pixel (row-major order, the reference's loop order):
//
//   k_bp_count   per-CTA number of accepted candidates (valid sensor depth, and for spawn the
//                current render's accumulated opacity below the threshold)
//   k_bp_scan    one CTA: exclusive scan of the CTA counts, total
//   k_bp_write   the same predicate + a CTA scan -> the candidate's slot after the existing map;
//                writes the backprojected primitive (fp64 geometry, fp32 SoA storage)
//
// The map SoA [field][P] is re-laid out to the new count by the host between scan and write.
#include "kernels.h"

namespace gsfk {

namespace {

__device__ __forceinline__ bool bp_accept(const BackprojectArgs& a, int64_t cell, int& x, int& y, int64_t& pi) {
  const int cx = static_cast<int>(cell % a.cells_x), cy = static_cast<int>(cell / a.cells_x);
  x = cx * a.stride;
  y = cy * a.stride;
  pi = static_cast<int64_t>(y) * a.W + x;
  const double d = a.depth[pi];   // sensor_valid_mask (losses.cpp:141-148)
  if (!(isfinite(d) && d > a.near_plane && d < a.far_plane)) return false;
  if (a.opacity && !(static_cast<double>(a.opacity[pi]) < a.threshold)) return false;   // mapper.cpp:160
  return true;
}

__global__ void __launch_bounds__(256) k_bp_count(BackprojectArgs a, uint32_t* __restrict__ blk_cnt) {
  __shared__ uint32_t s_w[8];
  const int64_t cell = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int x, y;
  int64_t pi;
  const bool ok = cell < a.cells && bp_accept(a, cell, x, y, pi);
  const uint32_t bits = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = static_cast<uint32_t>(__popc(bits));
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_w[w];
    blk_cnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_bp_scan(const uint32_t* __restrict__ cnt, int n, uint32_t* __restrict__ off,
                                                  uint32_t* total) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int t = base + tid;
    const uint32_t v = t < n ? cnt[t] : 0u;
    uint32_t xs = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yv = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= o) xs += yv;
    }
    if (lane == 31) s_warp[warp] = xs;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yv = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += yv;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const uint32_t incl = s_carry + (warp ? s_warp[warp - 1] : 0u) + xs;
    if (t < n) off[t] = incl - v;
    __syncthreads();
    if (tid == 1023) s_carry = incl;
    __syncthreads();
  }
  if (tid == 0) *total = s_carry;
}

__global__ void __launch_bounds__(256) k_bp_write(BackprojectArgs a, const uint32_t* __restrict__ blk_off, int64_t P_old,
                                                  int64_t P_new, float* __restrict__ params, double* __restrict__ nu,
                                                  uint8_t* __restrict__ observed) {
  __shared__ uint32_t s_w[8];
  const int64_t cell = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = 0, y = 0;
  int64_t pi = 0;
  const bool ok = cell < a.cells && bp_accept(a, cell, x, y, pi);
  const uint32_t bits = __ballot_sync(0xffffffffu, ok);
  if (lane == 0) s_w[warp] = static_cast<uint32_t>(__popc(bits));
  __syncthreads();
  if (!ok) return;
  uint32_t local = __popc(bits & ((1u << lane) - 1u));
  for (int w = 0; w < warp; ++w) local += s_w[w];
  const int64_t i = P_old + blk_off[blockIdx.x] + local;
  // backprojected_primitive (mapper.cpp:12-26): p_cam = K^-1 (x + .5, y + .5) d; mean = pose^-1 p_cam
  const double d = a.depth[pi];
  const double pc[3] = {(static_cast<double>(x) + 0.5 - a.cx) / a.fx * d, (static_cast<double>(y) + 0.5 - a.cy) / a.fy * d, d};
  for (int r = 0; r < 3; ++r) {
    const double m = a.Rinv[3 * r] * pc[0] + a.Rinv[3 * r + 1] * pc[1] + a.Rinv[3 * r + 2] * pc[2] + a.tinv[r];
    params[r * P_new + i] = static_cast<float>(m);
  }
  const float ls = static_cast<float>(log((d / a.fx) * a.stride * 0.5));
  for (int r = 0; r < 3; ++r) params[(3 + r) * P_new + i] = ls;
  params[6 * P_new + i] = 1.0f;
  params[7 * P_new + i] = params[8 * P_new + i] = params[9 * P_new + i] = 0.0f;
  params[10 * P_new + i] = static_cast<float>(a.logit0);
  const float* rgb = a.rgb + 3 * pi;
  for (int c = 0; c < 3; ++c)
    params[(11 + c) * P_new + i] = static_cast<float>((static_cast<double>(rgb[c]) - 0.5) / 0.28209479177387814);
  for (int k = 3; k < 3 * a.K; ++k) params[(11 + k) * P_new + i] = 0.0f;
  nu[i] = 0.0;
  observed[i] = 1;
}

}  // namespace

int64_t run_backproject_count(const BackprojectArgs& a, uint32_t* blk_cnt, uint32_t* blk_off, uint32_t* total,
                              cudaStream_t st, int64_t* L) {
  const int blocks = std::max(1, div_up(a.cells, 256));
  k_bp_count<<<blocks, 256, 0, st>>>(a, blk_cnt);
  k_bp_scan<<<1, 1024, 0, st>>>(blk_cnt, blocks, blk_off, total);
  *L += 2;
  return blocks;
}

void run_backproject_write(const BackprojectArgs& a, const uint32_t* blk_off, int64_t P_old, int64_t P_new, float* params,
                           double* nu, uint8_t* observed, cudaStream_t st, int64_t* L) {
  const int blocks = std::max(1, div_up(a.cells, 256));
  k_bp_write<<<blocks, 256, 0, st>>>(a, blk_off, P_old, P_new, params, nu, observed);
  ++*L;
}

}  // namespace gsfk
