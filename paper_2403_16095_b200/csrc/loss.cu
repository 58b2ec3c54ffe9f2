// loss.cu — loss finalisation, SSIM forward/adjoint and the anisotropy (iso) term on sm_100a.
//
//   k_loss_finalize  the scalar tails of evaluate_tracking_loss (losses.cpp:284-339) and
//                    evaluate_mapping_loss (:156-282): a fixed-order sum of the per-tile partials
//                    written by the blend epilogue, the normalisers w/m of every seed map, and
//                    the device-side loop checks of track_frame (tracker.cpp:45-60) / map_step
//                    (mapper.cpp:247-254) so no host round trip is needed per iteration.
//   SSIM             ssim.cpp:27-187: separable 11-tap blur with border renormalisation, fp64
//                    per-pixel terms, and the adjoint blur for d(ssim)/dx.
//   k_iso            iso term and its direct log-scale gradient (losses.cpp:195-216, 272-280).
#include "kernels.h"
#include "finalize.cuh"

namespace gsfk {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Sum one value per thread over a 256-thread block in a fixed tree; result valid in thread 0.
__device__ __forceinline__ double block_sum_d(double v, double* s_red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  v = warp_sum_d(v);
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (tid == 0)
    for (int w = 0; w < 8; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(1024) k_loss_finalize(const double* __restrict__ loss_part, int tiles, int64_t npix,
                                                        LossParams lp, int iteration, const double* __restrict__ ssim_part,
                                                        int ssim_blocks, const double* __restrict__ iso_part,
                                                        int iso_blocks, DevState* ds) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  // one pass over the three partial arrays (thread t owns rows t, t + 1024, ... of each: a fixed
  // order), one warp reduction and one barrier for all LS_NUM + 2 sums
  constexpr int NV = LS_NUM + 2;
  __shared__ double s_red[32][NV];
  __shared__ double s_tot[NV];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int r = tid; r < tiles; r += 1024) {
    const double* row = loss_part + static_cast<int64_t>(r) * LS_NUM;
#pragma unroll
    for (int q = 0; q < LS_NUM; ++q) acc[q] += __ldcg(row + q);
  }
  for (int r = tid; r < ssim_blocks; r += 1024) acc[LS_NUM] += __ldcg(ssim_part + r);
  for (int r = tid; r < iso_blocks; r += 1024) acc[LS_NUM + 1] += __ldcg(iso_part + r);
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double t = warp_sum_f64(acc[q]);
    if (lane == 0) s_red[warp][q] = t;
  }
  __syncthreads();
  if (tid < NV) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += s_red[w][tid];
    s_tot[tid] = t;
  }
  __syncthreads();
  if (tid == 0) loss_scalars(ds, lp, s_tot, s_tot[LS_NUM], s_tot[LS_NUM + 1], npix, iteration);
}

// ---- SSIM ------------------------------------------------------------------------------------
constexpr int kR = 5;
__constant__ float c_win[11];

__device__ __forceinline__ float axis_norm(int p, int n) {
  float z = 0.0f;
#pragma unroll
  for (int o = -kR; o <= kR; ++o)
    if (p + o >= 0 && p + o < n) z += c_win[o + kR];
  return z;
}

// SSIM (ssim.cpp:27-187), tiled: a CTA owns a 32x16 block of pixels and stages its inputs with a
// 5-pixel halo in shared memory; both separable blur passes run there (out-of-image taps read 0,
// which adds w*0 exactly like the reference's skipped taps), the per-pixel SSIM and its three
// adjoint seed maps in fp64; the adjoint blurs vertical first, then horizontal, each tap divided by
// its own border normaliser (ssim.cpp:60-80).
constexpr int kSX = 32, kSY = 16, kSW = kSX + 2 * kR, kSHh = kSY + 2 * kR;

// Register-blocked and channel-at-a-time (85 us per 1200x680 view, 94 us for the all-planes version).  The forward
// stages the six input planes of the 32x16 block (+5 px halo) once; then per channel the horizontal
// pass gives each thread 4 consecutive outputs of one row (14 input columns read once, the 5 product
// maps a, b, a^2, b^2, ab formed once per input, 11 taps per output from the constant window) and
// the vertical pass 2 consecutive rows of one column (12 staged rows read once), followed by the
// per-pixel fp64 SSIM of those two pixels.  The adjoint runs the same blocking per channel over its
// three seed planes (vertical: 4 rows x 1 column, horizontal: 2 columns x 1 row).
constexpr int kHG = 4;                   // horizontal outputs per thread
constexpr int kHItems = kSHh * (kSX / kHG);   // 26 rows x 8 groups = 208
constexpr size_t ssim_fwd2_smem() { return sizeof(float) * (6 * kSHh * kSW + 5 * kSHh * kSX); }
constexpr size_t ssim_bwd2_smem() { return sizeof(float) * (2 * 3 * kSHh * kSW + 3 * kSY * kSW); }

__global__ void __launch_bounds__(256) k_ssim_fwd2(const float* __restrict__ x, const float* __restrict__ y, int W, int H,
                                                   double weight, float* __restrict__ u, double* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_buf[];
  float (*s_in)[kSHh][kSW] = reinterpret_cast<float (*)[kSHh][kSW]>(s_buf);                  // x0..2, y0..2
  float (*s_h)[kSHh][kSX] = reinterpret_cast<float (*)[kSHh][kSX]>(s_buf + 6 * kSHh * kSW);   // 5 planes, one channel
  __shared__ double s_red[8];
  __shared__ float s_izx[kSX];
  const int64_t npix = static_cast<int64_t>(W) * H;
  const int bx = blockIdx.x * kSX, by = blockIdx.y * kSY;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < kSHh * kSW; idx += 256) {
    const int r = idx / kSW, c = idx - r * kSW;
    const int gx = bx - kR + c, gy = by - kR + r;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const int64_t j = static_cast<int64_t>(gy) * W + gx;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      s_in[ch][r][c] = in ? x[3 * j + ch] : 0.0f;
      s_in[3 + ch][r][c] = in ? y[3 * j + ch] : 0.0f;
    }
  }
  if (tid < kSX) s_izx[tid] = 1.0f / axis_norm(min(bx + tid, W - 1), W);
  // vertical-pass pixels of this thread: column vc, rows 2 vr and 2 vr + 1
  const int vc = tid & (kSX - 1), vr = tid >> 5;
  const int gx = bx + vc;
  double izy[2];
  bool vin[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int gy = by + 2 * vr + j;
    vin[j] = gx < W && gy < H;
    izy[j] = vin[j] ? 1.0 / static_cast<double>(axis_norm(gy, H)) : 0.0;
  }
  double ssum = 0.0;
  __syncthreads();
  for (int ch = 0; ch < 3; ++ch) {
    if (tid < kHItems) {   // horizontal pass: row hr, outputs hx .. hx + 3
      const int hr = tid / (kSX / kHG), hx = (tid - hr * (kSX / kHG)) * kHG;
      // outputs in pairs (hx, hx + 1), (hx + 2, hx + 3) on packed FFMA2: each lane rounds like the
      // scalar FMA, and a tap outside the window adds 0 * v (exact), so the sums equal the scalar ones
      float2 acc[5][kHG / 2];
#pragma unroll
      for (int q = 0; q < 5; ++q)
#pragma unroll
        for (int k = 0; k < kHG / 2; ++k) acc[q][k] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int p = 0; p < kHG + 2 * kR; ++p) {
        const float a = s_in[ch][hr][hx + p], b = s_in[3 + ch][hr][hx + p];
        const float v[5] = {a, b, a * a, b * b, a * b};
#pragma unroll
        for (int k = 0; k < kHG / 2; ++k) {
          const int o0 = p - 2 * k, o1 = o0 - 1;
          const bool in0 = o0 >= 0 && o0 <= 2 * kR, in1 = o1 >= 0 && o1 <= 2 * kR;
          if (in0 || in1) {
            const float2 w = make_float2(in0 ? c_win[in0 ? o0 : 0] : 0.0f, in1 ? c_win[in1 ? o1 : 0] : 0.0f);
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[q][k] = __ffma2_rn(w, make_float2(v[q], v[q]), acc[q][k]);
          }
        }
      }
      const float2 iz01 = make_float2(s_izx[hx], s_izx[hx + 1]), iz23 = make_float2(s_izx[hx + 2], s_izx[hx + 3]);
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const float2 lo = __fmul2_rn(acc[q][0], iz01), hi = __fmul2_rn(acc[q][1], iz23);
        *reinterpret_cast<float4*>(&s_h[q][hr][hx]) = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    }
    __syncthreads();
    {   // vertical pass + per-pixel SSIM of (vc, 2 vr) and (vc, 2 vr + 1)
      float2 acc2[5];   // rows (2 vr, 2 vr + 1), packed like the horizontal pass
#pragma unroll
      for (int q = 0; q < 5; ++q) acc2[q] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int p = 0; p < 2 + 2 * kR; ++p) {
        float v[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) v[q] = s_h[q][2 * vr + p][vc];
        const float2 w = make_float2(p <= 2 * kR ? c_win[p <= 2 * kR ? p : 0] : 0.0f, p >= 1 ? c_win[p >= 1 ? p - 1 : 0] : 0.0f);
#pragma unroll
        for (int q = 0; q < 5; ++q) acc2[q] = __ffma2_rn(w, make_float2(v[q], v[q]), acc2[q]);
      }
      float acc[5][2];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        acc[q][0] = acc2[q].x;
        acc[q][1] = acc2[q].y;
      }
      const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!vin[j]) continue;
        const int64_t i = static_cast<int64_t>(by + 2 * vr + j) * W + gx;
        const double mx = acc[0][j] * izy[j], my = acc[1][j] * izy[j], ex2 = acc[2][j] * izy[j],
                     ey2 = acc[3][j] * izy[j], exy = acc[4][j] * izy[j];
        const double a1 = 2.0 * mx * my + C1;
        const double a2 = 2.0 * (exy - mx * my) + C2;
        const double b1 = mx * mx + my * my + C1;
        const double b2 = (ex2 - mx * mx) + (ey2 - my * my) + C2;
        const double idn = 1.0 / (b1 * b2);
        const double sv = a1 * a2 * idn;
        ssum += sv;
        if (u) {
          const double d_a1 = a2 * idn, d_a2 = a1 * idn, d_b1 = -sv * b2 * idn, d_b2 = -sv * b1 * idn;
          u[ch * npix + i] = static_cast<float>((2.0 * my * d_a1 - 2.0 * my * d_a2 + 2.0 * mx * d_b1 - 2.0 * mx * d_b2) * weight);
          u[(3 + ch) * npix + i] = static_cast<float>(d_b2 * weight);
          u[(6 + ch) * npix + i] = static_cast<float>(2.0 * d_a2 * weight);
        }
      }
    }
    __syncthreads();   // s_h is rewritten by the next channel's horizontal pass
  }
  const double t = block_sum_d(ssum, s_red);
  if (tid == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

constexpr int kVG = 4;   // adjoint vertical outputs per thread (rows)

#ifndef GSF_SSIMB_MINB
#define GSF_SSIMB_MINB 4
#endif
__global__ void __launch_bounds__(256, GSF_SSIMB_MINB) k_ssim_bwd2(const float* __restrict__ u, const float* __restrict__ x,
                                                   const float* __restrict__ y, int W, int H, float* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_buf[];
  // two buffers of the channel's 3 adjoint planes + halo (channel ch + 1 streams in by cp.async
  // while ch is filtered), then the vertical pass's output
  float (*s_ub)[3][kSHh][kSW] = reinterpret_cast<float (*)[3][kSHh][kSW]>(s_buf);
  float (*s_t)[kSY][kSW] = reinterpret_cast<float (*)[kSY][kSW]>(s_buf + 2 * 3 * kSHh * kSW);
  __shared__ float s_wy[kSY][2 * kR + 1], s_wx[kSX][2 * kR + 1];
  const int64_t npix = static_cast<int64_t>(W) * H;
  const int bx = blockIdx.x * kSX, by = blockIdx.y * kSY;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < (kSY + kSX) * (2 * kR + 1); idx += 256) {
    const int row = idx / (2 * kR + 1), o = idx - row * (2 * kR + 1) - kR;
    if (row < kSY) {
      const int yy = by + row + o;
      s_wy[row][o + kR] = (yy >= 0 && yy < H) ? c_win[o + kR] / axis_norm(yy, H) : 0.0f;
    } else {
      const int xx = bx + (row - kSY) + o;
      s_wx[row - kSY][o + kR] = (xx >= 0 && xx < W) ? c_win[o + kR] / axis_norm(xx, W) : 0.0f;
    }
  }
  // horizontal-pass pixels of this thread: row hr, columns 2 hc and 2 hc + 1
  const int hr = tid >> 4, hc = (tid & 15) * 2;
  auto stage = [&](int ch) {
    for (int idx = tid; idx < kSHh * kSW; idx += 256) {
      const int r = idx / kSW, c = idx - r * kSW;
      const int gx = bx - kR + c, gy = by - kR + r;
      const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
      const int64_t j = in ? static_cast<int64_t>(gy) * W + gx : 0;
#pragma unroll
      for (int q = 0; q < 3; ++q) cp_async4_zfill(&s_ub[ch & 1][q][r][c], u + (3 * q + ch) * npix + j, in);
    }
    cp_async_commit();
  };
  stage(0);
  for (int ch = 0; ch < 3; ++ch) {
    __syncthreads();   // s_t and the buffer channel ch + 1 lands in (channel ch - 1's) are consumed
    if (ch + 1 < 3) {
      stage(ch + 1);
      cp_async_wait_1();   // channel ch has landed (this thread's copies)
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    float (*s_u)[kSHh][kSW] = s_ub[ch & 1];
    for (int item = tid; item < (kSY / kVG) * kSW; item += 256) {   // vertical adjoint: column c, rows r0 .. r0 + 3
      const int c = item % kSW, r0 = (item / kSW) * kVG;
      float2 acc[3][kVG / 2];   // rows (r0 + 2k, r0 + 2k + 1) on packed FFMA2 (0 * v outside the window: exact)
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int k = 0; k < kVG / 2; ++k) acc[q][k] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int p = 0; p < kVG + 2 * kR; ++p) {
        float v[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q] = s_u[q][r0 + p][c];
#pragma unroll
        for (int k = 0; k < kVG / 2; ++k) {
          const int o0 = p - 2 * k, o1 = o0 - 1;
          const bool in0 = o0 >= 0 && o0 <= 2 * kR, in1 = o1 >= 0 && o1 <= 2 * kR;
          if (in0 || in1) {
            const float2 w = make_float2(in0 ? s_wy[r0 + 2 * k][in0 ? o0 : 0] : 0.0f,
                                         in1 ? s_wy[r0 + 2 * k + 1][in1 ? o1 : 0] : 0.0f);
#pragma unroll
            for (int q = 0; q < 3; ++q) acc[q][k] = __ffma2_rn(w, make_float2(v[q], v[q]), acc[q][k]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int k = 0; k < kVG / 2; ++k) {
          s_t[q][r0 + 2 * k][c] = acc[q][k].x;
          s_t[q][r0 + 2 * k + 1][c] = acc[q][k].y;
        }
    }
    __syncthreads();
    {   // horizontal adjoint of (hc, hr), (hc + 1, hr)
      float2 acc2[3];   // columns (hc, hc + 1), packed
#pragma unroll
      for (int q = 0; q < 3; ++q) acc2[q] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int p = 0; p < 2 + 2 * kR; ++p) {
        float v[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q] = s_t[q][hr][hc + p];
        const float2 w = make_float2(p <= 2 * kR ? s_wx[hc][p <= 2 * kR ? p : 0] : 0.0f,
                                     p >= 1 ? s_wx[hc + 1][p >= 1 ? p - 1 : 0] : 0.0f);
#pragma unroll
        for (int q = 0; q < 3; ++q) acc2[q] = __ffma2_rn(w, make_float2(v[q], v[q]), acc2[q]);
      }
      float acc[3][2];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        acc[q][0] = acc2[q].x;
        acc[q][1] = acc2[q].y;
      }
      const int gy = by + hr;   // d_x = a0 + 2 a1 x + a2 y for this channel
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int gxx = bx + hc + j;
        if (gxx < W && gy < H) {
          const int64_t i = static_cast<int64_t>(gy) * W + gxx;
          dx[3 * i + ch] = acc[0][j] + 2.0f * acc[1][j] * x[3 * i + ch] + acc[2][j] * y[3 * i + ch];
        }
      }
    }
  }
}

// small-image fallback: global statistics (ssim.cpp:117-144), one block
__global__ void __launch_bounds__(256) k_ssim_global(const float* __restrict__ x, const float* __restrict__ y, int64_t n,
                                                     float* __restrict__ dx, double* part) {
  __shared__ double s_red[8];
  __shared__ double s_stat[15];
  __shared__ double s_part[9];
  for (int q = 0; q < 15; ++q) {
    const int c = q % 3, kind = q / 3;
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double xv = x[3 * i + c], yv = y[3 * i + c];
      a += kind == 0 ? xv : kind == 1 ? yv : kind == 2 ? xv * xv : kind == 3 ? yv * yv : xv * yv;
    }
    const double t = block_sum_d(a, s_red);
    if (threadIdx.x == 0) s_stat[q] = t / static_cast<double>(n);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double ssum = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double mx = s_stat[c], my = s_stat[3 + c], ex2 = s_stat[6 + c], ey2 = s_stat[9 + c], exy = s_stat[12 + c];
      const double a1 = 2.0 * mx * my + C1, a2 = 2.0 * (exy - mx * my) + C2;
      const double b1 = mx * mx + my * my + C1, b2 = (ex2 - mx * mx) + (ey2 - my * my) + C2;
      const double denom = b1 * b2, sv = a1 * a2 / denom;
      ssum += sv;
      const double d_a1 = a2 / denom, d_a2 = a1 / denom, d_b1 = -sv / b1, d_b2 = -sv / b2;
      s_part[c] = 2.0 * my * d_a1 - 2.0 * my * d_a2 + 2.0 * mx * d_b1 - 2.0 * mx * d_b2;
      s_part[3 + c] = d_b2;
      s_part[6 + c] = 2.0 * d_a2;
    }
    // reported as a per-pixel sum so the finaliser's 1 - sum/(3n) is the channel mean
    part[0] = ssum * static_cast<double>(n);
  }
  __syncthreads();
  if (dx) {
    const double inv = 1.0 / static_cast<double>(n);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      for (int c = 0; c < 3; ++c)
        dx[3 * i + c] = static_cast<float>((s_part[c] + 2.0 * s_part[3 + c] * x[3 * i + c] + s_part[6 + c] * y[3 * i + c]) *
                                           (inv / 3.0));
  }
}

__global__ void __launch_bounds__(256) k_iso(const float* __restrict__ params, int64_t P, const uint8_t* __restrict__ visible,
                                             const DevState* ds, double w_iso, double eps, int add_grad,
                                             float* __restrict__ grads, double* __restrict__ part) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  __shared__ double s_red[8];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (i < P && visible[i] && !ds->halt) {
    const double s[3] = {exp(static_cast<double>(params[3 * P + i])), exp(static_cast<double>(params[4 * P + i])),
                         exp(static_cast<double>(params[5 * P + i]))};
    int a = 0, b = 0;
    for (int c = 1; c < 3; ++c) {
      if (s[c] > s[a]) a = c;
      if (s[c] < s[b]) b = c;
    }
    const double ratio = s[a] / s[b];
    term = (ratio > eps ? ratio : eps) - eps;
    if (add_grad && ratio > eps && w_iso > 0.0) {
      const double g = w_iso * ratio / static_cast<double>(ds->V);
      grads[(3 + a) * P + i] = static_cast<float>(static_cast<double>(grads[(3 + a) * P + i]) + g);
      grads[(3 + b) * P + i] = static_cast<float>(static_cast<double>(grads[(3 + b) * P + i]) - g);
    }
  }
  if (add_grad) return;
  const double t = block_sum_d(term, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

}  // namespace

static bool g_win_ready = false;

static void ensure_window() {
  if (g_win_ready) return;
  float w[11];
  for (int i = 0; i <= 10; ++i) {
    const double d = i - 5;
    w[i] = static_cast<float>(std::exp(-d * d / (2.0 * 1.5 * 1.5)));
  }
  GSF_CUDA_CHECK(cudaMemcpyToSymbol(c_win, w, sizeof(w)));
  g_win_ready = true;
}

void run_loss_finalize(Workspace& ws, DevState* ds, const LossParams& lp, int tiles, int64_t npix, int iteration,
                       cudaStream_t st, int64_t* L) {
  // red_part layout: [0, 4096) ssim block partials, [4096, 8192+) iso block partials
  const int ssim_blocks = lp.mode == 2 && lp.w_ssim > 0.0 ? ws.ssim_blocks : 0;
  const int iso_blocks = lp.mode == 2 ? ws.iso_blocks : 0;
  if (ws.loss_rows > 0) tiles = ws.loss_rows;   // the producer's row count (4 per tile for k_blend_track_w)
  launch_pdl(k_loss_finalize, dim3(1), dim3(1024), 0, st, ws.loss_part, tiles, npix, lp, iteration, ws.red_part, ssim_blocks,
                                     ws.red_part + ws.red_iso_offset, iso_blocks, ds);
  ++*L;
}

void run_ssim(Workspace& ws, DevState* ds, const float* x, const float* y, int W, int H, float /*unused*/, float* d_out,
              cudaStream_t st, int64_t* L) {
  (void)ds;
  ensure_window();
  const int64_t npix = static_cast<int64_t>(W) * H;
  if (W < 11 || H < 11) {
    k_ssim_global<<<1, 256, 0, st>>>(x, y, npix, d_out, ws.red_part);
    ++*L;
    ws.ssim_blocks = 1;
    return;
  }
  static bool attr = false;
  if (!attr) {
    GSF_CUDA_CHECK(cudaFuncSetAttribute(k_ssim_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(ssim_fwd2_smem())));
    GSF_CUDA_CHECK(cudaFuncSetAttribute(k_ssim_bwd2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(ssim_bwd2_smem())));
    attr = true;
  }
  const dim3 grid(div_up(W, kSX), div_up(H, kSY));
  float* u = ws.ssim_tmp;                 // 9 adjoint seed planes
  if (ws.prof) ws.prof->begin(PROF_SSIM, st);
  launch_pdl(k_ssim_fwd2, grid, dim3(256), ssim_fwd2_smem(), st, x, y, W, H, 1.0 / (3.0 * static_cast<double>(npix)),
             d_out ? u : nullptr, ws.red_part);
  ++*L;
  ws.ssim_blocks = static_cast<int>(grid.x * grid.y);
  if (d_out) {
    launch_pdl(k_ssim_bwd2, grid, dim3(256), ssim_bwd2_smem(), st, u, x, y, W, H, d_out);
    ++*L;
  }
  if (ws.prof) ws.prof->end(st);
}

void run_iso(Workspace& ws, DevState* ds, const float* params, int64_t P, double w_iso, double eps, float* grads,
             cudaStream_t st, int64_t* L) {
  if (P <= 0) { ws.iso_blocks = 0; return; }
  const int blocks = div_up(P, 256);
  launch_pdl(k_iso, dim3(blocks), dim3(256), 0, st, params, P, ws.visible, ds, w_iso, eps, grads ? 1 : 0, grads, ws.red_part + ws.red_iso_offset);
  ++*L;
  if (!grads) ws.iso_blocks = blocks;
}

}  // namespace gsfk
