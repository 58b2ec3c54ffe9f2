// raster_fwd.cu — forward pass of the tile rasterizer on sm_100a.
//
//   k_preprocess   project_all (rasterizer.cpp:46-67) + validate_primitives (:34-44), fp64,
//                  one thread per primitive, SoA fp32 parameter reads (coalesced per field);
//                  also counts the visible primitives, histograms their tile rectangles
//                  (warp-cooperative atomics) and, for tracking, emits the pose Jacobians
//   binning        (binning.cu) per-tile lists in exact (depth, id) order (:69-79, :193-212)
//   k_blend        blend_pixel (:96-140) for a 16x16 tile per 256-thread CTA with the tile
//                  list staged through shared memory, plus the fused loss epilogue
//                  (losses.cpp:156-339: masks, residual sums and counts per tile)
#include "kernels.h"
#include "pixel_loss.cuh"
#include "finalize.cuh"

namespace gsfk {

namespace {

// Per-primitive linear map from the six screen-space partials of one (tile, primitive) pair
// (d_mean2d x/y, d_cov2d 00/01/11, d_depth [+ d_color for view-dependent SH]) to the SE(3)
// pose gradient: the camera part of render_backward phase 2 (rasterizer.cpp:495-526, 548-558)
// linearised per primitive in fp64, so the tracking backward can apply it right after its
// per-tile reduction instead of round-tripping every pair partial through memory.
// Output: the 6 x 9 matrix M with pose = sum_j M[:, j] s_j, column-major (kPjFloats floats):
// columns j = 0..5 take the screen partials s = (d_mean2d x, y, d_cov2d 00, 01, 11 without the
// 1/2 of d_conic, d_depth); columns 6..8 the view-dependent colour partials (zero unless K > 1).
// Rows: rot0 rot1 rot2 trans0 trans1 trans2, so the kernel accumulates three float2 pairs with
// packed FFMA2s.  In fp64: d = A s (A from J, Bc), rot = p_cam x d + Cr s_cov, trans = d.
__device__ void compute_posejac(const float* __restrict__ p, int64_t stride, const Cam& cam, int K, float* out,
                                const double* Sw, const BlendG* conic = nullptr) {
  const double m0 = p[0], m1 = p[stride], m2 = p[2 * stride];
  const double* W = cam.W;
  const double pc[3] = {W[0] * m0 + W[1] * m1 + W[2] * m2 + cam.t[0], W[3] * m0 + W[4] * m1 + W[5] * m2 + cam.t[1],
                        W[6] * m0 + W[7] * m1 + W[8] * m2 + cam.t[2]};
  const double iz = 1.0 / pc[2], iz2 = iz * iz, iz3 = iz2 * iz;
  const double J00 = cam.fx * iz, J02 = -cam.fx * pc[0] * iz2, J11 = cam.fy * iz, J12 = -cam.fy * pc[1] * iz2;
  double Cw[3][3], T1[3][3], V[3][3];
  if (Sw) {   // world covariance from the per-frame cache
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Cw[a][b] = Sw[3 * a + b];
  } else {
    const double qw0 = p[6 * stride], qx0 = p[7 * stride], qy0 = p[8 * stride], qz0 = p[9 * stride];
    const double ql = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
    const double w = qw0 / ql, x = qx0 / ql, y = qy0 / ql, z = qz0 / ql;
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    double s2[3];
    for (int a = 0; a < 3; ++a) {
      const double sa = exp(static_cast<double>(p[(3 + a) * stride]));
      s2[a] = sa * sa;
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Cw[a][b] = R[a][0] * s2[0] * R[b][0] + R[a][1] * s2[1] * R[b][1] + R[a][2] * s2[2] * R[b][2];
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) T1[a][b] = W[3 * a] * Cw[0][b] + W[3 * a + 1] * Cw[1][b] + W[3 * a + 2] * Cw[2][b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) V[a][b] = T1[a][0] * W[3 * b] + T1[a][1] * W[3 * b + 1] + T1[a][2] * W[3 * b + 2];
  double G[2][3];
  for (int b = 0; b < 3; ++b) {
    G[0][b] = J00 * V[0][b] + J02 * V[2][b];
    G[1][b] = J11 * V[1][b] + J12 * V[2][b];
  }
  const double ax = -cam.fx * iz2, ay = -cam.fy * iz2, bx = 2.0 * cam.fx * pc[0] * iz3, by = 2.0 * cam.fy * pc[1] * iz3;
  // d_p_cam from (s2, s3, s4) via d_jac = 2 dC J V (rasterizer.cpp:504-513)
  const double Bc[3][3] = {{2.0 * G[0][2] * ax, 2.0 * G[1][2] * ax, 0.0},
                           {0.0, 2.0 * G[0][2] * ay, 2.0 * G[1][2] * ay},
                           {2.0 * (ax * G[0][0] + bx * G[0][2]),
                            2.0 * (ax * G[1][0] + ay * G[0][1] + bx * G[1][2] + by * G[0][2]),
                            2.0 * (ay * G[1][1] + by * G[1][2])}};
  // rot += sum dCc .* (E_j V - V E_j) = -2 vee(V dCc - dCc V), dCc = s2 J0J0^T + s3 (J0J1^T + J1J0^T) + s4 J1J1^T
  const double J0[3] = {J00, 0.0, J02}, J1[3] = {0.0, J11, J12};
  double Cr[3][3];
  for (int k = 0; k < 3; ++k) {
    double Dk[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        Dk[a][b] = k == 0 ? J0[a] * J0[b] : (k == 1 ? J0[a] * J1[b] + J1[a] * J0[b] : J1[a] * J1[b]);
    double M[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double vd = 0.0, dv = 0.0;
        for (int c = 0; c < 3; ++c) { vd += V[a][c] * Dk[c][b]; dv += Dk[a][c] * V[c][b]; }
        M[a][b] = vd - dv;
      }
    Cr[0][k] = -2.0 * M[2][1];
    Cr[1][k] = -2.0 * M[0][2];
    Cr[2][k] = -2.0 * M[1][0];
  }
  double Tc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (K > 1) {   // view-dependent colour: trans += W (I - dir dir^T)/len * dDir/dColour (sh.cpp:88-108)
    const double d0 = m0 - cam.center[0], d1 = m1 - cam.center[1], d2 = m2 - cam.center[2];
    const double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (len > 1e-12) {
      const double dir[3] = {d0 / len, d1 / len, d2 / len};
      const int deg = sh_degree(K);
      double b[16], gb[48];
      sh_basis(deg, dir[0], dir[1], dir[2], b);
      sh_basis_grad_d(deg, dir[0], dir[1], dir[2], gb);
      double Dm[3][3];   // d_dir = Dm * d_colour
      for (int c = 0; c < 3; ++c) {
        double raw = 0.5;
        for (int k = 0; k < K; ++k) raw += b[k] * p[(11 + 3 * k + c) * stride];
        const double mask = raw < 0.0 ? 0.0 : 1.0;
        for (int a = 0; a < 3; ++a) {
          double acc = 0.0;
          for (int k = 1; k < K; ++k) acc += gb[3 * k + a] * p[(11 + 3 * k + c) * stride];
          Dm[a][c] = mask * acc;
        }
      }
      double Pm[3][3];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) Pm[a][c] = ((a == c ? 1.0 : 0.0) - dir[a] * dir[c]) / len;
      double PD[3][3];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) PD[a][c] = Pm[a][0] * Dm[0][c] + Pm[a][1] * Dm[1][c] + Pm[a][2] * Dm[2][c];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) Tc[a][c] = W[3 * a] * PD[0][c] + W[3 * a + 1] * PD[1][c] + W[3 * a + 2] * PD[2][c];
    }
  }
  const double A[3][6] = {{J00, 0.0, Bc[0][0], Bc[0][1], Bc[0][2], 0.0},
                          {0.0, J11, Bc[1][0], Bc[1][1], Bc[1][2], 0.0},
                          {J02, J12, Bc[2][0], Bc[2][1], Bc[2][2], 1.0}};
  double Mc[6][6];
  for (int j = 0; j < 6; ++j) {
    const double d0 = A[0][j], d1 = A[1][j], d2 = A[2][j];
    double col[6] = {pc[1] * d2 - pc[2] * d1, pc[2] * d0 - pc[0] * d2, pc[0] * d1 - pc[1] * d0, d0, d1, d2};
    if (j >= 2 && j <= 4)
      for (int a = 0; a < 3; ++a) col[a] += Cr[a][j - 2];
    const double scale = (j >= 2 && j <= 4) ? 0.5 : 1.0;   // the kernel's s_cov carries no 1/2
    for (int a = 0; a < 6; ++a) Mc[j][a] = scale * col[a];
  }
  if (conic) {
    // Columns re-expressed in the pixel-offset basis t = g (dx, dy, dx^2, dx dy, dy^2) the two-pixel
    // pose backward forms directly: with the record's conic (c00, c01, c11) the screen partials are
    // s0 = c00 t0 + c01 t1, s1 = c01 t0 + c11 t1, s2 = g ux^2, s3 = g ux uy, s4 = g uy^2 (ux, uy linear in dx, dy)
    const double c00 = conic->c00, c01 = 0.5 * static_cast<double>(conic->c01x2), c11 = conic->c11;
    double N[5][6];
    for (int a = 0; a < 6; ++a) {
      N[0][a] = c00 * Mc[0][a] + c01 * Mc[1][a];
      N[1][a] = c01 * Mc[0][a] + c11 * Mc[1][a];
      N[2][a] = c00 * c00 * Mc[2][a] + c00 * c01 * Mc[3][a] + c01 * c01 * Mc[4][a];
      N[3][a] = 2.0 * c00 * c01 * Mc[2][a] + (c00 * c11 + c01 * c01) * Mc[3][a] + 2.0 * c01 * c11 * Mc[4][a];
      N[4][a] = c01 * c01 * Mc[2][a] + c01 * c11 * Mc[3][a] + c11 * c11 * Mc[4][a];
    }
    for (int j = 0; j < 5; ++j)
      for (int a = 0; a < 6; ++a) Mc[j][a] = N[j][a];
  }
  for (int j = 0; j < 6; ++j)
    for (int a = 0; a < 6; ++a) out[6 * j + a] = static_cast<float>(Mc[j][a]);
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 6; ++a) out[36 + 6 * c + a] = a < 3 ? 0.0f : static_cast<float>(Tc[a - 3][c]);
  out[54] = out[55] = 0.0f;
}

// Validation + view-independent part of every primitive, once per tracked frame (the map is
// constant inside track_frame).  Invalid primitives get a NaN support and report bad_index.
__global__ void __launch_bounds__(256) k_world(const float* __restrict__ params, int64_t P, RasterParams rp,
                                               WorldG* __restrict__ world, double* __restrict__ support,
                                               int32_t* bad_index, uint32_t* ncand) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0 && ncand) *ncand = 0u;
  if (i >= P) return;
  const int D = kFieldsBase + 3 * rp.sh_coeffs;
  float v[kFieldsBase];
#pragma unroll
  for (int f = 0; f < kFieldsBase; ++f) v[f] = params[f * P + i];
  bool ok = true;
#pragma unroll
  for (int f = 0; f < kFieldsBase; ++f) ok &= isfinite(v[f]);
  for (int f = kFieldsBase; f < D; ++f) ok &= isfinite(params[f * P + i]);
  {
    const double qw = v[6], qx = v[7], qy = v[8], qz = v[9];
    ok &= dsqrt(dadd(dadd(dadd(dmul(qw, qw), dmul(qx, qx)), dmul(qy, qy)), dmul(qz, qz))) > 1e-12;
  }
  if (!ok) {
    atomicMin(bad_index, static_cast<int32_t>(i));
    support[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  support[i] = world_support(params + i, P, rp);
  world[i] = make_world(params + i, P, rp.sh_coeffs);
}

// Candidates of the tracking loop (once per frame, after k_world).  While the camera stays within
// (theta_max, dist_max) of the frame's first camera, a primitive's camera-space centre moves by at
// most eps = theta_max |p| + dist_max (p at the first camera; track_update checks the region after
// every step), so its support ball stays inside B(p, r + eps).  project_gaussian's necessary tests
// (projection.cpp:62-76: depth range, support ball in front of the camera, padded support box on
// the image; the box test is monotone in the radius) evaluated for that larger ball can only keep
// more primitives, never fewer: the lists the preprocess builds from the candidates are the full
// ones, bit for bit.  Margins of 1e-9 relative cover the rounding of this fp64 test.
__device__ __forceinline__ void axis_bounds_d(double a, double z, double r, double f, double c, double& lo, double& hi) {
  lo = 1e300;
  hi = -1e300;
  for (int e = 0; e < 4; ++e) {
    const double u = c + f * (a + ((e & 1) ? r : -r)) / (z + ((e & 2) ? r : -r));
    lo = fmin(lo, u);
    hi = fmax(hi, u);
  }
}

__global__ void __launch_bounds__(256) k_candidates(int64_t P, DevState* ds, RasterParams rp,
                                                    const float* __restrict__ params, const double* __restrict__ support,
                                                    double theta_max, double dist_max, uint32_t* __restrict__ cand) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const Cam& cam = ds->cam;
  if (i == 0) {
    for (int a = 0; a < 9; ++a) ds->cand_W0[a] = cam.W[a];
    for (int a = 0; a < 3; ++a) ds->cand_t0[a] = cam.t[a];
    ds->cand_cos_min = cos(theta_max);
    ds->cand_dist_max = dist_max;
    ds->cand_ok = 1;
  }
  bool keep = false;
  if (i < P) {
    const double r = support[i];
    if (!isnan(r)) {
      const double m0 = params[i], m1 = params[P + i], m2 = params[2 * P + i];
      double p[3];
      for (int a = 0; a < 3; ++a) p[a] = cam.W[3 * a] * m0 + cam.W[3 * a + 1] * m1 + cam.W[3 * a + 2] * m2 + cam.t[a];
      const double n = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
      const double eps = (theta_max * n + dist_max) * (1.0 + 1e-9) + 1e-9 * (1.0 + n);
      keep = p[2] + eps > cam.near_plane && p[2] - eps < cam.far_plane;   // depth range
      if (keep && r > 0.0) {
        keep = p[2] + eps - r > 0.0;                                      // ball in front
        const double R = r + eps;
        if (keep && p[2] - R > 0.0) {                                     // padded support box
          const double pad = rp.footprint_sigma * sqrt(fmax(0.0, rp.dilation)) + 1e-6;
          double ulo, uhi, vlo, vhi;
          axis_bounds_d(p[0], p[2], R, cam.fx, cam.cx, ulo, uhi);
          axis_bounds_d(p[1], p[2], R, cam.fy, cam.cy, vlo, vhi);
          keep = !(uhi + pad < 0.0 || ulo - pad > cam.width || vhi + pad < 0.0 || vlo - pad > cam.height);
        }
      }
    }
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0 && bits) base = atomicAdd(&ds->ncand, static_cast<uint32_t>(__popc(bits)));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) cand[base + __popc(bits & ((1u << lane) - 1u))] = static_cast<uint32_t>(i);
}

// CACHED: the world part comes from k_world (tracking loop); otherwise every primitive is
// validated and projected from its parameters (validate_primitives + project_all).
template <bool CACHED>
#ifndef GSF_PRE_MINB
#define GSF_PRE_MINB 4
#endif
__global__ void __launch_bounds__(256, CACHED ? GSF_PRE_MINB : 2) k_preprocess(const float* __restrict__ params, int64_t P, const DevState* ds,
                                                    RasterParams rp, BlendG* __restrict__ bg_id, GuardG* __restrict__ gg_id,
                                                    double* __restrict__ depth_id, int4* __restrict__ rect_id,
                                                    uint8_t* __restrict__ visible, int32_t* bad_index, BlendConsts kc,
                                                    uint32_t* counters, uint32_t* __restrict__ vis_list,
                                                    uint32_t* __restrict__ pj_slot, uint32_t* __restrict__ fill,
                                                    uint32_t bucket_cap, unsigned long long* __restrict__ bucket,
                                                    uint32_t* __restrict__ big_ids, uint32_t* __restrict__ pair_base,
                                                    const WorldG* __restrict__ world, const double* __restrict__ support,
                                                    const uint32_t* __restrict__ cand) {
  __shared__ uint32_t s_vis[8];
  __shared__ uint32_t s_base;
  __shared__ Cam s_cam;   // read through shared memory: 20 doubles need not live in registers
  pdl_wait();   // the camera comes from the previous iteration's pose step
  pdl_trigger();
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (cand && ds->cand_ok) {   // inside the trust region: only the frame's candidates (k_candidates)
    const uint32_t n = ds->ncand;
    if (static_cast<uint32_t>(blockIdx.x) * blockDim.x >= n) return;   // whole CTA, before any barrier
    i = i < n ? static_cast<int64_t>(cand[i]) : P;
  }
  if (threadIdx.x < sizeof(Cam) / 4)
    reinterpret_cast<uint32_t*>(&s_cam)[threadIdx.x] = reinterpret_cast<const uint32_t*>(&ds->cam)[threadIdx.x];
  __syncthreads();
  const Cam& cam = s_cam;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool vis = false;
  int4 q = make_int4(0, -1, 0, -1);
  if (i < P) {
    PreOut o;
    bool ok = true;
    if (CACHED) {
      const double sup = support[i];
      ok = !isnan(sup);
      if (ok) {
        const double m0 = params[i], m1 = params[P + i], m2 = params[2 * P + i];
        o = project_core(m0, m1, m2, sup, CachedSrc{world + i, ParamSrc{params + i, P, rp.sh_coeffs}}, cam, rp);
      }
    } else {
      // validate_primitives (rasterizer.cpp:34-44): every field finite and |q| > 1e-12
      // (all loads issued before any test: no short-circuit chain of dependent memory latencies)
      const int D = kFieldsBase + 3 * rp.sh_coeffs;
      float v[kFieldsBase];
#pragma unroll
      for (int f = 0; f < kFieldsBase; ++f) v[f] = params[f * P + i];
#pragma unroll
      for (int f = 0; f < kFieldsBase; ++f) ok &= isfinite(v[f]);
      for (int f = kFieldsBase; f < D; ++f) ok &= isfinite(params[f * P + i]);
      {
        const double qw = v[6], qx = v[7], qy = v[8], qz = v[9];
        ok &= dsqrt(dadd(dadd(dadd(dmul(qw, qw), dmul(qx, qx)), dmul(qy, qy)), dmul(qz, qz))) > 1e-12;
      }
      if (!ok) atomicMin(bad_index, static_cast<int32_t>(i));
      else o = preprocess_one(params + i, P, cam, rp);
    }
    if (!ok) {
      visible[i] = 0;
    } else {
      visible[i] = static_cast<uint8_t>(o.visible);
      if (o.visible) {
        vis = true;
        BlendG g = make_blend_g(o);
        blend_rho_bounds(g, kc);
        bg_id[i] = g;
        gg_id[i] = make_guard_g(o);
        depth_id[i] = o.depth;
        q = make_int4(o.tx0, o.tx1, o.ty0, o.ty1);
        rect_id[i] = q;
      }
    }
  }
  // a CTA with no visible primitive has no pair, slot or list entry to emit: skip the CTA scans
  if (!__syncthreads_or(vis)) return;
  const uint32_t bits = __ballot_sync(0xffffffffu, vis);
  if (lane == 0) s_vis[warp] = static_cast<uint32_t>(__popc(bits));
  // tile binning (binning.cu): every (tile, primitive) pair into its tile's bucket
  {
    const int tiles_x = rp.tiles_x;
    const int w = q.y - q.x + 1;
    int c = vis ? w * (q.w - q.z + 1) : 0;
    if (pair_base) {
      // primitive-major pair slots (pair_base[id] + rectangle index) for the mapping backward and
      // its chain: a CTA scan of the pair counts plus one atomic per CTA (any order is fine: the
      // chain reads each primitive's own slots in rectangle order)
      __shared__ uint32_t s_w[8];
      __shared__ uint32_t s_cta;
      const int ex = warp_excl_scan(c);
      if (lane == 31) s_w[warp] = static_cast<uint32_t>(ex + c);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s_w[k];
        s_cta = t ? atomicAdd(&counters[kCntPairAlloc], t) : 0u;
      }
      __syncthreads();
      if (vis) {
        uint32_t b = s_cta + static_cast<uint32_t>(ex);
        for (int k = 0; k < warp; ++k) b += s_w[k];
        pair_base[i] = b;
      }
    }
    if (c > kBigPairs) {   // k_scatter_big's
      big_ids[atomicAdd(&counters[kCntBig], 1u)] = static_cast<uint32_t>(i);
      c = 0;
    }
    const unsigned long long key = vis ? pair_key(depth_id[i], static_cast<uint32_t>(i)) : 0ull;
    const int excl = warp_excl_scan(c);
    const int total = __shfl_sync(0xffffffffu, excl + c, 31);
    // GSF_SCATTER_U pairs per lane per round: every fill-counter atomic of the round is in flight
    // before the first key store waits on its slot
#ifndef GSF_SCATTER_U
#define GSF_SCATTER_U 8
#endif
    constexpr int kScatterU = GSF_SCATTER_U;
    for (int base = 0; base < total; base += 32 * kScatterU) {
      int tt[kScatterU];
      unsigned long long kk[kScatterU];
      uint32_t sl[kScatterU];
#pragma unroll
      for (int u = 0; u < kScatterU; ++u) {
        const int k = base + 32 * u + lane;
        const int j = warp_owner(excl, k);   // lane whose pair range holds k
        const int qx0 = __shfl_sync(0xffffffffu, q.x, j), qy0 = __shfl_sync(0xffffffffu, q.z, j);
        const int wj = __shfl_sync(0xffffffffu, w, j), ej = __shfl_sync(0xffffffffu, excl, j);
        kk[u] = __shfl_sync(0xffffffffu, key, j);
        const int r = k - ej;
        const int row = r / max(wj, 1);
        tt[u] = k < total ? (qy0 + row) * tiles_x + qx0 + (r - row * wj) : -1;
      }
#pragma unroll
      for (int u = 0; u < kScatterU; ++u)
        if (tt[u] >= 0) sl[u] = atomicAdd(&fill[static_cast<int64_t>(tt[u]) * kBinStride], 1u);
#pragma unroll
      for (int u = 0; u < kScatterU; ++u)
        if (tt[u] >= 0 && sl[u] < bucket_cap) bucket[static_cast<int64_t>(tt[u]) * bucket_cap + sl[u]] = kk[u];
    }
  }
  // visible count (one atomic per CTA) and, for the pose Jacobians, the list of visible ids
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t n = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) n += s_vis[w];
    s_base = n ? atomicAdd(&counters[kCntVisible], n) : 0u;
  }
  __syncthreads();
  if (vis_list && vis) {
    uint32_t off = s_base;
    for (int w = 0; w < warp; ++w) off += s_vis[w];
    const uint32_t r = off + __popc(bits & ((1u << lane) - 1u));
    vis_list[r] = static_cast<uint32_t>(i);
    pj_slot[i] = r;
  }
}

// Pose Jacobians of the visible primitives (tracking), one thread per listed id; slot r of the
// list owns pj[kPjFloats r, kPjFloats (r + 1)), staged through shared memory so the CTA writes one contiguous,
// coalesced block.
constexpr int kPjThreads = 128;
#ifndef GSF_PJ_MINB
#define GSF_PJ_MINB 1
#endif
__global__ void __launch_bounds__(kPjThreads, GSF_PJ_MINB) k_posejac(const float* __restrict__ params, int64_t P, const DevState* ds, int K,
                                                 const uint32_t* __restrict__ vis_list, const uint32_t* counters,
                                                 const WorldG* __restrict__ world, float* __restrict__ pj,
                                                 const BlendG* __restrict__ bg_id, const GuardG* __restrict__ gg_id,
                                                 BlendG* __restrict__ bg_slot, GuardG* __restrict__ gg_slot) {
  __shared__ float s_out[kPjThreads * (kPjFloats + 1)];
  const uint32_t n = counters[kCntVisible];
  const uint32_t r0 = blockIdx.x * blockDim.x;
  if (r0 >= n || ds->halt) return;
  const uint32_t r = r0 + threadIdx.x;
  if (r < n) {
    const uint32_t id = vis_list[r];
    bg_slot[r] = bg_id[id];   // the tracking kernels read records by visible slot (compact, no id hop)
    gg_slot[r] = gg_id[id];
    float v[kPjFloats];
    // K == 1: columns in the two-pixel backward's offset basis (k_backward_track_w); the view-dependent
    // pose backward (k_backward_pose) takes the screen-partial basis
    const BlendG rec = bg_id[id];
    compute_posejac(params + id, P, ds->cam, K, v, world ? world[id].S : nullptr, K == 1 ? &rec : nullptr);
#pragma unroll
    for (int q = 0; q < kPjFloats; ++q) s_out[threadIdx.x * (kPjFloats + 1) + q] = v[q];
  }
  __syncthreads();
  const uint32_t cnt = min(static_cast<uint32_t>(kPjThreads), n - r0);
  float* dst = pj + kPjFloats * static_cast<size_t>(r0);
  for (uint32_t e = threadIdx.x; e < kPjFloats * cnt; e += kPjThreads)
    dst[e] = s_out[(e / kPjFloats) * (kPjFloats + 1) + e % kPjFloats];
}

__device__ __forceinline__ bool depth_valid(float d, double near_plane, double far_plane) {
  const double v = d;
  return isfinite(v) && v > near_plane && v < far_plane;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// pixel_accumulate (gsf_shared.cuh) with the colour / alpha-depth sums as two packed FFMA2s;
// every lane rounds like __fmaf_rn, so the state equals the mirror's bit for bit.
template <bool FLAG, bool DOM = true>
__device__ __forceinline__ void full_accumulate(PixelState& s, float2& rg, float2& bd, const BlendG& g, const PairEval& e,
                                                int32_t id, int32_t list_index, bool obs_valid, float obs,
                                                const BlendConsts& k) {
  const float w = fmul(e.alpha, s.T);
  if (FLAG) pixel_flag_step(s, e.alpha, e.clamped, w, fmul(s.T, fsub(1.0f, e.alpha)), k);
  const float2 ww = make_float2(w, w);
  rg = __ffma2_rn(ww, make_float2(g.r, g.g), rg);
  bd = __ffma2_rn(ww, make_float2(g.b, g.depth), bd);
  s.op = fadd(s.op, w);
  if (obs_valid) {
    const float d = fsub(g.depth, obs);
    s.unc = ffma(fmul(w, d), d, s.unc);
  }
  if (DOM) {   // the dominant contributor and the count: the render API and the uncertainty pass
    if (w > s.best) {
      s.best = w;
      s.dominant = id;
    }
    s.count += 1;
  }
  s.last = list_index + 1;
  const float t_next = fmul(s.T, fsub(1.0f, e.alpha));
  if (s.median < 0 && s.T >= 0.5f && t_next < 0.5f) {
    s.median = id;
    s.med_depth = g.depth;
  }
  s.T = t_next;
  if (s.T < k.term) s.done = 1;
}

// Plain render (LMODE 0) and the mapping forward with its fused loss partials (LMODE 2); the
// tracking forward is k_blend_track below.
template <int LMODE>
#ifndef GSF_BLEND_MINB
#define GSF_BLEND_MINB 4
#endif
__global__ void __launch_bounds__(256, GSF_BLEND_MINB) k_blend(const int2* __restrict__ ranges, const uint32_t* __restrict__ sid,
                                               const BlendG* __restrict__ bg, const GuardG* __restrict__ gg,
                                               const float* __restrict__ obs, const float* __restrict__ loss_rgb,
                                               const float* __restrict__ loss_depth, int W, int H, int tiles_x,
                                               BlendConsts kc, double near_plane, double far_plane, LossParams lp,
                                               DevState* ds, float* __restrict__ o_color, float* __restrict__ o_ad,
                                               float* __restrict__ o_md, uint8_t* __restrict__ o_mv,
                                               float* __restrict__ o_op, float* __restrict__ o_unc,
                                               float* __restrict__ o_T, int32_t* __restrict__ o_count,
                                               int32_t* __restrict__ o_dom, int32_t* __restrict__ o_med,
                                               float* __restrict__ o_domw, int32_t* __restrict__ o_last,
                                               double* __restrict__ loss_part, int fuse_final, int iteration,
                                               uint32_t* ticket, uint32_t* __restrict__ fix_list, uint32_t* fix_cnt,
                                               int2* __restrict__ qstat) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  __shared__ __align__(16) BlendG s_g[256];
  __shared__ uint32_t s_ws[8];
  __shared__ int32_t s_id[256];
  __shared__ uint8_t s_mask[256];
  __shared__ double s_red[8][LS_NUM];
  if (ds->halt) return;
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x = tx * kTile + tile_lx(tid), y = ty * kTile + tile_ly(tid);
  const bool inside = x < W && y < H;
  const int64_t pi = static_cast<int64_t>(y) * W + x;
  const int2 rg = ranges[tile];
  PixelState s;
  pixel_init(s);
  if (!inside) s.done = 1;
  float2 frg = make_float2(0.0f, 0.0f), fbd = make_float2(0.0f, 0.0f);   // colour (r, g), (b, alpha depth)
  bool obs_valid = false;
  float ov = 0.0f;
  if (obs && inside) {
    ov = obs[pi];
    obs_valid = depth_valid(ov, near_plane, far_plane);
  }
  const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
  const int lane = tid & 31, warp = tid >> 5;
  const float tile_x0 = static_cast<float>(tx * kTile), tile_y0 = static_cast<float>(ty * kTile);
  uint32_t wsteps = 0u;   // this warp's (warp, entry) steps: the LPT cost of the mapping backward's quadrants
  for (int start = rg.x; start < rg.y; start += 256) {
    if (__syncthreads_and(s.done)) break;
    const int j = start + tid;
    if (j < rg.y) {
      const int id = static_cast<int>(sid[j]);
      const BlendG gj = bg[id];
      s_g[tid] = gj;
      s_id[tid] = id;
      s_mask[tid] = static_cast<uint8_t>(warp_block_mask(gj, tile_x0, tile_y0, kc));
    }
    __syncthreads();
    const int cnt = min(256, rg.y - start);
    // each warp walks only the entries whose footprint can reach its 8x4 block, in list order
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int kk = c0 + lane;
      uint32_t bits = __ballot_sync(0xffffffffu, kk < cnt && ((s_mask[kk] >> warp) & 1u));
      wsteps += __popc(bits);
      while (bits) {
        const int k = c0 + __ffs(bits) - 1;
        bits &= bits - 1u;
        if (s.done) continue;
        const BlendG g = s_g[k];
        const PairEval e = eval_pair(px, py, g, gg + s_id[k], kc);
        // the mapping objective reads neither the dominant contributor nor the count (LMODE 2)
        if (e.code) full_accumulate<LMODE == 0, LMODE != 2>(s, frg, fbd, g, e, s_id[k], start + k - rg.x, obs_valid, ov, kc);
      }
    }
  }
  s.cr = frg.x;
  s.cg = frg.y;
  s.cb = fbd.x;
  s.ad = fbd.y;
  if (inside) {
    o_color[3 * pi + 0] = s.cr;
    o_color[3 * pi + 1] = s.cg;
    o_color[3 * pi + 2] = s.cb;
    o_ad[pi] = s.ad;
    o_op[pi] = s.op;
    o_T[pi] = s.T;
    o_last[pi] = s.last;
    o_md[pi] = s.med_depth;
    o_mv[pi] = s.median >= 0 ? 1 : 0;
    o_unc[pi] = s.unc;
    if (LMODE != 2) {
      o_count[pi] = s.count;
      o_dom[pi] = s.dominant;
      o_domw[pi] = s.best;
    }
    o_med[pi] = s.median;
    if (LMODE == 0 && s.flag) fix_list[atomicAdd(fix_cnt, 1u)] = static_cast<uint32_t>(pi);
  }
  if (LMODE == 0) return;
  // fused loss epilogue: per-tile residual sums and mask counts (deterministic tree)
  double v[LS_NUM];
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) v[q] = 0.0;
  if (inside)
    loss_pixel<LMODE>(v, s.cr, s.cg, s.cb, s.ad, s.med_depth, s.median >= 0, s.op, s.unc, loss_rgb + 3 * pi, loss_depth, pi,
                      obs != nullptr, near_plane, far_plane, lp.opacity_floor);
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) {
    const double t = warp_sum_d(v[q]);
    if (lane == 0) s_red[warp][q] = t;
  }
  if (qstat && lane == 0) s_ws[warp] = wsteps;
  __syncthreads();
  if (tid < LS_NUM) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_red[w][tid];
    loss_part[static_cast<int64_t>(tile) * LS_NUM + tid] = t;
  }
  // quadrant q (8x8) = the 8x4 warp blocks q & 1 + 4 (q >> 1) and + 2
  if (qstat && tid >= 32 && tid < 36) {
    const int q = tid - 32, wa = (q & 1) + 4 * (q >> 1);
    qstat[tile * 4 + q] = make_int2(static_cast<int>(s_ws[wa] + s_ws[wa + 2]), rg.y - rg.x);
  }
  (void)fuse_final;
  (void)iteration;
  (void)ticket;
}

// Exact-decision fix-up of the render API (gsf_shared.cuh: pixel_flag_step / exact_*): one warp
// per flagged pixel re-blends its tile list in fp64 with the reference's formulas.  The lanes
// evaluate 32 entries' decisions and alphas at once (exact_alpha from the fp64 guard copies); lane
// 0 then accumulates them in list order (the reference's sequential rounding), and its results
// replace the pixel's fp32 ones.  ~1e-5..1e-3 of the pixels of a frame are flagged.
constexpr int kFixCtas = 296;
__global__ void __launch_bounds__(256) k_pixel_fixup(
    const uint32_t* __restrict__ fix_list, const uint32_t* fix_cnt, const int2* __restrict__ ranges,
    const uint32_t* __restrict__ sid, const BlendG* __restrict__ bg, const GuardG* __restrict__ gg,
    const float* __restrict__ obs, int W, int tiles_x, BlendConsts kc, double near_plane, double far_plane,
    float* __restrict__ o_color, float* __restrict__ o_ad, float* __restrict__ o_md, uint8_t* __restrict__ o_mv,
    float* __restrict__ o_op, float* __restrict__ o_unc, float* __restrict__ o_T, int32_t* __restrict__ o_count,
    int32_t* __restrict__ o_dom, int32_t* __restrict__ o_med, float* __restrict__ o_domw, int32_t* __restrict__ o_last,
    const DevState* ds) {
  __shared__ double s_a[8][32];
  __shared__ int32_t s_i[8][32];
  pdl_wait();
  pdl_trigger();
  if (ds->halt) return;
  const uint32_t n = *fix_cnt;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (uint32_t f = blockIdx.x * 8u + static_cast<uint32_t>(wib); f < n; f += gridDim.x * 8u) {
    const uint32_t pi = fix_list[f];
    const int x = static_cast<int>(pi % static_cast<uint32_t>(W)), y = static_cast<int>(pi / static_cast<uint32_t>(W));
    const int2 rg = ranges[(y / kTile) * tiles_x + x / kTile];
    const double px = static_cast<double>(static_cast<float>(x) + 0.5f), py = static_cast<double>(static_cast<float>(y) + 0.5f);
    bool obs_valid = false;
    double ov = 0.0;
    if (obs) {
      const float o = obs[pi];
      const double d = o;
      obs_valid = isfinite(d) && d > near_plane && d < far_plane;
      ov = d;
    }
    ExactPixel q;
    exact_init(q);
    for (int c = rg.x; c < rg.y; c += 32) {
      const int j = c + lane;
      double a = 0.0;
      int id = -1;
      if (j < rg.y) {
        id = static_cast<int>(sid[j]);
        if (!exact_alpha(px, py, gg[id], kc, &a)) id = -1;
      }
      s_a[wib][lane] = a;
      s_i[wib][lane] = id;
      __syncwarp();
      int done = 0;
      if (lane == 0) {
        const int cnt = min(32, rg.y - c);
        for (int k = 0; k < cnt && !q.done; ++k)
          if (s_i[wib][k] >= 0)
            exact_accumulate(q, s_a[wib][k], bg[s_i[wib][k]], s_i[wib][k], c + k - rg.x, obs_valid, ov, kc);
        done = q.done;
      }
      __syncwarp();
      if (__shfl_sync(0xffffffffu, done, 0)) break;
    }
    if (lane == 0) {
      o_color[3 * pi + 0] = static_cast<float>(q.cr);
      o_color[3 * pi + 1] = static_cast<float>(q.cg);
      o_color[3 * pi + 2] = static_cast<float>(q.cb);
      o_ad[pi] = static_cast<float>(q.ad);
      o_op[pi] = static_cast<float>(q.op);
      o_T[pi] = static_cast<float>(q.T);
      o_last[pi] = q.last;
      o_md[pi] = static_cast<float>(q.med_depth);
      o_mv[pi] = q.median >= 0 ? 1 : 0;
      o_unc[pi] = static_cast<float>(q.unc);
      o_count[pi] = q.count;
      o_dom[pi] = q.dominant;
      o_med[pi] = q.median;
      o_domw[pi] = static_cast<float>(q.best);
    }
  }
}

// Tracking forward (the tracking loss's maps and its fused loss) with two pixels per lane: warp w of the
// 128-thread CTA owns the 8x8 block (8 (w & 1), 8 (w >> 1)) of the tile and lane l the pixels
// (l & 7, l >> 3) and (l & 7, (l >> 3) + 4).  Both pixels share dx, so rho and exp run on packed
// FP32x2 and every per-entry cost (ballot walk, staging reads) is paid once for two pixels; an
// 8x8 block meets ~0.6x as many (block, entry) pairs as two 8x4 blocks.  Each packed lane rounds
// like the scalar op in the scalar order, and a pixel that does not take an entry sees alpha 0
// (w = 0, T * 1): the maps equal the plain render's, and the mirror's, bit for bit.
constexpr int kTrkThreads = 128;
constexpr int kTrkBatch = 256;

#ifndef GSF_TRK_MINB
#define GSF_TRK_MINB 8
#endif
// QM: 0 = each pixel's last contributor as a list index (o_last); 1 = the pose backward's
// per-quadrant work lists (qlist) and the last contributor as a work-list position (o_lastc);
// 2 = both.
template <int QM>
__global__ void __launch_bounds__(kTrkThreads, GSF_TRK_MINB) k_blend_track(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ sid, const BlendG* __restrict__ bg,
    const GuardG* __restrict__ gg, const float* __restrict__ loss_rgb, const float* __restrict__ loss_depth, int W, int H,
    int tiles_x, BlendConsts kc, double near_plane, double far_plane, LossParams lp, DevState* ds,
    float* __restrict__ o_color, float* __restrict__ o_ad, float* __restrict__ o_op, float* __restrict__ o_T,
    int32_t* __restrict__ o_last, double* __restrict__ loss_part, int fuse_final, int iteration, uint32_t* ticket,
    uint32_t* __restrict__ qlist, int32_t* __restrict__ o_lastc, uint8_t* __restrict__ o_code, uint32_t* clean_bins,
    int64_t clean_cnt_off,
    const uint32_t* __restrict__ order, int2* __restrict__ qstat) {
  __shared__ __align__(16) BlendG s_g[kTrkBatch];
  __shared__ int32_t s_id[kTrkBatch];
  __shared__ uint8_t s_mask[kTrkBatch];
  __shared__ double s_red[kTrkThreads / 32][LS_NUM];
  pdl_wait();
  pdl_trigger();
  if (clean_bins) {   // the binning is consumed: leave the bins zeroed for the next iteration (no memset)
    if (threadIdx.x < 4) clean_bins[static_cast<int64_t>(blockIdx.x) * kBinStride + threadIdx.x] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      clean_bins[static_cast<int64_t>(clean_cnt_off) + kCntVisible] = 0u;
      clean_bins[static_cast<int64_t>(clean_cnt_off) + kCntBig] = 0u;
      clean_bins[static_cast<int64_t>(clean_cnt_off) + kCntSortTicket] = 0u;
    }
  }
  if (ds->halt) return;
  // longest-first CTA order (k_lpt; order[0] = the tile count it was built for, else identity)
  const int tile = (order && order[0] == gridDim.x) ? static_cast<int>(order[1 + blockIdx.x]) : blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the tile's list: positions [lo, hi) of sid; this warp's work list at qbase of qlist
  const int2 rg = ranges[tile];
  const int lo = rg.x, hi = rg.y;
  const int64_t qbase = 4 * static_cast<int64_t>(lo) + static_cast<int64_t>(warp) * (hi - lo);
  const uint32_t sgb = opaque_smem_base(s_g);
  uint32_t wsteps = 0u;   // this warp's (warp, entry) steps: k_lpt's cost of the tile and of the
                          // quadrant's pose backward (which walks the same block mask)
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x = tx * kTile + 8 * (warp & 1) + (lane & 7);
  const int ya = ty * kTile + 8 * (warp >> 1) + (lane >> 3), yb = ya + 4;
  const bool in_a = x < W && ya < H, in_b = x < W && yb < H;
  float2 rg_a = make_float2(0.f, 0.f), bd_a = rg_a, rg_b = rg_a, bd_b = rg_a;
  // a pixel is done once T < term (T never grows); pixels outside the image start done (T = 0)
  float2 op = make_float2(0.f, 0.f), T = make_float2(in_a ? 1.f : 0.f, in_b ? 1.f : 0.f);
  int last_a = 0, last_b = 0;
  int lc_a = 0, lc_b = 0;   // the same, as positions in this warp's work list (qlist)
  float px = static_cast<float>(x) + 0.5f;
  float2 py = make_float2(static_cast<float>(ya) + 0.5f, static_cast<float>(yb) + 0.5f);
  const float tile_x0 = static_cast<float>(tx * kTile), tile_y0 = static_cast<float>(ty * kTile);
  for (int start = lo; start < hi; start += kTrkBatch) {
    if (__syncthreads_and(T.x < kc.term && T.y < kc.term)) break;
#pragma unroll
    for (int h = 0; h < kTrkBatch / kTrkThreads; ++h) {
      const int e = tid + h * kTrkThreads, j = start + e;
      if (j < hi) {
        const int id = static_cast<int>(sid[j]);
        const BlendG gj = bg[id];
        s_g[e] = gj;
        s_id[e] = id;
        const uint8_t mk = static_cast<uint8_t>(warp_block_mask8(gj, tile_x0, tile_y0, kc));
        s_mask[e] = mk;
      }
    }
    __syncthreads();
    const int cnt = min(kTrkBatch, hi - start);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      if (__all_sync(0xffffffffu, T.x < kc.term && T.y < kc.term)) break;
      const int kk = c0 + lane;
      uint32_t bits = __ballot_sync(0xffffffffu, kk < cnt && ((s_mask[kk] >> warp) & 1u));
      // the pose backward's work list: this block's entries in list order (its only staging input)
      if (QM != 0 && ((bits >> lane) & 1u))
        qlist[qbase + wsteps + static_cast<uint32_t>(__popc(bits & ((1u << lane) - 1u)))] = static_cast<uint32_t>(s_id[kk]);
      uint32_t ci = wsteps;
      wsteps += __popc(bits);
      while (bits) {
        const int k = c0 + __ffs(bits) - 1;
        bits &= bits - 1u;
        ++ci;
#ifndef GSF_NO_PIN_PX
        // keep the pixel centres in registers: at the 64-register cap ptxas otherwise re-forms
        // them with I2F + FADD (XU pipe) on every step
        asm volatile("" : "+f"(px), "+f"(py.x), "+f"(py.y));
#endif
        const BlendG g = lds_blend(sgb + 48u * k);
        const float dx = __fadd_rn(px, -g.mx);
        const float2 dy = __fadd2_rn(py, make_float2(-g.my, -g.my));
        const float2 rho = pair_rho2(dx, dy, g);
        const bool skip_a = T.x < kc.term || rho.x > g.rho_hi, skip_b = T.y < kc.term || rho.y > g.rho_hi;
        // warp-uniform control (4 us faster than per-lane branches here; the pose backward measured
        // the opposite): a lane whose pixels skip runs the step masked (alpha 0: w = 0, T * 1)
        if (__all_sync(0xffffffffu, skip_a && skip_b)) continue;
        const bool fast_a = rho.x < g.rho_fast, fast_b = rho.y < g.rho_fast;
        float2 al = __fmul2_rn(make_float2(g.sigma, g.sigma), exp_neg_half_inrange2(rho));
        bool ca = !skip_a && fast_a, cb = !skip_b && fast_b;
        if (__any_sync(0xffffffffu, (!skip_a && !fast_a) || (!skip_b && !fast_b))) {
        if (!skip_a && !fast_a) {   // guard band: eval_pair's full decision
          al.x = guard_decide(px, py.x, g, gg + s_id[k], &kc).alpha;
          ca = al.x >= 0.0f;
        }
        if (!skip_b && !fast_b) {
          al.y = guard_decide(px, py.y, g, gg + s_id[k], &kc).alpha;
          cb = al.y >= 0.0f;
        }
        }
        const float2 am = make_float2(ca ? al.x : 0.0f, cb ? al.y : 0.0f);
        const float2 w = __fmul2_rn(am, T);
        rg_a = __ffma2_rn(make_float2(w.x, w.x), make_float2(g.r, g.g), rg_a);
        bd_a = __ffma2_rn(make_float2(w.x, w.x), make_float2(g.b, g.depth), bd_a);
        rg_b = __ffma2_rn(make_float2(w.y, w.y), make_float2(g.r, g.g), rg_b);
        bd_b = __ffma2_rn(make_float2(w.y, w.y), make_float2(g.b, g.depth), bd_b);
        op = __fadd2_rn(op, w);
        T = __fmul2_rn(T, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-am.x, -am.y)));
        if (QM != 1) {
          const int li = start + k - lo + 1;
          if (ca) last_a = li;
          if (cb) last_b = li;
        }
        if (QM != 0) {
          if (ca) lc_a = static_cast<int>(ci);
          if (cb) lc_b = static_cast<int>(ci);
        }
      }
    }
  }
  if (qstat && lane == 0)
    qstat[tile * 4 + warp] = make_int2(static_cast<int>(wsteps), hi - lo);
  double v[LS_NUM], vb[LS_NUM];
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) v[q] = vb[q] = 0.0;
  if (in_a) {
    const int64_t pi = static_cast<int64_t>(ya) * W + x;
    if (o_color) {
      o_color[3 * pi + 0] = rg_a.x;
      o_color[3 * pi + 1] = rg_a.y;
      o_color[3 * pi + 2] = bd_a.x;
      o_ad[pi] = bd_a.y;
      o_op[pi] = op.x;
    }
    o_T[pi] = T.x;
    if (QM != 1) o_last[pi] = last_a;
    if (QM != 0) o_lastc[pi] = lc_a;
    const float* Ia = loss_rgb + 3 * pi;
    const float* Dl = loss_depth;
    const int64_t da = pi;
    if (loss_rgb)
      loss_pixel<1>(v, rg_a.x, rg_a.y, bd_a.x, bd_a.y, 0.0f, false, op.x, 0.0f, Ia, Dl, da, false,
                    near_plane, far_plane, lp.opacity_floor);
    if (o_code)
      o_code[pi] = pixel_seed_code(rg_a.x, rg_a.y, bd_a.x, bd_a.y, op.x, Ia, Dl, da, near_plane,
                                   far_plane, lp.opacity_floor);
  }
  if (in_b) {
    const int64_t pi = static_cast<int64_t>(yb) * W + x;
    if (o_color) {
      o_color[3 * pi + 0] = rg_b.x;
      o_color[3 * pi + 1] = rg_b.y;
      o_color[3 * pi + 2] = bd_b.x;
      o_ad[pi] = bd_b.y;
      o_op[pi] = op.y;
    }
    o_T[pi] = T.y;
    if (QM != 1) o_last[pi] = last_b;
    if (QM != 0) o_lastc[pi] = lc_b;
    const float* Ib = loss_rgb + 3 * pi;
    const float* Dl = loss_depth;
    const int64_t db = pi;
    if (loss_rgb)
      loss_pixel<1>(vb, rg_b.x, rg_b.y, bd_b.x, bd_b.y, 0.0f, false, op.y, 0.0f, Ib, Dl, db, false,
                    near_plane, far_plane, lp.opacity_floor);
    if (o_code)
      o_code[pi] = pixel_seed_code(rg_b.x, rg_b.y, bd_b.x, bd_b.y, op.y, Ib, Dl, db, near_plane,
                                   far_plane, lp.opacity_floor);
  }
  if (!loss_rgb) return;
  // the tracking loss has two residual sums and two mask counts (losses.cpp:284-339); the counts
  // are ballots (exact in fp64), the align / var slots of the mapping loss stay zero
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) {
    double t = 0.0;
    if (q == LS_COLOR_SUM || q == LS_GEO_SUM)
      t = warp_sum_d(v[q] + vb[q]);
    else if (q == LS_COLOR_CNT || q == LS_GEO_CNT)
      t = static_cast<double>(__popc(__ballot_sync(0xffffffffu, v[q] != 0.0)) +
                              __popc(__ballot_sync(0xffffffffu, vb[q] != 0.0)));
    if (lane == 0) s_red[warp][q] = t;
  }
  __syncthreads();
  if (tid < LS_NUM) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kTrkThreads / 32; ++w) t += s_red[w][tid];
    loss_part[static_cast<int64_t>(tile) * LS_NUM + tid] = t;
  }
  if (fuse_final) {
    __shared__ int s_last;
    __shared__ double s_tot[LS_NUM];
    if (last_cta(ticket, &s_last, tid < LS_NUM)) {
      block_reduce_rows<LS_NUM, kTrkThreads>(loss_part, gridDim.x, s_tot, s_red);
      if (tid == 0) loss_scalars(ds, lp, s_tot, 0.0, 0.0, static_cast<int64_t>(W) * H, iteration);
    }
  }
}

// Mapping forward (blend_pixel, rasterizer.cpp:96-140, with the mapping loss's partials,
// losses.cpp:156-282) as independent single-warp CTAs: CTA 4 t + q owns quadrant q (8x8 pixels,
// two per lane, the layout of k_blend_track) of tile t and walks the tile list front to back in
// chunks of 32 entries: lane e stages entry e of the chunk (record by cp.async, id two chunks
// ahead), tests it against the quadrant's block (block_hit8) and the warp walks the set bits with
// the forward's exact decision path.  No CTA barriers; the quadrant's loss partials are one row
// of loss_part (4 rows per tile) and its (warp, entry) steps the backward's LPT cost (qstat).
// Per pixel the state updates run in pixel_accumulate's operation order (packed FP32x2 rounds like
// the scalar op), so the maps equal k_blend<2>'s.
#ifndef GSF_FQ_MINB
#define GSF_FQ_MINB 24
#endif
__global__ void __launch_bounds__(32, GSF_FQ_MINB) k_blend_mq(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ sid, const BlendG* __restrict__ bg,
    const GuardG* __restrict__ gg, const float* __restrict__ obs, const float* __restrict__ loss_rgb,
    const float* __restrict__ loss_depth, int W, int H, int tiles_x, BlendConsts kc, double near_plane,
    double far_plane, LossParams lp, DevState* ds, float* __restrict__ o_color, float* __restrict__ o_ad,
    float* __restrict__ o_md, uint8_t* __restrict__ o_mv, float* __restrict__ o_op, float* __restrict__ o_unc,
    float* __restrict__ o_T, int32_t* __restrict__ o_med, int32_t* __restrict__ o_last, double* __restrict__ loss_part,
    int2* __restrict__ qstat) {
  __shared__ float4 s_buf[2 * 3 * 32 + 16];   // two buffers of 32 records (1536 B) + their ids (128 B) at 3072 + 128 b
  pdl_wait();
  pdl_trigger();
  if (ds->halt) return;
  const int lane = threadIdx.x;
  const uint32_t sb = opaque_smem_base(s_buf);
  const int item = static_cast<int>(blockIdx.x);
  const int tile = item >> 2, qd = item & 3;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int bx0 = tx * kTile + 8 * (qd & 1), by0 = ty * kTile + 8 * (qd >> 1);
  const int x = bx0 + (lane & 7);
  const int ya = by0 + (lane >> 3), yb = ya + 4;
  const bool in_a = x < W && ya < H, in_b = x < W && yb < H;
  const int64_t pa = static_cast<int64_t>(ya) * W + x, pb = static_cast<int64_t>(yb) * W + x;
  const int2 rg = ranges[tile];
  float2 rg_a = make_float2(0.f, 0.f), bd_a = rg_a, rg_b = rg_a, bd_b = rg_a;
  float2 op = make_float2(0.f, 0.f), unc = make_float2(0.f, 0.f);
  float2 T = make_float2(in_a ? 1.f : 0.f, in_b ? 1.f : 0.f);   // outside the image: done from the start
  int last_a = 0, last_b = 0, med_a = -1, med_b = -1;
  float md_a = 0.0f, md_b = 0.0f;
  bool ov_a = false, ov_b = false;
  float obs_a = 0.0f, obs_b = 0.0f;
  if (obs) {
    if (in_a) { obs_a = obs[pa]; ov_a = depth_valid(obs_a, near_plane, far_plane); }
    if (in_b) { obs_b = obs[pb]; ov_b = depth_valid(obs_b, near_plane, far_plane); }
  }
  const float px = static_cast<float>(x) + 0.5f;
  const float2 py = make_float2(static_cast<float>(ya) + 0.5f, static_cast<float>(yb) + 0.5f);
  const float qx0 = static_cast<float>(bx0), qy0 = static_cast<float>(by0);
  const int len = rg.y - rg.x;
  const int nch = (len + 31) / 32;
  auto fetch = [&](int c) -> int32_t {
    const int j = rg.x + 32 * c + lane;
    return (c < nch && j < rg.y) ? static_cast<int32_t>(__ldg(sid + j)) : -1;
  };
  auto issue = [&](int c, int32_t id) {
    if (c < nch && id >= 0) {
      const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 1536u;
      const float4* rec = reinterpret_cast<const float4*>(bg + id);
      cp_async16_to(buf + 48u * lane, rec);
      cp_async16_to(buf + 48u * lane + 16u, rec + 1);
      cp_async16_to(buf + 48u * lane + 32u, rec + 2);
      sts_s32(sb + 3072u + static_cast<uint32_t>(c & 1) * 128u + 4u * lane, id);
    }
    cp_async_commit();
  };
  uint32_t steps = 0u;
  int32_t id0 = fetch(0), id1 = fetch(1);
  issue(0, id0);
  for (int c = 0; c < nch; ++c) {
    if (__all_sync(0xffffffffu, T.x < kc.term && T.y < kc.term)) break;
    issue(c + 1, id1);
    const int32_t id2 = fetch(c + 2);
    cp_async_wait_1();
    __syncwarp();
    const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 1536u, idb = sb + 3072u + static_cast<uint32_t>(c & 1) * 128u;
    bool hit = false;
    if (id0 >= 0) hit = block_hit8(lds_blend(buf + 48u * lane), qx0, qy0, kc);
    uint32_t bits = __ballot_sync(0xffffffffu, hit);
    steps += __popc(bits);
    while (bits) {
      const int e = __ffs(bits) - 1;   // lowest lane = earliest entry: front to back
      bits &= bits - 1u;
      const BlendG g = lds_blend(buf + 48u * e);
      const float dx = __fadd_rn(px, -g.mx);
      const float2 dy = __fadd2_rn(py, make_float2(-g.my, -g.my));
      const float2 rho = pair_rho2(dx, dy, g);
      const bool skip_a = T.x < kc.term || rho.x > g.rho_hi, skip_b = T.y < kc.term || rho.y > g.rho_hi;
      if (__all_sync(0xffffffffu, skip_a && skip_b)) continue;
      const bool fast_a = rho.x < g.rho_fast, fast_b = rho.y < g.rho_fast;
      float2 al = __fmul2_rn(make_float2(g.sigma, g.sigma), exp_neg_half_inrange2(rho));
      bool ca = !skip_a && fast_a, cb = !skip_b && fast_b;
      const int32_t eid = lds_s32(idb + 4u * e);
      if (__any_sync(0xffffffffu, (!skip_a && !fast_a) || (!skip_b && !fast_b))) {
        if (!skip_a && !fast_a) {
          al.x = guard_decide(px, py.x, g, gg + eid, &kc).alpha;
          ca = al.x >= 0.0f;
        }
        if (!skip_b && !fast_b) {
          al.y = guard_decide(px, py.y, g, gg + eid, &kc).alpha;
          cb = al.y >= 0.0f;
        }
      }
      const float2 am = make_float2(ca ? al.x : 0.0f, cb ? al.y : 0.0f);
      const float2 w = __fmul2_rn(am, T);
      rg_a = __ffma2_rn(make_float2(w.x, w.x), make_float2(g.r, g.g), rg_a);
      bd_a = __ffma2_rn(make_float2(w.x, w.x), make_float2(g.b, g.depth), bd_a);
      rg_b = __ffma2_rn(make_float2(w.y, w.y), make_float2(g.r, g.g), rg_b);
      bd_b = __ffma2_rn(make_float2(w.y, w.y), make_float2(g.b, g.depth), bd_b);
      op = __fadd2_rn(op, w);
      if (ca && ov_a) { const float d = __fadd_rn(g.depth, -obs_a); unc.x = __fmaf_rn(__fmul_rn(w.x, d), d, unc.x); }
      if (cb && ov_b) { const float d = __fadd_rn(g.depth, -obs_b); unc.y = __fmaf_rn(__fmul_rn(w.y, d), d, unc.y); }
      const float2 tn = __fmul2_rn(T, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-am.x, -am.y)));
      if (ca && med_a < 0 && T.x >= 0.5f && tn.x < 0.5f) { med_a = eid; md_a = g.depth; }
      if (cb && med_b < 0 && T.y >= 0.5f && tn.y < 0.5f) { med_b = eid; md_b = g.depth; }
      T = tn;
      const int li = 32 * c + e + 1;
      if (ca) last_a = li;
      if (cb) last_b = li;
    }
    __syncwarp();   // buffer c & 1 is refilled by issue(c + 2)
    id0 = id1;
    id1 = id2;
  }
  cp_async_wait_all();
  if (qstat && lane == 0) qstat[item] = make_int2(static_cast<int>(steps), len);
  double v[LS_NUM], vb[LS_NUM];
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) v[q] = vb[q] = 0.0;
  const bool has_unc = obs != nullptr;
  if (in_a) {
    o_color[3 * pa + 0] = rg_a.x; o_color[3 * pa + 1] = rg_a.y; o_color[3 * pa + 2] = bd_a.x;
    o_ad[pa] = bd_a.y; o_op[pa] = op.x; o_T[pa] = T.x; o_last[pa] = last_a;
    o_md[pa] = md_a; o_mv[pa] = med_a >= 0 ? 1 : 0; o_unc[pa] = unc.x; o_med[pa] = med_a;
    if (loss_rgb)
      loss_pixel<2>(v, rg_a.x, rg_a.y, bd_a.x, bd_a.y, md_a, med_a >= 0, op.x, unc.x, loss_rgb + 3 * pa, loss_depth, pa,
                    has_unc, near_plane, far_plane, lp.opacity_floor);
  }
  if (in_b) {
    o_color[3 * pb + 0] = rg_b.x; o_color[3 * pb + 1] = rg_b.y; o_color[3 * pb + 2] = bd_b.x;
    o_ad[pb] = bd_b.y; o_op[pb] = op.y; o_T[pb] = T.y; o_last[pb] = last_b;
    o_md[pb] = md_b; o_mv[pb] = med_b >= 0 ? 1 : 0; o_unc[pb] = unc.y; o_med[pb] = med_b;
    if (loss_rgb)
      loss_pixel<2>(vb, rg_b.x, rg_b.y, bd_b.x, bd_b.y, md_b, med_b >= 0, op.y, unc.y, loss_rgb + 3 * pb, loss_depth, pb,
                    has_unc, near_plane, far_plane, lp.opacity_floor);
  }
  if (!loss_rgb) return;
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) {
    const double t = warp_sum_d(v[q] + vb[q]);
    if (lane == 0) loss_part[static_cast<int64_t>(item) * LS_NUM + q] = t;
  }
}

// Stand-alone loss partials over stored maps (evaluate_*_loss called on a RenderResult).
template <int LMODE>
__global__ void __launch_bounds__(256) k_loss_tiles(const float* __restrict__ color, const float* __restrict__ ad,
                                                    const float* __restrict__ md, const uint8_t* __restrict__ mv,
                                                    const float* __restrict__ op, const float* __restrict__ unc,
                                                    const float* __restrict__ rgb, const float* __restrict__ depth, int W,
                                                    int H, int tiles_x, bool has_unc, double near_plane, double far_plane,
                                                    float floor, double* __restrict__ loss_part) {
  __shared__ double s_red[8][LS_NUM];
  const int tile = blockIdx.x, tid = threadIdx.x;
  const int x = (tile % tiles_x) * kTile + tile_lx(tid), y = (tile / tiles_x) * kTile + tile_ly(tid);
  double v[LS_NUM];
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) v[q] = 0.0;
  if (x < W && y < H) {
    const int64_t pi = static_cast<int64_t>(y) * W + x;
    loss_pixel<LMODE>(v, color[3 * pi], color[3 * pi + 1], color[3 * pi + 2], ad[pi], md[pi], mv[pi] != 0, op[pi], unc[pi],
                      rgb + 3 * pi, depth, pi, has_unc, near_plane, far_plane, floor);
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int q = 0; q < LS_NUM; ++q) {
    const double t = warp_sum_d(v[q]);
    if (lane == 0) s_red[warp][q] = t;
  }
  __syncthreads();
  if (tid < LS_NUM) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_red[w][tid];
    loss_part[static_cast<int64_t>(tile) * LS_NUM + tid] = t;
  }
}

}  // namespace

void run_forward(Workspace& ws, DevState* ds, const FwdArgs& a, cudaStream_t st, int64_t* L) {
  const int64_t P = a.P;
  const int tiles_x = a.rp.tiles_x, tiles_y = a.rp.tiles_y;
  const int ntiles = tiles_x * tiles_y;
  Profiler* pf = ws.prof;
  if (!a.bins_clean)
    GSF_CUDA_CHECK(cudaMemsetAsync(ws.bins, 0, sizeof(uint32_t) * (ws.tiles_cap * kBinStride + kCntNum), st));
  if (pf) pf->begin(PROF_PREPROCESS, st);
  if (P > 0) {
#define GSF_PRE(CV)                                                                                                    \
  launch_pdl(k_preprocess<CV>, dim3(div_up(P, 256)), dim3(256), 0, st, a.params, P, ds, a.rp, ws.bg_id, ws.gg_id,       \
             ws.depth_id, ws.rect_id,                                                                                  \
                                                   ws.visible, &ds->bad_index, a.kc, ws.bin_counters,                    \
                                                   ws.vis_list, ws.pj_slot, ws.tile_fill,                                 \
                                                   static_cast<uint32_t>(ws.bucket_cap), ws.bucket, ws.big_ids,           \
                                                   a.want_pair_base ? ws.pair_base : nullptr, ws.world, ws.support,        \
                                                   a.cand)
    if (a.use_world) GSF_PRE(true); else GSF_PRE(false);
#undef GSF_PRE
    ++*L;
  }
  if (pf) pf->end(st);
  // the pose Jacobians (and the slot-indexed records) only depend on k_preprocess: a side branch
  // beside the binning, joined before the blend (captured graphs keep the fork/join)
  const bool side = P > 0 && a.want_posejac;
  if (side) {
    GSF_CUDA_CHECK(cudaEventRecord(ws.ev_fork, st));
    GSF_CUDA_CHECK(cudaStreamWaitEvent(ws.side, ws.ev_fork, 0));
    if (pf) pf->begin(PROF_POSEJAC, ws.side);
    k_posejac<<<div_up(P, kPjThreads), kPjThreads, 0, ws.side>>>(a.params, P, ds, a.K, ws.vis_list, ws.bin_counters,
                                                     a.use_world ? ws.world : nullptr, ws.pj_id, ws.bg_id, ws.gg_id,
                                                     ws.bg_slot, ws.gg_slot);
    ++*L;
    if (pf) pf->end(ws.side);
    GSF_CUDA_CHECK(cudaEventRecord(ws.ev_join, ws.side));
  }
  // tracking loop (two-pixel pose backward): the sort runs inside the blend (k_blend_track<1, true>)
  // the tracking loop's and the mapping forward's lists are only read back through `ranges` (never
  // exported): k_tile_sort places each with one atomic instead of the ordered look-back scan
#ifdef GSF_NO_ANY_ORDER
  const bool any_order = false;
#else
  const bool any_order = a.loss_rgb && ((a.lp.mode == 1 && a.want_posejac && a.qmode == 1 && a.fuse_loss_final &&
                                         a.clean_bins) || a.lp.mode == 2);
#endif
  if (pf) pf->begin(PROF_SORT, st);
  run_binning(ws, ds, P, tiles_x, ntiles, st, L, a.want_posejac, any_order);
  if (pf) pf->end(st);
  if (side) GSF_CUDA_CHECK(cudaStreamWaitEvent(st, ws.ev_join, 0));
  const float* loss_rgb = a.loss_rgb;
#define GSF_BLEND_ARGS                                                                                                 \
  ws.ranges, ws.sid, ws.bg_id, ws.gg_id, a.obs, loss_rgb, a.loss_depth, a.W, a.H,                                     \
      tiles_x, a.kc, a.near_plane, a.far_plane, a.lp, ds, ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid, \
      ws.opacity, ws.uncertainty, ws.final_T, ws.count, ws.dominant, ws.median_prim, ws.dominant_w, ws.last, ws.loss_part, \
      a.fuse_loss_final ? 1 : 0, a.iteration, ws.bin_counters + kCntBlendTicket, ws.fix_list, ws.bin_counters + kCntFixup, \
      a.lp.mode == 2 ? ws.qstat : nullptr
  if (pf) pf->begin(PROF_BLEND, st);
  ws.loss_rows = ntiles;
  if (a.lp.mode == 1 && loss_rgb) {   // tracking loss: colour, alpha depth, opacity, T, last; two pixels per lane
    // with pose Jacobians (a pose backward follows) the lists and records are read by visible slot
    // and the entries' block masks are kept for the backward
    const bool sl = a.want_posejac;
    if (a.join_order) GSF_CUDA_CHECK(cudaStreamWaitEvent(st, ws.ev_ljoin, 0));
    const int qm = sl ? a.qmode : 0;
#define GSF_BLEND_TRACK(QMV)                                                                                           \
    launch_pdl(k_blend_track<QMV>, dim3(ntiles), dim3(kTrkThreads), 0, st, ws.ranges, sl ? ws.sslot : ws.sid,          \
               sl ? ws.bg_slot : ws.bg_id, sl ? ws.gg_slot : ws.gg_id, loss_rgb, a.loss_depth, a.W, a.H, tiles_x, a.kc, \
               a.near_plane, a.far_plane, a.lp, ds, a.keep_maps ? ws.color : nullptr, ws.alpha_depth, ws.opacity,       \
               ws.final_T, ws.last, ws.loss_part, a.fuse_loss_final ? 1 : 0, a.iteration,                              \
               ws.bin_counters + kCntBlendTicket, ws.qlist, ws.lastc, sl ? ws.pxcode : nullptr,                        \
               a.clean_bins ? ws.bins : nullptr, static_cast<int64_t>(ws.tiles_cap) * kBinStride, a.order,               \
               sl ? ws.qstat : nullptr)
    if (qm == 1) GSF_BLEND_TRACK(1);
    else if (qm == 2) GSF_BLEND_TRACK(2);
    else GSF_BLEND_TRACK(0);
#undef GSF_BLEND_TRACK
  }
  else if (a.lp.mode == 2 && loss_rgb) {
#ifdef GSF_MAP_FWD8
    launch_pdl(k_blend<2>, dim3(ntiles), dim3(256), 0, st, GSF_BLEND_ARGS);
#else
    // the mapping forward as per-quadrant single-warp CTAs, one loss row per quadrant
    ws.loss_rows = 4 * ntiles;
    launch_pdl(k_blend_mq, dim3(4 * ntiles), dim3(32), 0, st, ws.ranges, ws.sid, ws.bg_id, ws.gg_id, a.obs, loss_rgb,
               a.loss_depth, a.W, a.H, tiles_x, a.kc, a.near_plane, a.far_plane, a.lp, ds, ws.color, ws.alpha_depth,
               ws.median_depth, ws.median_valid, ws.opacity, ws.uncertainty, ws.final_T, ws.median_prim, ws.last,
               ws.loss_part, ws.qstat);
#endif
  }
  else {
    launch_pdl(k_blend<0>, dim3(ntiles), dim3(256), 0, st, GSF_BLEND_ARGS);
    ++*L;
    // the render API's exact discrete decisions: flagged pixels re-blended in fp64
    launch_pdl(k_pixel_fixup, dim3(kFixCtas), dim3(256), 0, st, ws.fix_list, ws.bin_counters + kCntFixup, ws.ranges, ws.sid,
               ws.bg_id, ws.gg_id, a.obs, a.W, tiles_x, a.kc, a.near_plane, a.far_plane, ws.color, ws.alpha_depth,
               ws.median_depth, ws.median_valid, ws.opacity, ws.uncertainty, ws.final_T, ws.count, ws.dominant,
               ws.median_prim, ws.dominant_w, ws.last, ds);
  }
#undef GSF_BLEND_ARGS
  ++*L;
  if (pf) pf->end(st);
  (void)tiles_y;
}

// Longest-first CTA orders for the tracking loop's tile kernels.  The hardware hands CTAs to SMs
// roughly in blockIdx order, so a grid whose long tiles come last ends with a few SMs finishing
// them while the rest idle (ncu: the average SM active 83-86 % of the kernel).  From the previous
// iteration's per-(tile, quadrant) counts (the lists change little between iterations) one CTA
// counting-sorts the tiles by their longest warp walk plus a quarter of the list length (the
// staging) and the (tile, quadrant) items by their walk (the pose backward walks the same block
// masks), longest first.  Measured per-CTA cycles as the cost (clock64) and a refined mask of
// only the entries a block took were both slower: the bookkeeping costs more than it balances.
// Only the dispatch order changes: every CTA still writes its tile's rows, and the reductions over them run in tile order.
constexpr int kLptThreads = 1024, kLptBuckets = 2048;
__global__ void __launch_bounds__(kLptThreads) k_lpt(const int2* __restrict__ qstat, int ntiles, uint32_t* __restrict__ out,
                                                    int64_t tiles_cap) {
  __shared__ uint32_t hist[kLptBuckets];
  __shared__ uint32_t s_wsum[kLptThreads / 32];
  __shared__ uint32_t s_max;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    const int n = pass == 0 ? ntiles : 4 * ntiles;
    uint32_t* ord = out + 1 + (pass == 0 ? 0 : tiles_cap);
    auto key = [&](int i) -> uint32_t {
      if (pass == 0) {   // a tile CTA: its 4 warps walk concurrently after staging the list
        const int2 a = qstat[4 * i], b = qstat[4 * i + 1], c = qstat[4 * i + 2], d = qstat[4 * i + 3];
        return static_cast<uint32_t>(max(max(a.x, b.x), max(max(c.x, d.x), 0)) + max(a.y, 0) / 4);
      }
      return static_cast<uint32_t>(max(qstat[i].x, 0));
    };
    for (int b = tid; b < kLptBuckets; b += kLptThreads) hist[b] = 0u;
    if (tid == 0) s_max = 1u;
    __syncthreads();
    uint32_t m = 0u;
    for (int i = tid; i < n; i += kLptThreads) m = max(m, key(i));
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) atomicMax(&s_max, m);
    __syncthreads();
    const uint64_t mx = s_max;
    // bucket kLptBuckets-1-q for quantised cost q: ascending bucket index = descending cost
    auto bucket = [&](uint32_t k) {
      return kLptBuckets - 1 - static_cast<int>((static_cast<uint64_t>(k) * (kLptBuckets - 1)) / mx);
    };
    for (int i = tid; i < n; i += kLptThreads) atomicAdd(&hist[bucket(key(i))], 1u);
    __syncthreads();
    // exclusive scan of the 2048 buckets, two per thread
    const uint32_t h0 = hist[2 * tid], h1 = hist[2 * tid + 1];
    uint32_t incl = h0 + h1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_wsum[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      s_wsum[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t base = s_wsum[warp] + incl - (h0 + h1);
    hist[2 * tid] = base;
    hist[2 * tid + 1] = base + h0;
    __syncthreads();
    for (int i = tid; i < n; i += kLptThreads) ord[atomicAdd(&hist[bucket(key(i))], 1u)] = static_cast<uint32_t>(i);
    __syncthreads();
  }
  if (tid == 0) out[0] = static_cast<uint32_t>(ntiles);
}

void run_lpt(Workspace& ws, int ntiles, uint32_t* out, cudaStream_t st, int64_t* L) {
  k_lpt<<<1, kLptThreads, 0, st>>>(ws.qstat, ntiles, out, ws.tiles_cap);
  ++*L;
}

void run_world(Workspace& ws, DevState* ds, const float* params, int64_t P, const RasterParams& rp, cudaStream_t st,
               int64_t* L) {
  if (P <= 0) return;
  k_world<<<div_up(P, 256), 256, 0, st>>>(params, P, rp, ws.world, ws.support, &ds->bad_index, &ds->ncand);
  ++*L;
}

void run_candidates(Workspace& ws, DevState* ds, const float* params, int64_t P, const RasterParams& rp,
                    double theta_max, double dist_max, cudaStream_t st, int64_t* L) {
  if (P <= 0) return;
  k_candidates<<<div_up(P, 256), 256, 0, st>>>(P, ds, rp, params, ws.support, theta_max, dist_max, ws.cand);
  ++*L;
}

void run_loss_tiles(Workspace& ws, int mode, const float* rgb, const float* depth, bool has_unc, int W, int H,
                    double near_plane, double far_plane, float floor, cudaStream_t st, int64_t* L) {
  const int tiles_x = (W + kTile - 1) / kTile, tiles_y = (H + kTile - 1) / kTile;
  ws.loss_rows = tiles_x * tiles_y;
  if (mode == 1)
    k_loss_tiles<1><<<tiles_x * tiles_y, 256, 0, st>>>(ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid, ws.opacity,
                                                        ws.uncertainty, rgb, depth, W, H, tiles_x, has_unc, near_plane,
                                                        far_plane, floor, ws.loss_part);
  else
    k_loss_tiles<2><<<tiles_x * tiles_y, 256, 0, st>>>(ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid, ws.opacity,
                                                        ws.uncertainty, rgb, depth, W, H, tiles_x, has_unc, near_plane,
                                                        far_plane, floor, ws.loss_part);
  ++*L;
}

}  // namespace gsfk
