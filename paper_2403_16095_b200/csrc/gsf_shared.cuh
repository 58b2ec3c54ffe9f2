// gsf_shared.cuh — the decision-path arithmetic shared by the sm_100a kernels and the CPU
// mirror (oracle/mirror.cpp).  Everything here is __host__ __device__ and written with
// explicitly-rounded operations, so the device (which would otherwise contract a*b+c into
// FFMA) and the host (compiled with -ffp-contract=off) produce identical bits.  That is what
// makes tile keys, depth order, tile ranges, per-pixel contributor counts and ids bit-exact
// between the GPU and the mirror.
//
// Reference semantics restated here:
//   project_gaussian      projection.cpp:54-104 (+ axis_bounds :40-50, jacobian :26-33)
//   project_all           rasterizer.cpp:46-67 (support radius, sigmoid, SH colour)
//   eval_sh_color         sh.cpp:79-86, bases :21-42
//   tile rectangle        rasterizer.cpp:199-208
//   blend_pixel           rasterizer.cpp:96-140
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>
#if !defined(__CUDACC__)
#include <cmath>
#endif

#if defined(__CUDACC__)
#define GSF_HD __host__ __device__ __forceinline__
#else
#define GSF_HD inline
#endif

namespace gsfk {

// ---------------------------------------------------------------------------------------
// Explicitly rounded arithmetic.
// ---------------------------------------------------------------------------------------
#if defined(__CUDA_ARCH__)
GSF_HD float fmul(float a, float b) { return __fmul_rn(a, b); }
GSF_HD float fadd(float a, float b) { return __fadd_rn(a, b); }
GSF_HD float fsub(float a, float b) { return __fsub_rn(a, b); }
GSF_HD float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
GSF_HD float fdiv(float a, float b) { return __fdiv_rn(a, b); }
GSF_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
GSF_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
GSF_HD double dsub(double a, double b) { return __dsub_rn(a, b); }
GSF_HD double ddiv(double a, double b) { return __ddiv_rn(a, b); }
GSF_HD double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
GSF_HD double dsqrt(double a) { return __dsqrt_rn(a); }
GSF_HD double drint(double a) { return rint(a); }
GSF_HD float frint(float a) { return rintf(a); }
GSF_HD int64_t dbits(double a) { return __double_as_longlong(a); }
GSF_HD double bitsd(int64_t a) { return __longlong_as_double(a); }
GSF_HD int32_t fbits(float a) { return __float_as_int(a); }
GSF_HD float bitsf(int32_t a) { return __int_as_float(a); }
#else
GSF_HD float fmul(float a, float b) { return a * b; }
GSF_HD float fadd(float a, float b) { return a + b; }
GSF_HD float fsub(float a, float b) { return a - b; }
GSF_HD float ffma(float a, float b, float c) { return fmaf(a, b, c); }
GSF_HD float fdiv(float a, float b) { return a / b; }
GSF_HD double dmul(double a, double b) { return a * b; }
GSF_HD double dadd(double a, double b) { return a + b; }
GSF_HD double dsub(double a, double b) { return a - b; }
GSF_HD double ddiv(double a, double b) { return a / b; }
GSF_HD double dfma(double a, double b, double c) { return fma(a, b, c); }
GSF_HD double dsqrt(double a) { return sqrt(a); }
GSF_HD double drint(double a) { return rint(a); }
GSF_HD float frint(float a) { return rintf(a); }
GSF_HD int64_t dbits(double a) { int64_t r; memcpy(&r, &a, 8); return r; }
GSF_HD double bitsd(int64_t a) { double r; memcpy(&r, &a, 8); return r; }
GSF_HD int32_t fbits(float a) { int32_t r; memcpy(&r, &a, 4); return r; }
GSF_HD float bitsf(int32_t a) { float r; memcpy(&r, &a, 4); return r; }
#endif

#if defined(__CUDA_ARCH__)
GSF_HD bool disfinite(double a) { return isfinite(a); }
#else
GSF_HD bool disfinite(double a) { return std::isfinite(a); }
#endif
GSF_HD double dinf() { return bitsd(0x7ff0000000000000LL); }
GSF_HD float finf() { return bitsf(0x7f800000); }

GSF_HD double dmax(double a, double b) { return a > b ? a : b; }
GSF_HD double dmin(double a, double b) { return a < b ? a : b; }
GSF_HD float fminf_(float a, float b) { return a < b ? a : b; }

// Deterministic exp (fp64): Cody-Waite reduction by ln2 then a degree-13 Taylor polynomial
// on |r| <= 0.35, all in fused multiply-adds.  < 1 ulp from glibc on the ranges used here.
GSF_HD double exp_d(double x) {
  if (!(x == x)) return x;
  if (x > 709.78) return dinf();
  if (x < -745.2) return 0.0;
  const double n = drint(dmul(x, 1.4426950408889634));
  double r = dfma(n, -6.93147180369123816490e-01, x);
  r = dfma(n, -1.90821492927058770002e-10, r);
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = dfma(p, r, 1.0 / 479001600.0);
  p = dfma(p, r, 1.0 / 39916800.0);
  p = dfma(p, r, 1.0 / 3628800.0);
  p = dfma(p, r, 1.0 / 362880.0);
  p = dfma(p, r, 1.0 / 40320.0);
  p = dfma(p, r, 1.0 / 5040.0);
  p = dfma(p, r, 1.0 / 720.0);
  p = dfma(p, r, 1.0 / 120.0);
  p = dfma(p, r, 1.0 / 24.0);
  p = dfma(p, r, 1.0 / 6.0);
  p = dfma(p, r, 0.5);
  p = dfma(p, r, 1.0);
  p = dfma(p, r, 1.0);
  int ni = static_cast<int>(n);
  // scale by 2^n in two steps so subnormal results stay exact enough
  if (ni < -1000) {
    p = dmul(p, bitsd(static_cast<int64_t>(1023 - 1000) << 52));
    ni += 1000;
  }
  if (ni > 1000) {
    p = dmul(p, bitsd(static_cast<int64_t>(1023 + 1000) << 52));
    ni -= 1000;
  }
  return dmul(p, bitsd(static_cast<int64_t>(1023 + ni) << 52));
}

// Deterministic exp(-rho/2) (fp32) for the blend, rho >= -tiny: 2^y with y = rho * (-log2(e)/2)
// split as y = n + f, |f| <= 1/2, and 2^f by its degree-6 Taylor polynomial in Horner form.
// |relative error| < 3e-7 (truncation 1.2e-7 + roundings), far inside the 5e-4 alpha guard band;
// 12 instructions.  The in-range form skips the underflow test (fast path: rho < cutoff < 170).
GSF_HD float exp_neg_half_inrange(float rho) {
  const float y = fmul(rho, -0.72134752044448170368f);
  const float n = frint(y);
  const float f = fsub(y, n);
  float p = 1.5403530393381606e-4f;
  p = ffma(p, f, 1.3333558146428443e-3f);
  p = ffma(p, f, 9.6181291076284772e-3f);
  p = ffma(p, f, 5.5504108664821580e-2f);
  p = ffma(p, f, 2.4022650695910071e-1f);
  p = ffma(p, f, 6.9314718055994531e-1f);
  p = ffma(p, f, 1.0f);
  return fmul(p, bitsf((127 + static_cast<int>(n)) << 23));
}
GSF_HD float exp_neg_half(float rho) {
  if (fmul(rho, -0.72134752044448170368f) < -126.0f) return 0.0f;   // 2^n must stay normal
  return exp_neg_half_inrange(rho);
}

// ---------------------------------------------------------------------------------------
// Camera (fp64).  W is row-major world->camera rotation exp(rotation_tangent).
// ---------------------------------------------------------------------------------------
struct Cam {
  double W[9];
  double t[3];
  double center[3];   // -W^T t
  double fx, fy, cx, cy;
  double near_plane, far_plane;
  int32_t width, height;
};

struct RasterParams {
  double footprint_sigma, dilation, alpha_clamp, alpha_skip, termination;
  int32_t tile;        // 16
  int32_t tiles_x, tiles_y;
  int32_t sh_coeffs;
};

// ---------------------------------------------------------------------------------------
// Preprocess of one primitive (fp64): project_all + project_gaussian + tile rectangle.
// ---------------------------------------------------------------------------------------
struct PreOut {
  int visible;
  double depth;
  double mx, my;
  double c00, c01, c11;   // conic (inverse screen covariance); conic(1,0) == conic(0,1)
  double radius;
  double sigma;
  double color[3];
  int32_t tx0, tx1, ty0, ty1;
};

GSF_HD void axis_bounds_d(double a, double z, double r, double f, double c, double& lo, double& hi) {
  // projection.cpp:40-50: extremes over the corners of [a-r, a+r] x [z-r, z+r]
  lo = dinf();
  hi = -lo;
  for (int i = 0; i < 2; ++i) {
    const double da = i == 0 ? -r : r;
    for (int j = 0; j < 2; ++j) {
      const double dz = j == 0 ? -r : r;
      const double u = dadd(c, ddiv(dmul(f, dadd(a, da)), dadd(z, dz)));
      lo = dmin(lo, u);
      hi = dmax(hi, u);
    }
  }
}

GSF_HD int tile_clamp(double v, int hi) {
  const double f = floor(v);
  if (f < 0.0) return 0;
  if (f > static_cast<double>(hi)) return hi;
  return static_cast<int>(f);
}

// SH bases, degree <= 3 (sh.cpp:21-42).
GSF_HD void sh_basis(int degree, double x, double y, double z, double* b) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  b[0] = C0;
  if (degree < 1) return;
  b[1] = dmul(-C1, y);
  b[2] = dmul(C1, z);
  b[3] = dmul(-C1, x);
  if (degree < 2) return;
  const double xx = dmul(x, x), yy = dmul(y, y), zz = dmul(z, z);
  b[4] = dmul(dmul(1.0925484305920792, x), y);
  b[5] = dmul(dmul(-1.0925484305920792, y), z);
  b[6] = dmul(0.31539156525252005, dsub(dsub(dmul(2.0, zz), xx), yy));
  b[7] = dmul(dmul(-1.0925484305920792, x), z);
  b[8] = dmul(0.5462742152960396, dsub(xx, yy));
  if (degree < 3) return;
  b[9] = dmul(dmul(-0.5900435899266435, y), dsub(dmul(3.0, xx), yy));
  b[10] = dmul(dmul(dmul(2.890611442640554, x), y), z);
  b[11] = dmul(dmul(-0.4570457994644658, y), dsub(dsub(dmul(4.0, zz), xx), yy));
  b[12] = dmul(dmul(0.3731763325901154, z), dsub(dsub(dmul(2.0, zz), dmul(3.0, xx)), dmul(3.0, yy)));
  b[13] = dmul(dmul(-0.4570457994644658, x), dsub(dsub(dmul(4.0, zz), xx), yy));
  b[14] = dmul(dmul(1.445305721320277, z), dsub(xx, yy));
  b[15] = dmul(dmul(-0.5900435899266435, x), dsub(xx, dmul(3.0, yy)));
}

// Direction gradients of the SH bases (sh.cpp:44-72), g[3*k + axis].
GSF_HD void sh_basis_grad_d(int degree, double x, double y, double z, double* g) {
  for (int i = 0; i < 48; ++i) g[i] = 0.0;
  if (degree < 1) return;
  const double C1 = 0.4886025119029199;
  g[4] = -C1;
  g[8] = C1;
  g[9] = -C1;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  const double c20 = 1.0925484305920792, c21 = -1.0925484305920792, c22 = 0.31539156525252005, c23 = -1.0925484305920792,
               c24 = 0.5462742152960396;
  g[12] = c20 * y; g[13] = c20 * x;
  g[16] = c21 * z; g[17] = c21 * y;
  g[18] = c22 * (-2.0 * x); g[19] = c22 * (-2.0 * y); g[20] = c22 * (4.0 * z);
  g[21] = c23 * z; g[23] = c23 * x;
  g[24] = c24 * (2.0 * x); g[25] = c24 * (-2.0 * y);
  if (degree < 3) return;
  const double c30 = -0.5900435899266435, c31 = 2.890611442640554, c32 = -0.4570457994644658, c33 = 0.3731763325901154,
               c34 = -0.4570457994644658, c35 = 1.445305721320277, c36 = -0.5900435899266435;
  g[27] = c30 * (6.0 * x * y); g[28] = c30 * (3.0 * xx - 3.0 * yy);
  g[30] = c31 * (y * z); g[31] = c31 * (x * z); g[32] = c31 * (x * y);
  g[33] = c32 * (-2.0 * x * y); g[34] = c32 * (4.0 * zz - xx - 3.0 * yy); g[35] = c32 * (8.0 * y * z);
  g[36] = c33 * (-6.0 * x * z); g[37] = c33 * (-6.0 * y * z); g[38] = c33 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
  g[39] = c34 * (4.0 * zz - 3.0 * xx - yy); g[40] = c34 * (-2.0 * x * y); g[41] = c34 * (8.0 * x * z);
  g[42] = c35 * (2.0 * x * z); g[43] = c35 * (-2.0 * y * z); g[44] = c35 * (xx - yy);
  g[45] = c36 * (3.0 * xx - 3.0 * yy); g[46] = c36 * (-6.0 * x * y);
}

GSF_HD int sh_degree(int K) { return K >= 16 ? 3 : (K >= 9 ? 2 : (K >= 4 ? 1 : 0)); }

// View-independent part of one primitive, cached per map version by the tracking loop (the
// map is constant during track_frame): exactly the values project_core would compute.
struct WorldG {
  double S[9];       // world covariance R diag(exp(2 ls)) R^T (primitive.hpp:46-50)
  double sigma;      // sigmoid(opacity_logit) (primitive.hpp:11,33)
  double color[3];   // SH colour; view-independent when sh_coeffs <= 1
  double pad;
};

// support = footprint_sigma * exp(max log_scale)  (rasterizer.cpp:55)
GSF_HD double world_support(const float* p, int64_t stride, const RasterParams& rp) {
  const double l0 = p[3 * stride], l1 = p[4 * stride], l2 = p[5 * stride];
  return dmul(rp.footprint_sigma, exp_d(dmax(dmax(l0, l1), l2)));
}

// Parameters read straight from the SoA [field][stride] fp32 block (mean 0-2, log_scale 3-5,
// quat 6-9, opacity_logit 10, sh 11+3b+c); p points at field 0 of this primitive.
struct ParamSrc {
  const float* p;
  int64_t stride;
  int K;
  GSF_HD void cov(double* S) const {
    const double l0 = p[3 * stride], l1 = p[4 * stride], l2 = p[5 * stride];
    const double qw = p[6 * stride], qx = p[7 * stride], qy = p[8 * stride], qz = p[9 * stride];
    const double qn = dsqrt(dadd(dadd(dadd(dmul(qw, qw), dmul(qx, qx)), dmul(qy, qy)), dmul(qz, qz)));
    const double w = ddiv(qw, qn), x = ddiv(qx, qn), y = ddiv(qy, qn), z = ddiv(qz, qn);
    double R[9];
    R[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
    R[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
    R[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
    R[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
    R[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
    R[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
    R[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
    R[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
    R[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
    const double s2[3] = {exp_d(dmul(2.0, l0)), exp_d(dmul(2.0, l1)), exp_d(dmul(2.0, l2))};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        S[3 * i + j] = dadd(dadd(dmul(dmul(R[3 * i + 0], s2[0]), R[3 * j + 0]), dmul(dmul(R[3 * i + 1], s2[1]), R[3 * j + 1])),
                            dmul(dmul(R[3 * i + 2], s2[2]), R[3 * j + 2]));
  }
  GSF_HD double sigma() const { return ddiv(1.0, dadd(1.0, exp_d(-static_cast<double>(p[10 * stride])))); }
  // colour through SH along the normalized view direction (rasterizer.cpp:60-63)
  GSF_HD void color(const Cam& cam, double m0, double m1, double m2, double* out) const {
    const double d0 = dsub(m0, cam.center[0]), d1 = dsub(m1, cam.center[1]), d2 = dsub(m2, cam.center[2]);
    const double len = dsqrt(dadd(dadd(dmul(d0, d0), dmul(d1, d1)), dmul(d2, d2)));
    double dx = 0.0, dy = 0.0, dz = 1.0;
    if (len > 1e-12) { dx = ddiv(d0, len); dy = ddiv(d1, len); dz = ddiv(d2, len); }
    if (K <= 0) {
      out[0] = out[1] = out[2] = 0.5;
      return;
    }
    double b[16];
    sh_basis(sh_degree(K), dx, dy, dz, b);
    for (int c = 0; c < 3; ++c) {
      double acc = 0.5;
      for (int k = 0; k < K; ++k) acc = dadd(acc, dmul(b[k], static_cast<double>(p[(11 + 3 * k + c) * stride])));
      out[c] = dmax(acc, 0.0);
    }
  }
};

// The world part from the cache (colour from the parameters when it is view-dependent).
struct CachedSrc {
  const WorldG* w;
  ParamSrc ps;
  GSF_HD void cov(double* S) const {
    for (int i = 0; i < 9; ++i) S[i] = w->S[i];
  }
  GSF_HD double sigma() const { return w->sigma; }
  GSF_HD void color(const Cam& cam, double m0, double m1, double m2, double* out) const {
    if (ps.K <= 1) {
      out[0] = w->color[0]; out[1] = w->color[1]; out[2] = w->color[2];
    } else {
      ps.color(cam, m0, m1, m2, out);
    }
  }
};

// WorldG of one primitive (the colour is evaluated along +z: exact when sh_coeffs <= 1).
GSF_HD WorldG make_world(const float* p, int64_t stride, int K) {
  WorldG g;
  const ParamSrc ps{p, stride, K};
  ps.cov(g.S);
  g.sigma = ps.sigma();
  g.color[0] = g.color[1] = g.color[2] = 0.5;
  if (K == 1) {
    for (int c = 0; c < 3; ++c) g.color[c] = dmax(dadd(0.5, dmul(0.28209479177387814, static_cast<double>(p[(11 + c) * stride]))), 0.0);
  }
  g.pad = 0.0;
  return g;
}

// Camera part of project_all + project_gaussian + tile rectangle for one primitive; the world
// quantities are pulled from src only once the cheap culling tests have passed.
template <class Src>
GSF_HD PreOut project_core(double m0, double m1, double m2, double support, const Src& src, const Cam& cam,
                           const RasterParams& rp) {
  PreOut o;
  o.visible = 0;
  o.depth = 0.0;
  o.mx = o.my = o.c00 = o.c01 = o.c11 = o.radius = o.sigma = 0.0;
  o.color[0] = o.color[1] = o.color[2] = 0.0;
  o.tx0 = o.tx1 = o.ty0 = o.ty1 = 0;
  const double* W = cam.W;
  // p_cam = W * mean + t
  const double pc0 = dadd(dadd(dadd(dmul(W[0], m0), dmul(W[1], m1)), dmul(W[2], m2)), cam.t[0]);
  const double pc1 = dadd(dadd(dadd(dmul(W[3], m0), dmul(W[4], m1)), dmul(W[5], m2)), cam.t[1]);
  const double pc2 = dadd(dadd(dadd(dmul(W[6], m0), dmul(W[7], m1)), dmul(W[8], m2)), cam.t[2]);
  o.depth = pc2;
  if (!(pc2 > cam.near_plane) || !(pc2 < cam.far_plane)) return o;
  if (support > 0.0) {
    if (!(dsub(pc2, support) > 0.0)) return o;
    const double pad = dmul(rp.footprint_sigma, dsqrt(dmax(0.0, rp.dilation)));
    double u_lo, u_hi, v_lo, v_hi;
    axis_bounds_d(pc0, pc2, support, cam.fx, cam.cx, u_lo, u_hi);
    axis_bounds_d(pc1, pc2, support, cam.fy, cam.cy, v_lo, v_hi);
    if (dadd(u_hi, pad) < 0.0 || dsub(u_lo, pad) > static_cast<double>(cam.width) ||
        dadd(v_hi, pad) < 0.0 || dsub(v_lo, pad) > static_cast<double>(cam.height))
      return o;
  }
  o.mx = dadd(ddiv(dmul(cam.fx, pc0), pc2), cam.cx);
  o.my = dadd(ddiv(dmul(cam.fy, pc1), pc2), cam.cy);
  double S[9];
  src.cov(S);
  // J (projection.cpp:26-33)
  const double iz = ddiv(1.0, pc2);
  const double iz2 = dmul(iz, iz);
  const double J[6] = {dmul(cam.fx, iz), 0.0, dmul(dmul(-cam.fx, pc0), iz2),
                       0.0, dmul(cam.fy, iz), dmul(dmul(-cam.fy, pc1), iz2)};
  // cov2d = ((((J W) S) W^T) J^T), left to right as projection.cpp:81
  double A[6], B[6], C[6];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      A[3 * i + j] = dadd(dadd(dmul(J[3 * i + 0], W[0 * 3 + j]), dmul(J[3 * i + 1], W[1 * 3 + j])), dmul(J[3 * i + 2], W[2 * 3 + j]));
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      B[3 * i + j] = dadd(dadd(dmul(A[3 * i + 0], S[0 * 3 + j]), dmul(A[3 * i + 1], S[1 * 3 + j])), dmul(A[3 * i + 2], S[2 * 3 + j]));
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)  // times W^T: (W^T)(k,j) = W(j,k)
      C[3 * i + j] = dadd(dadd(dmul(B[3 * i + 0], W[3 * j + 0]), dmul(B[3 * i + 1], W[3 * j + 1])), dmul(B[3 * i + 2], W[3 * j + 2]));
  double cv[4];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      cv[2 * i + j] = dadd(dadd(dmul(C[3 * i + 0], J[3 * j + 0]), dmul(C[3 * i + 1], J[3 * j + 1])), dmul(C[3 * i + 2], J[3 * j + 2]));
  cv[0] = dadd(cv[0], rp.dilation);
  cv[3] = dadd(cv[3], rp.dilation);
  const double det = dsub(dmul(cv[0], cv[3]), dmul(cv[1], cv[2]));
  const bool fin = disfinite(cv[0]) && disfinite(cv[1]) && disfinite(cv[2]) && disfinite(cv[3]);
  if (!(det > 0.0) || !fin) return o;
  const double inv_det = ddiv(1.0, det);
  o.c00 = dmul(cv[3], inv_det);
  o.c01 = dmul(-cv[1], inv_det);
  o.c11 = dmul(cv[0], inv_det);
  const double mid = dmul(0.5, dadd(cv[0], cv[3]));
  const double lmax2 = dadd(mid, dsqrt(dmax(0.0, dsub(dmul(mid, mid), det))));
  o.radius = dmul(rp.footprint_sigma, dsqrt(lmax2));
  if (dadd(o.mx, o.radius) < 0.0 || dsub(o.mx, o.radius) > static_cast<double>(cam.width) ||
      dadd(o.my, o.radius) < 0.0 || dsub(o.my, o.radius) > static_cast<double>(cam.height))
    return o;
  o.visible = 1;
  o.sigma = src.sigma();
  src.color(cam, m0, m1, m2, o.color);
  // inclusive tile rectangle (rasterizer.cpp:199-208)
  const double ts = static_cast<double>(rp.tile);
  o.tx0 = tile_clamp(ddiv(dsub(o.mx, o.radius), ts), rp.tiles_x - 1);
  o.tx1 = tile_clamp(ddiv(dadd(o.mx, o.radius), ts), rp.tiles_x - 1);
  o.ty0 = tile_clamp(ddiv(dsub(o.my, o.radius), ts), rp.tiles_y - 1);
  o.ty1 = tile_clamp(ddiv(dadd(o.my, o.radius), ts), rp.tiles_y - 1);
  return o;
}

// One primitive from its parameters: project_all + project_gaussian + tile rectangle.
GSF_HD PreOut preprocess_one(const float* p, int64_t stride, const Cam& cam, const RasterParams& rp) {
  const double m0 = p[0 * stride], m1 = p[1 * stride], m2 = p[2 * stride];
  return project_core(m0, m1, m2, world_support(p, stride, rp), ParamSrc{p, stride, rp.sh_coeffs}, cam, rp);
}

// exp_map (lie.cpp:15-28) in explicit fp64; sin/cos are the platform's.
GSF_HD void exp_map_d(const double* v, double* R) {
  const double th2 = dadd(dadd(dmul(v[0], v[0]), dmul(v[1], v[1])), dmul(v[2], v[2]));
  const double th = dsqrt(th2);
  double a, b;
  if (th < 1e-8) {
    a = dsub(1.0, ddiv(th2, 6.0));
    b = dsub(0.5, ddiv(th2, 24.0));
  } else {
    a = ddiv(sin(th), th);
    b = ddiv(dsub(1.0, cos(th)), th2);
  }
  const double k[9] = {0.0, -v[2], v[1], v[2], 0.0, -v[0], -v[1], v[0], 0.0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double kk = dadd(dadd(dmul(k[3 * i + 0], k[0 * 3 + j]), dmul(k[3 * i + 1], k[1 * 3 + j])), dmul(k[3 * i + 2], k[2 * 3 + j]));
      R[3 * i + j] = dadd(dadd(i == j ? 1.0 : 0.0, dmul(a, k[3 * i + j])), dmul(b, kk));
    }
}

// Camera from a pose tangent (pose.hpp:24,41) and intrinsics.
GSF_HD Cam make_cam(const double* rot, const double* trans, double fx, double fy, double cx, double cy,
                    int width, int height, double near_plane, double far_plane) {
  Cam c;
  exp_map_d(rot, c.W);
  for (int i = 0; i < 3; ++i) c.t[i] = trans[i];
  for (int i = 0; i < 3; ++i)
    c.center[i] = -dadd(dadd(dmul(c.W[0 * 3 + i], trans[0]), dmul(c.W[1 * 3 + i], trans[1])), dmul(c.W[2 * 3 + i], trans[2]));
  c.fx = fx; c.fy = fy; c.cx = cx; c.cy = cy;
  c.width = width; c.height = height;
  c.near_plane = near_plane; c.far_plane = far_plane;
  return c;
}

// Depth sort key: IEEE bits of the fp32-rounded depth, offset by the near plane.  Rounding
// is monotone so the key order agrees with the fp64 order up to ties, which the fixup pass
// resolves with the exact (fp64 depth, id) comparison of rasterizer.cpp:74-77.
GSF_HD uint32_t depth_key(double depth, uint32_t near_bits) {
  return static_cast<uint32_t>(fbits(static_cast<float>(depth))) - near_bits;
}

// ---------------------------------------------------------------------------------------
// Blend (fp32) with an fp64 guard band on the two discrete tests of blend_pixel.
// ---------------------------------------------------------------------------------------
struct BlendG {       // per visible primitive, rank order, 3 x float4 on the device
  float mx, my, sigma, rho_hi;       // rho_hi, rho_fast: blend_rho_bounds
  float c00, c01x2, c11, rho_fast;
  float r, g, b, depth;              // (b, depth) adjacent: one register pair for packed FMAs
};
struct GuardG {       // fp64 copies read only inside the guard band
  double mx, my, c00, c01, c11, sigma;
};
GSF_HD BlendG make_blend_g(const PreOut& o) {
  BlendG g;
  g.mx = static_cast<float>(o.mx);
  g.my = static_cast<float>(o.my);
  g.depth = static_cast<float>(o.depth);
  g.sigma = static_cast<float>(o.sigma);
  g.c00 = static_cast<float>(o.c00);
  g.c01x2 = static_cast<float>(dmul(2.0, o.c01));
  g.c11 = static_cast<float>(o.c11);
  g.rho_fast = -1.0f;   // rho_hi / rho_fast: blend_rho_bounds, once the raster constants are known
  g.rho_hi = 3.0e38f;
  g.r = static_cast<float>(o.color[0]);
  g.g = static_cast<float>(o.color[1]);
  g.b = static_cast<float>(o.color[2]);
  return g;
}
GSF_HD GuardG make_guard_g(const PreOut& o) {
  GuardG g;
  g.mx = o.mx; g.my = o.my; g.c00 = o.c00; g.c01 = o.c01; g.c11 = o.c11; g.sigma = o.sigma;
  return g;
}

struct BlendConsts {
  float cutoff;       // footprint_sigma^2
  float skip, clamp, term;
  double cutoff_d, skip_d, clamp_d;
  float rho_band, alpha_band;
  // precomputed decision thresholds (same explicit ops as the full path below)
  float rho_hi, rho_lo, rho_min;      // cutoff + band, cutoff - band, band
  float skip_lo, skip_hi, clamp_lo, clamp_hi;
  int32_t fast_ok;                    // exp_neg_half needs no range check on the fast path
  // exact-decision fix-up (pixel_flag_step / exact_*): fp64 termination threshold, the relative
  // error bound of an unclamped fp32 alpha, the error of the fp32 clamp value and of the fp32
  // termination threshold against their fp64 configuration values
  double term_d;
  float alpha_rel, clamp_err, term_err;
};

GSF_HD BlendConsts make_blend_consts(const RasterParams& rp) {
  BlendConsts k;
  k.cutoff_d = dmul(rp.footprint_sigma, rp.footprint_sigma);
  k.cutoff = static_cast<float>(k.cutoff_d);
  k.skip_d = rp.alpha_skip;
  k.clamp_d = rp.alpha_clamp;
  k.skip = static_cast<float>(rp.alpha_skip);
  k.clamp = static_cast<float>(rp.alpha_clamp);
  k.term = static_cast<float>(rp.termination);
  k.rho_band = static_cast<float>(4e-3 + 2e-4 * k.cutoff_d);
  k.alpha_band = 5e-4f;
  k.rho_hi = fadd(k.cutoff, k.rho_band);
  k.rho_lo = fsub(k.cutoff, k.rho_band);
  k.rho_min = k.rho_band;
  const float sb = fmul(k.skip, k.alpha_band), cb = fmul(k.clamp, k.alpha_band);
  k.skip_lo = fsub(k.skip, sb);
  k.skip_hi = fadd(k.skip, sb);
  k.clamp_lo = fsub(k.clamp, cb);
  k.clamp_hi = fadd(k.clamp, cb);
  k.fast_ok = k.cutoff_d < 170.0 ? 1 : 0;
  k.term_d = rp.termination;
  // fp32 alpha = sigma_f * exp_poly(rho_f): sigma rounding (u/2), the polynomial (< 3e-7), fmul (u/2)
  // and the rho error inside the guard band (band_i / 2 <= 1e-6 relative for the bands the fast
  // path admits; larger bands resolve on the fp64 guard path, whose alpha is the same fp32 product)
  k.alpha_rel = 2e-6f;
  k.clamp_err = static_cast<float>(dmax(rp.alpha_clamp - static_cast<double>(k.clamp),
                                        static_cast<double>(k.clamp) - rp.alpha_clamp)) + 1e-9f;
  k.term_err = static_cast<float>(dmax(rp.termination - static_cast<double>(k.term),
                                       static_cast<double>(k.term) - rp.termination) * 2.0) + 1e-30f;
  return k;
}

GSF_HD double guard_rho(double px, double py, const GuardG& g) {
  const double dx = dsub(px, g.mx), dy = dsub(py, g.my);
  // conic00*dx*dx + 2*conic01*dx*dy + conic11*dy*dy (rasterizer.cpp:108-109)
  return dadd(dadd(dmul(dmul(g.c00, dx), dx), dmul(dmul(dmul(2.0, g.c01), dx), dy)), dmul(dmul(g.c11, dy), dy));
}

// Result of the per-pair test.  code: 0 = skip, 1 = contributes.
struct PairEval {
  int code;
  int clamped;   // sigma*g > alpha_clamp (gradient stop, rasterizer.cpp:451)
  float alpha;   // min(sigma*g, clamp)
  float gval;    // exp(-rho/2)
  float dx, dy;
};

GSF_HD float pair_rho(float dx, float dy, const BlendG& g) {
  return ffma(fmul(g.c00, dx), dx, ffma(fmul(g.c01x2, dx), dy, fmul(fmul(g.c11, dy), dy)));
}

// Full decision (rasterizer.cpp:106-114) with the fp64 guard band around both thresholds.
GSF_HD PairEval eval_pair_full(float px, float py, const BlendG& g, const GuardG* gp, const BlendConsts& k) {
  PairEval e;
  e.dx = fsub(px, g.mx);
  e.dy = fsub(py, g.my);
  const float rho = pair_rho(e.dx, e.dy, g);
  e.code = 0;
  e.clamped = 0;
  e.alpha = 0.0f;
  e.gval = 0.0f;
  double rho_d = -1.0;
  bool have_d = false;
  if (rho > k.rho_hi) return e;                       // rho > cutoff || rho < 0 -> skip
  if (rho >= k.rho_lo || rho < k.rho_min) {
    rho_d = guard_rho(static_cast<double>(px), static_cast<double>(py), *gp);
    have_d = true;
    if (rho_d > k.cutoff_d || rho_d < 0.0) return e;
  }
  e.gval = exp_neg_half(rho);
  const float raw = fmul(g.sigma, e.gval);
  if (raw < k.skip_lo) return e;                      // raw < alpha_skip -> skip
  if (raw <= k.skip_hi) {
    if (!have_d) { rho_d = guard_rho(static_cast<double>(px), static_cast<double>(py), *gp); have_d = true; }
    const double raw_d = dmul(gp->sigma, exp_d(dmul(-0.5, rho_d)));
    if (raw_d < k.skip_d) return e;
  }
  if (raw > k.clamp_hi) {                             // alpha clamp decision
    e.clamped = 1;
  } else if (raw >= k.clamp_lo) {
    if (!have_d) { rho_d = guard_rho(static_cast<double>(px), static_cast<double>(py), *gp); have_d = true; }
    const double raw_d = dmul(gp->sigma, exp_d(dmul(-0.5, rho_d)));
    e.clamped = raw_d > k.clamp_d ? 1 : 0;
  }
  e.alpha = e.clamped ? k.clamp : fminf_(raw, k.clamp);
  e.code = 1;
  return e;
}

// Per-primitive decision bounds.  The fp32 rho of a pixel differs from the fp64 reference's by at
// most band_i, which depends on the primitive (rounding of mean2d, whose error grows with |mean2d|
// and is amplified by the slope of the quadratic form at rho ~ cutoff, plus the rounding of the
// conic and of the evaluation); the global rho_band of BlendConsts is its worst case.  With
// cutoff - band_i and cutoff + band_i as the primitive's own band edges the fp64 guard only runs
// for pixels that can really sit on the cutoff.
//   rho_hi:   rho > rho_hi certainly fails the footprint test (skip)
//   rho_fast: rho < rho_fast is certainly "contributes, unclamped, alpha = sigma*exp(-rho/2)" —
//             rho is below the cutoff band, alpha is above the skip band (margin 1e-5 in log space,
//             >> the exp error of 3e-7) and sigma is below the clamp band.  No lower bound is
//             needed: the fp64 guard for rho < rho_min only rejects rho_d < 0, and for a conic with
//             det >= 1e-5 c00 c11 (condition number < 4e5, in fp32 and hence in fp64) the fp64
//             quadratic form is non-negative everywhere (its rounding error is < 1e-15 of its
//             largest term), so there the guard never fires.  -1 disables the fast path.
// Both only select the evaluation path, never a result, so the mirror and the kernels stay
// bit-identical either way.
//
// Bound (u = 2^-24; a, b, c the conic, Q = rho, K = max of (|a dx^2| + 2|b dx dy| + |c dy^2|) / Q
// = 2 sqrt(ac) / (sqrt(ac) - |b|)): |dx - dx_d| <= u (|mx| + |dx|); |grad_x Q| <= 2 sqrt(a Q) on
// the ellipse Q; the five roundings of pair_rho and the conic's own rounding <= 6 u K Q.  band_i
// takes Q = cutoff + 1, doubles every term, then a factor 4 and 1e-6 absolute on top.
GSF_HD void blend_rho_bounds(BlendG& g, const BlendConsts& k) {
  g.rho_hi = k.rho_hi;
  g.rho_fast = -1.0f;
  const double a = g.c00, b = 0.5 * static_cast<double>(g.c01x2), c = g.c11;
  if (!(a > 0.0 && c > 0.0 && a * c - b * b >= 1e-5 * a * c)) return;   // the global band and the full path
  const double det = a * c - b * b, sac = sqrt(a * c);
  const double qm = k.cutoff_d + 1.0;
  const double K = 2.0 * sac / (sac - fabs(b));
  const double dxm = sqrt(qm * c / det), dym = sqrt(qm * a / det);
  const double u = 5.9604644775390625e-8;
  const double e = 2.0 * (6.0 * u * qm * K + 2.0 * sqrt(a * qm) * u * (fabs(static_cast<double>(g.mx)) + dxm + 1.0) +
                          2.0 * sqrt(c * qm) * u * (fabs(static_cast<double>(g.my)) + dym + 1.0));
  const double band = fmin(4.0 * e + 1e-6, static_cast<double>(k.rho_band));
  float hi = static_cast<float>(k.cutoff_d + band);
  if (static_cast<double>(hi) < k.cutoff_d + band) hi = nextafterf(hi, 3.0e38f);
  g.rho_hi = fminf(hi, k.rho_hi);
  const float sigma = g.sigma;
  if (!k.fast_ok || !(static_cast<double>(sigma) * (1.0 + 1e-6) < static_cast<double>(k.clamp_lo))) return;
  if (!(sigma > k.skip_hi)) return;
  const double ra = 2.0 * (log(static_cast<double>(sigma) / static_cast<double>(k.skip_hi)) - 1e-5);
  const double lo = k.cutoff_d - band;
  const double r = ra < lo ? ra : lo;
  g.rho_fast = r > 0.0 ? static_cast<float>(r * (1.0 - 1e-6)) : -1.0f;
}

// exp(-rho/2) on the hardware exp2 unit (|rel err| < 2^-21): used by the pose backward only
// where the decision is already certain (the rho_fast path).  Its alpha then differs from the
// forward's in the last bits, which only perturbs the recovered T at the 1e-7 level; every
// forward stays on the exact polynomial (bit-identical to the mirror, and a track_frame at the
// optimum sees exactly zero residuals, test_tracker.cpp:192-244).
GSF_HD float exp_neg_half_fast(float rho) {
#ifdef __CUDA_ARCH__
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(rho * -0.72134752044448170f));
  return y;
#else
  return exp_neg_half_inrange(rho);
#endif
}

// Same decisions as eval_pair_full; the common cases are resolved inline and only band cases
// take the fp64 path.  `gp` is only dereferenced on that path.
template <bool FAST>
GSF_HD PairEval eval_pair_t(float px, float py, const BlendG& g, const GuardG* gp, const BlendConsts& k) {
  PairEval e;
#ifdef __CUDA_ARCH__
  {   // one packed FADD2; p - m == p + (-m) exactly, so the bits equal the two fsub's
    const float2 d = __fadd2_rn(make_float2(px, py), make_float2(-g.mx, -g.my));
    e.dx = d.x;
    e.dy = d.y;
  }
#else
  e.dx = fsub(px, g.mx);
  e.dy = fsub(py, g.my);
#endif
  const float rho = pair_rho(e.dx, e.dy, g);
  e.code = 0;
  e.clamped = 0;
  e.alpha = 0.0f;
  e.gval = 0.0f;
  if (rho > g.rho_hi) return e;
  if (rho < g.rho_fast) {
    e.gval = FAST ? exp_neg_half_fast(rho) : exp_neg_half_inrange(rho);
    e.alpha = fmul(g.sigma, e.gval);
    e.code = 1;
    return e;
  }
  return eval_pair_full(px, py, g, gp, k);
}

GSF_HD PairEval eval_pair(float px, float py, const BlendG& g, const GuardG* gp, const BlendConsts& k) {
  return eval_pair_t<false>(px, py, g, gp, k);
}

struct PixelState {
  float T;
  float cr, cg, cb, ad, op, unc, best, med_depth;
  int32_t count, dominant, median, last;   // last = list index + 1 of the last contributor
  int32_t done;
  float eT;        // bound on |T_fp32 - T_fp64| / T (exact-decision fix-up, render API only)
  int32_t flag;    // a discrete decision lies within the fp32 error of its threshold
};

GSF_HD void pixel_init(PixelState& s) {
  s.T = 1.0f;
  s.cr = s.cg = s.cb = s.ad = s.op = s.unc = s.best = s.med_depth = 0.0f;
  s.count = 0;
  s.dominant = -1;
  s.median = -1;
  s.last = 0;
  s.done = 0;
  s.eT = 0.0f;
  s.flag = 0;
}

// Accumulate one contributing pair (rasterizer.cpp:116-137).  `id` is the primitive id.
GSF_HD void pixel_flag_step(PixelState& s, float alpha, int clamped, float w, float t_next, const BlendConsts& k);

GSF_HD void pixel_accumulate(PixelState& s, const BlendG& g, const PairEval& e, int32_t id, int32_t list_index,
                             bool obs_valid, float obs, const BlendConsts& k, bool flag_exact = false) {
  const float w = fmul(e.alpha, s.T);
  if (flag_exact) pixel_flag_step(s, e.alpha, e.clamped, w, fmul(s.T, fsub(1.0f, e.alpha)), k);
  s.cr = ffma(w, g.r, s.cr);
  s.cg = ffma(w, g.g, s.cg);
  s.cb = ffma(w, g.b, s.cb);
  s.ad = ffma(w, g.depth, s.ad);
  s.op = fadd(s.op, w);
  if (obs_valid) {
    const float d = fsub(g.depth, obs);
    s.unc = ffma(fmul(w, d), d, s.unc);
  }
  if (w > s.best) {
    s.best = w;
    s.dominant = id;
  }
  s.count += 1;
  s.last = list_index + 1;
  const float t_next = fmul(s.T, fsub(1.0f, e.alpha));
  if (s.median < 0 && s.T >= 0.5f && t_next < 0.5f) {
    s.median = id;
    s.med_depth = g.depth;
  }
  s.T = t_next;
  if (s.T < k.term) s.done = 1;
}

// Tracking variant: only the maps the tracking loss and the pose backward read (colour, alpha
// depth, opacity, T, last contributor).  Same operations in the same order as pixel_accumulate
// for those fields, so the values are identical to a full render's.
GSF_HD void pixel_accumulate_min(PixelState& s, const BlendG& g, const PairEval& e, int32_t list_index,
                                 const BlendConsts& k) {
  const float w = fmul(e.alpha, s.T);
  s.cr = ffma(w, g.r, s.cr);
  s.cg = ffma(w, g.g, s.cg);
  s.cb = ffma(w, g.b, s.cb);
  s.ad = ffma(w, g.depth, s.ad);
  s.op = fadd(s.op, w);
  s.last = list_index + 1;
  s.T = fmul(s.T, fsub(1.0f, e.alpha));
  if (s.T < k.term) s.done = 1;
}

// ---------------------------------------------------------------------------------------------
// Exact discrete decisions of the render API (rasterizer.cpp:116-137 in fp64).
//
// The fp32 blend agrees with the fp64 reference on every per-pair decision (the fp64 guard
// bands above), but T, w = alpha T and the running maximum are fp32 accumulations: where the
// termination test (T < 1e-8), the median crossing (T >= 0.5 > T') or the dominant's strict
// maximum sits within their rounding error of its threshold, the fp64 reference can decide the
// other way (~1e-5 of pixels on a saturated 500k-primitive frame).  pixel_flag_step carries a
// bound on T's relative error along the walk and flags such pixels; exact_alpha /
// exact_accumulate re-blend a flagged pixel in fp64 with the reference's formulas, and that
// result replaces the fp32 one.  Device and mirror run the same functions, so they stay
// bit-identical, and the flagged pixels' integer outputs are the fp64 reference's.
// ---------------------------------------------------------------------------------------------
GSF_HD void pixel_flag_step(PixelState& s, float alpha, int clamped, float w, float t_next, const BlendConsts& k) {
  const float u = 5.9604645e-8f;
  const float ea = clamped ? k.clamp_err : fmul(k.alpha_rel, alpha);   // |alpha_f - alpha_d|
  const float om = fsub(1.0f, alpha);
  const float e_pre = s.eT;
  s.eT = fadd(fadd(e_pre, fdiv(ffma(u, om, ea), om)), u);               // + rel. error of (1 - alpha), fmul
  const float m = fmul(4.0f, s.eT);
  // termination: T' < term
  if (fabsf(fsub(t_next, k.term)) <= fadd(fmul(m, k.term), k.term_err)) s.flag = 1;
  // median crossing at 0.5 while no median is chosen (the first step's T = 1 is exact)
  if (s.median < 0 && fabsf(fsub(t_next, 0.5f)) <= fmul(m, 0.5f)) s.flag = 1;
  // dominant: first strict maximum of w (error of w: T's before the step, alpha's, the fmul)
  if (s.best > 0.0f) {
    const float ew = fadd(fadd(e_pre, fdiv(ea, alpha)), u);
    const float big = w > s.best ? w : s.best;
    if (fabsf(fsub(w, s.best)) <= fmul(fmul(8.0f, fadd(ew, fadd(e_pre, u))), big)) s.flag = 1;
  }
}

// The reference's per-pair decision in fp64 (rasterizer.cpp:106-114) from the fp64 guard copies:
// returns 0 (skip) or 1 with alpha = min(sigma g, clamp).
GSF_HD int exact_alpha(double px, double py, const GuardG& g, const BlendConsts& k, double* alpha) {
  const double rho = guard_rho(px, py, g);
  if (rho > k.cutoff_d || rho < 0.0) return 0;
  const double raw = dmul(g.sigma, exp_d(dmul(-0.5, rho)));
  if (raw < k.skip_d) return 0;
  *alpha = raw > k.clamp_d ? k.clamp_d : raw;
  return 1;
}

struct ExactPixel {
  double T, cr, cg, cb, ad, op, unc, best, med_depth;
  int32_t count, dominant, median, last, done;
};

GSF_HD void exact_init(ExactPixel& s) {
  s.T = 1.0;
  s.cr = s.cg = s.cb = s.ad = s.op = s.unc = s.best = s.med_depth = 0.0;
  s.count = 0;
  s.dominant = -1;
  s.median = -1;
  s.last = 0;
  s.done = 0;
}

// blend_pixel's accumulation (rasterizer.cpp:116-137) in fp64; colour and depth are the fp32
// per-primitive values the fp32 path blends.
GSF_HD void exact_accumulate(ExactPixel& s, double alpha, const BlendG& g, int32_t id, int32_t list_index, bool obs_valid,
                             double obs, const BlendConsts& k) {
  const double w = dmul(alpha, s.T);
  s.cr = dadd(s.cr, dmul(w, static_cast<double>(g.r)));
  s.cg = dadd(s.cg, dmul(w, static_cast<double>(g.g)));
  s.cb = dadd(s.cb, dmul(w, static_cast<double>(g.b)));
  s.ad = dadd(s.ad, dmul(w, static_cast<double>(g.depth)));
  s.op = dadd(s.op, w);
  if (obs_valid) {
    const double d = dsub(static_cast<double>(g.depth), obs);
    s.unc = dadd(s.unc, dmul(dmul(w, d), d));
  }
  if (w > s.best) {
    s.best = w;
    s.dominant = id;
  }
  s.count += 1;
  s.last = list_index + 1;
  const double t_next = dmul(s.T, dsub(1.0, alpha));
  if (s.median < 0 && s.T >= 0.5 && t_next < 0.5) {
    s.median = id;
    s.med_depth = static_cast<double>(g.depth);
  }
  s.T = t_next;
  if (s.T < k.term_d) s.done = 1;
}

}  // namespace gsfk
