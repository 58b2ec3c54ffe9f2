// gsf_oracle.cpp — TEST INFRASTRUCTURE ONLY (see gsf_oracle.h).
//
// A line-by-line fp64 restatement of the reference hot path, without Eigen.  Each function
// names the reference file:line it restates (paths relative to /root/reference/proj/src or
// include/gsfield).  Small fixed-size linear algebra is spelled out with the reference's
// evaluation order (left-to-right products, index-ordered dot products).
//
// Third-party arithmetic in the reference: Eigen3 (>= 3.3, unpinned, not vendored) carries
// the fixed-size matrix products.  Its vectorised reductions may differ from this scalar
// restatement in the last ulp; the reference's own tests never pin bits across Eigen builds
// (KATs use 1e-12 tolerances), so neither do we.

#include "gsf_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <limits>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

// parallel_for (core/parallel.hpp:13-31): static chunks over std::threads; threads from
// ORACLE_THREADS or the hardware concurrency, like RasterConfig::threads = 0.
int oracle_threads() {
  static const int n = [] {
    const char* e = std::getenv("ORACLE_THREADS");
    if (e && std::atoi(e) > 0) return std::atoi(e);
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
  }();
  return n;
}
template <class F>
void parallel_for(size_t n, F&& body) {
  const int threads = oracle_threads();
  if (n == 0) return;
  if (threads <= 1 || n == 1) { body(size_t(0), n); return; }
  const size_t workers = std::min<size_t>(static_cast<size_t>(threads), n);
  const size_t chunk = (n + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (size_t w = 1; w < workers; ++w) {
    const size_t lo = w * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&body, lo, hi] { body(lo, hi); });
  }
  body(size_t(0), std::min(n, chunk));
  for (auto& t : pool) t.join();
}

struct V2 {
  double x = 0, y = 0;
  V2() = default;
  V2(double a, double b) : x(a), y(b) {}
};
struct V3 {
  double v[3] = {0, 0, 0};
  V3() = default;
  V3(double a, double b, double c) { v[0] = a; v[1] = b; v[2] = c; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
struct V4 {
  double v[4] = {0, 0, 0, 0};
  V4() = default;
  V4(double a, double b, double c, double d) { v[0] = a; v[1] = b; v[2] = c; v[3] = d; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double* operator[](int i) { return m[i]; }
  const double* operator[](int i) const { return m[i]; }
  static M3 I() { M3 r; r[0][0] = r[1][1] = r[2][2] = 1.0; return r; }
};
struct M2 { double m[2][2] = {{0, 0}, {0, 0}}; };
struct M23 { double m[2][3] = {{0, 0, 0}, {0, 0, 0}}; };

inline V3 operator+(const V3& a, const V3& b) { return V3(a[0] + b[0], a[1] + b[1], a[2] + b[2]); }
inline V3 operator-(const V3& a, const V3& b) { return V3(a[0] - b[0], a[1] - b[1], a[2] - b[2]); }
inline V3 operator*(double s, const V3& a) { return V3(s * a[0], s * a[1], s * a[2]); }
inline V3 operator/(const V3& a, double s) { return V3(a[0] / s, a[1] / s, a[2] / s); }
inline V3 operator-(const V3& a) { return V3(-a[0], -a[1], -a[2]); }
inline V3& operator+=(V3& a, const V3& b) { for (int i = 0; i < 3; ++i) a[i] += b[i]; return a; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double sqnorm(const V3& a) { return dot(a, a); }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(const V3& a, const V3& b) {
  return V3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}
inline bool finite3(const V3& a) { return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]); }
inline bool zero3(const V3& a) { return a[0] == 0.0 && a[1] == 0.0 && a[2] == 0.0; }

inline M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i][j] = a[i][0] * b[0][j] + a[i][1] * b[1][j] + a[i][2] * b[2][j];
  return r;
}
inline V3 mul(const M3& a, const V3& v) {
  return V3(a[0][0] * v[0] + a[0][1] * v[1] + a[0][2] * v[2],
            a[1][0] * v[0] + a[1][1] * v[1] + a[1][2] * v[2],
            a[2][0] * v[0] + a[2][1] * v[1] + a[2][2] * v[2]);
}
inline M3 tr(const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i][j] = a[j][i];
  return r;
}
inline M3 add(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i][j] = a[i][j] + b[i][j];
  return r;
}
inline M3 scale(double s, const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i][j] = s * a[i][j];
  return r;
}
inline M23 mul(const M23& a, const M3& b) {
  M23 r;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][0] * b[0][j] + a.m[i][1] * b[1][j] + a.m[i][2] * b[2][j];
  return r;
}

// ---- lie.cpp:7-52 ------------------------------------------------------------------------
M3 skew(const V3& v) {
  M3 s;
  s[0][0] = 0.0; s[0][1] = -v[2]; s[0][2] = v[1];
  s[1][0] = v[2]; s[1][1] = 0.0; s[1][2] = -v[0];
  s[2][0] = -v[1]; s[2][1] = v[0]; s[2][2] = 0.0;
  return s;
}

M3 exp_map(const V3& t) {
  const double theta2 = sqnorm(t);
  const double theta = std::sqrt(theta2);
  double a, b;
  if (theta < 1e-8) {
    a = 1.0 - theta2 / 6.0;
    b = 0.5 - theta2 / 24.0;
  } else {
    a = std::sin(theta) / theta;
    b = (1.0 - std::cos(theta)) / theta2;
  }
  const M3 k = skew(t);
  return add(add(M3::I(), scale(a, k)), scale(b, mul(k, k)));
}

V3 log_map(const M3& r) {
  const double trace = r[0][0] + r[1][1] + r[2][2];
  const double cos_theta = std::clamp((trace - 1.0) * 0.5, -1.0, 1.0);
  const double theta = std::acos(cos_theta);
  const V3 vee(r[2][1] - r[1][2], r[0][2] - r[2][0], r[1][0] - r[0][1]);
  if (theta < 1e-8) return (0.5 * (1.0 + theta * theta / 6.0)) * vee;
  if (theta > M_PI - 1e-3) {
    M3 sym;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sym[i][j] = 0.5 * (r[i][j] + r[j][i]);
    M3 outer;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) outer[i][j] = (sym[i][j] - cos_theta * (i == j ? 1.0 : 0.0)) / (1.0 - cos_theta);
    int axis_idx = 0;
    for (int i = 1; i < 3; ++i)
      if (outer[i][i] > outer[axis_idx][axis_idx]) axis_idx = i;
    const double sq = std::sqrt(outer[axis_idx][axis_idx]);
    V3 axis(outer[0][axis_idx] / sq, outer[1][axis_idx] / sq, outer[2][axis_idx] / sq);
    if (dot(axis, vee) < 0.0) axis = -axis;
    return theta * axis;
  }
  return (theta / (2.0 * std::sin(theta))) * vee;
}

// ---- pose.hpp:13-49 -----------------------------------------------------------------------
struct Pose {
  V3 rot, trans;
  M3 rotation() const { return exp_map(rot); }
  V3 center() const { return -(mul(tr(rotation()), trans)); }
  Pose perturbed(const double d[6]) const {
    const M3 d_rot = exp_map(V3(d[0], d[1], d[2]));
    const M3 r_new = mul(d_rot, rotation());
    return {log_map(r_new), mul(d_rot, trans) + V3(d[3], d[4], d[5])};
  }
};
Pose to_pose(const gsf_pose* p) {
  Pose r;
  for (int i = 0; i < 3; ++i) { r.rot[i] = p->rotation_tangent[i]; r.trans[i] = p->translation[i]; }
  return r;
}
void from_pose(const Pose& p, gsf_pose* out) {
  for (int i = 0; i < 3; ++i) { out->rotation_tangent[i] = p.rot[i]; out->translation[i] = p.trans[i]; }
}

// ---- primitive.hpp:16-59 ----------------------------------------------------------------
inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }
inline double logit(double p) { return std::log(p / (1.0 - p)); }

struct Prim {
  V3 mean, log_scale;
  V4 quat{1, 0, 0, 0};
  double opacity_logit = 0.0;
  std::vector<V3> sh;
  double uncertainty = 0.0;
  bool observed = false;

  V3 scale() const { return V3(std::exp(log_scale[0]), std::exp(log_scale[1]), std::exp(log_scale[2])); }
  double opacity() const { return sigmoid(opacity_logit); }
  V4 qn() const {
    const double n = std::sqrt(quat[0] * quat[0] + quat[1] * quat[1] + quat[2] * quat[2] + quat[3] * quat[3]);
    return V4(quat[0] / n, quat[1] / n, quat[2] / n, quat[3] / n);
  }
  double qnorm() const {
    return std::sqrt(quat[0] * quat[0] + quat[1] * quat[1] + quat[2] * quat[2] + quat[3] * quat[3]);
  }
  M3 rotation() const {
    const V4 q = qn();
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    M3 r;
    r[0][0] = 1 - 2 * (y * y + z * z); r[0][1] = 2 * (x * y - w * z); r[0][2] = 2 * (x * z + w * y);
    r[1][0] = 2 * (x * y + w * z); r[1][1] = 1 - 2 * (x * x + z * z); r[1][2] = 2 * (y * z - w * x);
    r[2][0] = 2 * (x * z - w * y); r[2][1] = 2 * (y * z + w * x); r[2][2] = 1 - 2 * (x * x + y * y);
    return r;
  }
  // covariance(): R diag(exp(2 log_scale)) R^T (primitive.hpp:46-50)
  M3 covariance() const {
    const M3 r = rotation();
    const V3 s2(std::exp(2.0 * log_scale[0]), std::exp(2.0 * log_scale[1]), std::exp(2.0 * log_scale[2]));
    M3 rd;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) rd[i][j] = r[i][j] * s2[j];
    return mul(rd, tr(r));
  }
};

std::vector<Prim> load_map(const gsf_map_host* m) {
  if (m->count < 0) throw std::invalid_argument("map: negative primitive count");
  std::vector<Prim> p(static_cast<size_t>(m->count));
  const int K = m->sh_coeffs;
  for (int64_t i = 0; i < m->count; ++i) {
    Prim& q = p[i];
    for (int a = 0; a < 3; ++a) { q.mean[a] = m->mean[3 * i + a]; q.log_scale[a] = m->log_scale[3 * i + a]; }
    for (int a = 0; a < 4; ++a) q.quat[a] = m->quat[4 * i + a];
    q.opacity_logit = m->opacity_logit[i];
    q.sh.resize(K);
    for (int b = 0; b < K; ++b)
      for (int c = 0; c < 3; ++c) q.sh[b][c] = m->sh[(3 * K) * i + 3 * b + c];
    q.uncertainty = m->uncertainty ? m->uncertainty[i] : 0.0;
    q.observed = m->observed ? m->observed[i] != 0 : false;
  }
  return p;
}

void store_map(const std::vector<Prim>& p, gsf_map_host* m) {
  const int K = m->sh_coeffs;
  for (size_t i = 0; i < p.size(); ++i) {
    const Prim& q = p[i];
    if (m->mean) for (int a = 0; a < 3; ++a) m->mean[3 * i + a] = q.mean[a];
    if (m->log_scale) for (int a = 0; a < 3; ++a) m->log_scale[3 * i + a] = q.log_scale[a];
    if (m->quat) for (int a = 0; a < 4; ++a) m->quat[4 * i + a] = q.quat[a];
    if (m->opacity_logit) m->opacity_logit[i] = q.opacity_logit;
    if (m->sh)
      for (int b = 0; b < K && b < static_cast<int>(q.sh.size()); ++b)
        for (int c = 0; c < 3; ++c) m->sh[(3 * K) * i + 3 * b + c] = q.sh[b][c];
    if (m->uncertainty) m->uncertainty[i] = q.uncertainty;
    if (m->observed) m->observed[i] = q.observed ? 1 : 0;
  }
}

// ---- camera.hpp:9-36 ----------------------------------------------------------------------
void validate_intrinsics(const gsf_intrinsics& k) {
  if (!(k.fx > 0.0) || !(k.fy > 0.0)) throw std::invalid_argument("intrinsics: focal lengths must be positive");
  if (k.width <= 0 || k.height <= 0) throw std::invalid_argument("intrinsics: image size must be positive");
  if (!(k.depth_scale > 0.0)) throw std::invalid_argument("intrinsics: depth_scale must be positive");
  if (!(k.near_plane > 0.0) || !(k.far_plane > k.near_plane))
    throw std::invalid_argument("intrinsics: need 0 < near < far");
}

// ---- projection.cpp:10-104 -------------------------------------------------------------------
struct Proj {
  V2 mean2d;
  M2 cov2d, conic;
  double depth = 0.0, radius = 0.0;
  bool visible = false;
};

M23 projection_jacobian(const V3& p, const gsf_intrinsics& k) {
  const double iz = 1.0 / p[2];
  const double iz2 = iz * iz;
  M23 j;
  j.m[0][0] = k.fx * iz; j.m[0][1] = 0.0; j.m[0][2] = -k.fx * p[0] * iz2;
  j.m[1][0] = 0.0; j.m[1][1] = k.fy * iz; j.m[1][2] = -k.fy * p[1] * iz2;
  return j;
}

void axis_bounds(double a, double z, double r, double f, double c, double& lo, double& hi) {
  lo = std::numeric_limits<double>::infinity();
  hi = -lo;
  for (double da : {-r, r})
    for (double dz : {-r, r}) {
      const double u = c + f * (a + da) / (z + dz);
      lo = std::min(lo, u);
      hi = std::max(hi, u);
    }
}

Proj project_gaussian(const V3& mean_world, const M3& cov_world, const M3& w, const V3& t,
                      const gsf_intrinsics& k, double dilation, double footprint_sigma,
                      double support_radius) {
  Proj out;
  const V3 p_cam = mul(w, mean_world) + t;
  out.depth = p_cam[2];
  if (!(p_cam[2] > k.near_plane) || !(p_cam[2] < k.far_plane)) return out;
  if (support_radius > 0.0) {
    if (!(p_cam[2] - support_radius > 0.0)) return out;
    const double pad = footprint_sigma * std::sqrt(std::max(0.0, dilation));
    double u_lo, u_hi, v_lo, v_hi;
    axis_bounds(p_cam[0], p_cam[2], support_radius, k.fx, k.cx, u_lo, u_hi);
    axis_bounds(p_cam[1], p_cam[2], support_radius, k.fy, k.cy, v_lo, v_hi);
    if (u_hi + pad < 0.0 || u_lo - pad > k.width || v_hi + pad < 0.0 || v_lo - pad > k.height) return out;
  }
  out.mean2d = V2(k.fx * p_cam[0] / p_cam[2] + k.cx, k.fy * p_cam[1] / p_cam[2] + k.cy);
  const M23 j = projection_jacobian(p_cam, k);
  // j * w * cov_world * w^T * j^T, evaluated left to right (projection.cpp:81)
  const M23 jw = mul(j, w);
  const M23 jwc = mul(jw, cov_world);
  const M23 jwcw = mul(jwc, tr(w));
  M2 cov2d;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      cov2d.m[a][b] = jwcw.m[a][0] * j.m[b][0] + jwcw.m[a][1] * j.m[b][1] + jwcw.m[a][2] * j.m[b][2];
  cov2d.m[0][0] += dilation;
  cov2d.m[1][1] += dilation;
  out.cov2d = cov2d;
  const double det = cov2d.m[0][0] * cov2d.m[1][1] - cov2d.m[0][1] * cov2d.m[1][0];
  const bool fin = std::isfinite(cov2d.m[0][0]) && std::isfinite(cov2d.m[0][1]) &&
                   std::isfinite(cov2d.m[1][0]) && std::isfinite(cov2d.m[1][1]);
  if (!(det > 0.0) || !fin) return out;
  const double inv_det = 1.0 / det;
  out.conic.m[0][0] = cov2d.m[1][1] * inv_det;
  out.conic.m[0][1] = -cov2d.m[0][1] * inv_det;
  out.conic.m[1][0] = -cov2d.m[1][0] * inv_det;
  out.conic.m[1][1] = cov2d.m[0][0] * inv_det;
  const double mid = 0.5 * (cov2d.m[0][0] + cov2d.m[1][1]);
  const double lambda_max = mid + std::sqrt(std::max(0.0, mid * mid - det));
  out.radius = footprint_sigma * std::sqrt(lambda_max);
  if (out.mean2d.x + out.radius < 0.0 || out.mean2d.x - out.radius > k.width ||
      out.mean2d.y + out.radius < 0.0 || out.mean2d.y - out.radius > k.height)
    return out;
  out.visible = true;
  return out;
}

// ---- sh.cpp:9-108 ----------------------------------------------------------------------
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                           -1.0925484305920792, 0.5462742152960396};
constexpr double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                           0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                           -0.5900435899266435};

int sh_degree_from_count(int count) {
  switch (count) {
    case 1: return 0;
    case 4: return 1;
    case 9: return 2;
    case 16: return 3;
    default: throw std::invalid_argument("sh coefficient count must be 1, 4, 9 or 16");
  }
}

void basis_values(int degree, double x, double y, double z, double* b) {
  b[0] = kC0;
  if (degree < 1) return;
  b[1] = -kC1 * y;
  b[2] = kC1 * z;
  b[3] = -kC1 * x;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  b[4] = kC2[0] * x * y;
  b[5] = kC2[1] * y * z;
  b[6] = kC2[2] * (2.0 * zz - xx - yy);
  b[7] = kC2[3] * x * z;
  b[8] = kC2[4] * (xx - yy);
  if (degree < 3) return;
  b[9] = kC3[0] * y * (3.0 * xx - yy);
  b[10] = kC3[1] * x * y * z;
  b[11] = kC3[2] * y * (4.0 * zz - xx - yy);
  b[12] = kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  b[13] = kC3[4] * x * (4.0 * zz - xx - yy);
  b[14] = kC3[5] * z * (xx - yy);
  b[15] = kC3[6] * x * (xx - 3.0 * yy);
}

void basis_gradients(int degree, double x, double y, double z, V3* g) {
  g[0] = V3();
  if (degree < 1) return;
  g[1] = V3(0.0, -kC1, 0.0);
  g[2] = V3(0.0, 0.0, kC1);
  g[3] = V3(-kC1, 0.0, 0.0);
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  g[4] = kC2[0] * V3(y, x, 0.0);
  g[5] = kC2[1] * V3(0.0, z, y);
  g[6] = kC2[2] * V3(-2.0 * x, -2.0 * y, 4.0 * z);
  g[7] = kC2[3] * V3(z, 0.0, x);
  g[8] = kC2[4] * V3(2.0 * x, -2.0 * y, 0.0);
  if (degree < 3) return;
  g[9] = kC3[0] * V3(6.0 * x * y, 3.0 * xx - 3.0 * yy, 0.0);
  g[10] = kC3[1] * V3(y * z, x * z, x * y);
  g[11] = kC3[2] * V3(-2.0 * x * y, 4.0 * zz - xx - 3.0 * yy, 8.0 * y * z);
  g[12] = kC3[3] * V3(-6.0 * x * z, -6.0 * y * z, 6.0 * zz - 3.0 * xx - 3.0 * yy);
  g[13] = kC3[4] * V3(4.0 * zz - 3.0 * xx - yy, -2.0 * x * y, 8.0 * x * z);
  g[14] = kC3[5] * V3(2.0 * x * z, -2.0 * y * z, xx - yy);
  g[15] = kC3[6] * V3(3.0 * xx - 3.0 * yy, -6.0 * x * y, 0.0);
}

V3 eval_sh_color(const std::vector<V3>& sh, const V3& dir) {
  const int degree = sh_degree_from_count(static_cast<int>(sh.size()));
  double b[16];
  basis_values(degree, dir[0], dir[1], dir[2], b);
  V3 c(0.5, 0.5, 0.5);
  for (size_t i = 0; i < sh.size(); ++i) c += b[i] * sh[i];
  return V3(std::max(c[0], 0.0), std::max(c[1], 0.0), std::max(c[2], 0.0));
}

void eval_sh_color_backward(const std::vector<V3>& sh, const V3& dir, const V3& d_color,
                            std::vector<V3>& d_sh, V3& d_dir) {
  const int degree = sh_degree_from_count(static_cast<int>(sh.size()));
  double b[16];
  basis_values(degree, dir[0], dir[1], dir[2], b);
  V3 raw(0.5, 0.5, 0.5);
  for (size_t i = 0; i < sh.size(); ++i) raw += b[i] * sh[i];
  V3 masked = d_color;
  for (int c = 0; c < 3; ++c)
    if (raw[c] < 0.0) masked[c] = 0.0;
  for (size_t i = 0; i < sh.size(); ++i) d_sh[i] += b[i] * masked;
  if (degree >= 1) {
    V3 g[16];
    basis_gradients(degree, dir[0], dir[1], dir[2], g);
    for (size_t i = 1; i < sh.size(); ++i) d_dir += dot(masked, sh[i]) * g[i];
  }
}

// ---- rasterizer.cpp ------------------------------------------------------------------------
struct PrimCache {
  Proj proj;
  V3 color;
  double sigma = 0.0;
};
struct Contrib {
  int32_t id;
  double alpha, transmittance;
};

struct Image3 {
  int w = 0, h = 0;
  std::vector<V3> d;
};

struct RenderOut {
  int width = 0, height = 0;
  std::vector<V3> color;
  std::vector<double> alpha_depth, median_depth, opacity, uncertainty, final_t, dom_w;
  std::vector<uint8_t> median_valid;
  std::vector<int32_t> count;
  bool has_uncertainty = false;
  void init(int w, int h) {
    width = w; height = h;
    const size_t n = static_cast<size_t>(w) * h;
    color.assign(n, V3());
    alpha_depth.assign(n, 0.0); median_depth.assign(n, 0.0); opacity.assign(n, 0.0);
    uncertainty.assign(n, 0.0); final_t.assign(n, 1.0); dom_w.assign(n, 0.0);
    median_valid.assign(n, 0); count.assign(n, 0);
    has_uncertainty = false;
  }
};
struct Record {
  int width = 0, height = 0, num_primitives = 0;
  std::vector<uint32_t> row_start;
  std::vector<int32_t> prim;
  std::vector<double> alpha, transmittance;
  std::vector<int32_t> dominant, median_prim;
  std::vector<uint8_t> visible;
};

// rasterizer.cpp:34-44
void validate_primitives(const std::vector<Prim>& prims, int64_t* bad_index = nullptr) {
  for (size_t i = 0; i < prims.size(); ++i) {
    const Prim& p = prims[i];
    bool ok = finite3(p.mean) && finite3(p.log_scale) && std::isfinite(p.quat[0]) &&
              std::isfinite(p.quat[1]) && std::isfinite(p.quat[2]) && std::isfinite(p.quat[3]) &&
              std::isfinite(p.opacity_logit) && p.qnorm() > 1e-12;
    for (const V3& c : p.sh) ok = ok && finite3(c);
    if (!ok) {
      if (bad_index) *bad_index = static_cast<int64_t>(i);
      throw std::invalid_argument("render: primitive " + std::to_string(i) + " has non-finite parameters");
    }
  }
}

// rasterizer.cpp:46-67
std::vector<PrimCache> project_all(const std::vector<Prim>& prims, const Pose& pose,
                                   const gsf_intrinsics& k, const gsf_raster_cfg& cfg) {
  std::vector<PrimCache> cache(prims.size());
  const V3 cam_center = pose.center();
  const M3 w = pose.rotation();
  parallel_for(prims.size(), [&](size_t lo_i, size_t hi_i) {
  for (size_t i = lo_i; i < hi_i; ++i) {
    const Prim& p = prims[i];
    PrimCache& c = cache[i];
    const double support = cfg.footprint_sigma * std::exp(std::max({p.log_scale[0], p.log_scale[1], p.log_scale[2]}));
    c.proj = project_gaussian(p.mean, p.covariance(), w, pose.trans, k, cfg.dilation, cfg.footprint_sigma, support);
    if (!c.proj.visible) continue;
    c.sigma = p.opacity();
    V3 dir = p.mean - cam_center;
    const double len = norm(dir);
    dir = len > 1e-12 ? dir / len : V3(0, 0, 1);
    c.color = p.sh.empty() ? V3(0.5, 0.5, 0.5) : eval_sh_color(p.sh, dir);
  }
  });
  return cache;
}

// rasterizer.cpp:69-79
std::vector<int32_t> sorted_visible(const std::vector<PrimCache>& cache) {
  std::vector<int32_t> ids;
  for (size_t i = 0; i < cache.size(); ++i)
    if (cache[i].proj.visible) ids.push_back(static_cast<int32_t>(i));
  std::sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
    const double da = cache[a].proj.depth, db = cache[b].proj.depth;
    return da < db || (da == db && a < b);
  });
  return ids;
}

struct PixelResult {
  V3 color;
  double alpha_depth = 0.0, opacity = 0.0, uncertainty = 0.0, final_t = 1.0, median_depth = 0.0, best = 0.0;
  int32_t median_prim = -1, dominant = -1, count = 0;
};

// rasterizer.cpp:96-140
void blend_pixel(double px, double py, const int32_t* ids, size_t n, const std::vector<PrimCache>& cache,
                 double obs_depth, bool obs_valid, const gsf_raster_cfg& cfg, bool allow_termination,
                 PixelResult& r, std::vector<Contrib>* contribs) {
  const double cutoff = cfg.footprint_sigma * cfg.footprint_sigma;
  double t = 1.0;
  double best_weight = 0.0;
  for (size_t s = 0; s < n; ++s) {
    const int32_t id = ids[s];
    const PrimCache& c = cache[id];
    const double dx = px - c.proj.mean2d.x;
    const double dy = py - c.proj.mean2d.y;
    const double rho = c.proj.conic.m[0][0] * dx * dx + 2.0 * c.proj.conic.m[0][1] * dx * dy +
                       c.proj.conic.m[1][1] * dy * dy;
    if (rho > cutoff || rho < 0.0) continue;
    const double g = std::exp(-0.5 * rho);
    const double raw_alpha = c.sigma * g;
    if (raw_alpha < cfg.alpha_skip) continue;
    const double alpha = std::min(raw_alpha, cfg.alpha_clamp);
    const double w = alpha * t;
    r.color += w * c.color;
    r.alpha_depth += w * c.proj.depth;
    r.opacity += w;
    if (obs_valid) {
      const double e = c.proj.depth - obs_depth;
      r.uncertainty += w * e * e;
    }
    if (w > best_weight) {
      best_weight = w;
      r.dominant = id;
    }
    if (contribs) contribs->push_back({id, alpha, t});
    ++r.count;
    const double t_next = t * (1.0 - alpha);
    if (r.median_prim < 0 && t >= 0.5 && t_next < 0.5) {
      r.median_prim = id;
      r.median_depth = c.proj.depth;
    }
    t = t_next;
    if (allow_termination && t < cfg.termination_threshold) break;
  }
  r.final_t = t;
  r.best = best_weight;
}

inline bool depth_sample_valid(double d, const gsf_intrinsics& k) {
  return std::isfinite(d) && d > k.near_plane && d < k.far_plane;
}

void store_pixel(const PixelResult& r, size_t i, RenderOut& out, Record* rec) {
  out.color[i] = r.color;
  out.alpha_depth[i] = r.alpha_depth;
  out.median_depth[i] = r.median_depth;
  out.median_valid[i] = r.median_prim >= 0 ? 1 : 0;
  out.opacity[i] = r.opacity;
  out.uncertainty[i] = r.uncertainty;
  out.final_t[i] = r.final_t;
  out.count[i] = r.count;
  out.dom_w[i] = r.best;
  if (rec) {
    rec->dominant[i] = r.dominant;
    rec->median_prim[i] = r.median_prim;
  }
}

struct Result {
  RenderOut out;
  Record record;
};

// rasterizer.cpp:168-261 (render) and :263-296 (render_reference)
Result render(const std::vector<Prim>& prims, const Pose& pose, const gsf_intrinsics& k,
              const double* obs, const gsf_raster_cfg& cfg, bool brute_force) {
  validate_intrinsics(k);
  validate_primitives(prims);
  const int w = k.width, h = k.height;
  Result res;
  RenderOut& out = res.out;
  Record& rec = res.record;
  out.init(w, h);
  out.has_uncertainty = obs != nullptr;
  rec.width = w;
  rec.height = h;
  rec.num_primitives = static_cast<int>(prims.size());
  rec.dominant.assign(static_cast<size_t>(w) * h, -1);
  rec.median_prim.assign(static_cast<size_t>(w) * h, -1);
  rec.visible.assign(prims.size(), 0);

  const std::vector<PrimCache> cache = project_all(prims, pose, k, cfg);
  for (size_t i = 0; i < cache.size(); ++i) rec.visible[i] = cache[i].proj.visible ? 1 : 0;
  const std::vector<int32_t> sorted = sorted_visible(cache);

  if (brute_force) {
    parallel_for(static_cast<size_t>(h), [&](size_t y_lo, size_t y_hi) {
    for (int y = static_cast<int>(y_lo); y < static_cast<int>(y_hi); ++y)
      for (int x = 0; x < w; ++x) {
        const size_t i = static_cast<size_t>(y) * w + x;
        PixelResult r;
        double obs_d = 0.0;
        bool obs_ok = false;
        if (obs) { obs_d = obs[i]; obs_ok = depth_sample_valid(obs_d, k); }
        blend_pixel(x + 0.5, y + 0.5, sorted.data(), sorted.size(), cache, obs_d, obs_ok, cfg, false, r, nullptr);
        store_pixel(r, i, out, &rec);
      }
    });
    rec.row_start.assign(static_cast<size_t>(w) * h + 1, 0);
    return res;
  }

  const int ts = cfg.tile_size;
  const int tiles_x = (w + ts - 1) / ts;
  const int tiles_y = (h + ts - 1) / ts;
  std::vector<std::vector<int32_t>> tile_lists(static_cast<size_t>(tiles_x) * tiles_y);
  auto tclamp = [](double v, int hi) {
    const double f = std::floor(v);
    if (f < 0.0) return 0;
    if (f > hi) return hi;
    return static_cast<int>(f);
  };
  for (const int32_t id : sorted) {
    const Proj& p = cache[id].proj;
    const int tx0 = tclamp((p.mean2d.x - p.radius) / ts, tiles_x - 1);
    const int tx1 = tclamp((p.mean2d.x + p.radius) / ts, tiles_x - 1);
    const int ty0 = tclamp((p.mean2d.y - p.radius) / ts, tiles_y - 1);
    const int ty1 = tclamp((p.mean2d.y + p.radius) / ts, tiles_y - 1);
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) tile_lists[static_cast<size_t>(ty) * tiles_x + tx].push_back(id);
  }

  std::vector<std::vector<Contrib>> per_pixel(static_cast<size_t>(w) * h);
  parallel_for(tile_lists.size(), [&](size_t t_lo, size_t t_hi) {
  for (size_t t = t_lo; t < t_hi; ++t) {
    const auto& list = tile_lists[t];
    const int tx = static_cast<int>(t) % tiles_x;
    const int ty = static_cast<int>(t) / tiles_x;
    const int x1 = std::min(w, (tx + 1) * ts);
    const int y1 = std::min(h, (ty + 1) * ts);
    for (int y = ty * ts; y < y1; ++y)
      for (int x = tx * ts; x < x1; ++x) {
        const size_t i = static_cast<size_t>(y) * w + x;
        PixelResult r;
        double obs_d = 0.0;
        bool obs_ok = false;
        if (obs) { obs_d = obs[i]; obs_ok = depth_sample_valid(obs_d, k); }
        blend_pixel(x + 0.5, y + 0.5, list.data(), list.size(), cache, obs_d, obs_ok, cfg, true, r, &per_pixel[i]);
        store_pixel(r, i, out, &rec);
      }
  }
  });
  size_t total = 0;
  rec.row_start.resize(static_cast<size_t>(w) * h + 1);
  for (size_t p = 0; p < per_pixel.size(); ++p) {
    rec.row_start[p] = static_cast<uint32_t>(total);
    total += per_pixel[p].size();
  }
  rec.row_start.back() = static_cast<uint32_t>(total);
  rec.prim.resize(total);
  rec.alpha.resize(total);
  rec.transmittance.resize(total);
  size_t at = 0;
  for (const auto& list : per_pixel)
    for (const Contrib& c : list) {
      rec.prim[at] = c.id;
      rec.alpha[at] = c.alpha;
      rec.transmittance[at] = c.transmittance;
      ++at;
    }
  return res;
}

struct Grads {
  std::vector<V3> d_mean, d_log_scale;
  std::vector<V4> d_quat;
  std::vector<double> d_opacity_logit;
  std::vector<std::vector<V3>> d_sh;
  std::vector<V2> d_mean2d;
  double d_pose[6] = {0, 0, 0, 0, 0, 0};
  void init(const std::vector<Prim>& p) {
    const size_t n = p.size();
    d_mean.assign(n, V3()); d_log_scale.assign(n, V3()); d_quat.assign(n, V4());
    d_opacity_logit.assign(n, 0.0); d_mean2d.assign(n, V2());
    d_sh.resize(n);
    for (size_t i = 0; i < n; ++i) d_sh[i].assign(p[i].sh.size(), V3());
    for (double& v : d_pose) v = 0.0;
  }
  // output.cpp:24-48
  void add(const Grads& o) {
    for (size_t i = 0; i < d_mean.size(); ++i) {
      d_mean[i] += o.d_mean[i];
      d_log_scale[i] += o.d_log_scale[i];
      for (int a = 0; a < 4; ++a) d_quat[i][a] += o.d_quat[i][a];
      d_opacity_logit[i] += o.d_opacity_logit[i];
      d_mean2d[i].x += o.d_mean2d[i].x;
      d_mean2d[i].y += o.d_mean2d[i].y;
      for (size_t j = 0; j < d_sh[i].size(); ++j) d_sh[i][j] += o.d_sh[i][j];
    }
    for (int a = 0; a < 6; ++a) d_pose[a] += o.d_pose[a];
  }
};

struct Upstream {
  std::vector<V3> d_color;
  std::vector<double> d_alpha_depth, d_median_depth, d_opacity, d_uncertainty;
};

struct ScreenGrad {
  V2 d_mean2d;
  double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
  double d_sigma = 0.0;
  V3 d_color;
  double d_depth = 0.0;
  bool zero() const {
    return d_mean2d.x == 0.0 && d_mean2d.y == 0.0 && c00 == 0.0 && c01 == 0.0 && c10 == 0.0 &&
           c11 == 0.0 && d_sigma == 0.0 && zero3(d_color) && d_depth == 0.0;
  }
};

// rasterizer.cpp:320-335
void rotation_quat_jacobians(const V4& q, M3 j[4]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double a[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                          {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                          {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                          {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
  for (int k = 0; k < 4; ++k)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) j[k][r][c] = 2.0 * a[k][3 * r + c];
}

// rasterizer.cpp:339-572
Grads render_backward(const std::vector<Prim>& prims, const Pose& pose, const gsf_intrinsics& k,
                      const Record& rec, const Upstream& up, const double* obs, const gsf_raster_cfg& cfg) {
  validate_intrinsics(k);
  validate_primitives(prims);
  if (rec.num_primitives != static_cast<int>(prims.size()))
    throw std::invalid_argument("render_backward: record does not match the primitive list");
  if (rec.width != k.width || rec.height != k.height)
    throw std::invalid_argument("render_backward: record dimensions do not match intrinsics");
  const int w = k.width, h = k.height;
  const bool use_color = !up.d_color.empty();
  const bool use_adepth = !up.d_alpha_depth.empty();
  const bool use_mdepth = !up.d_median_depth.empty();
  const bool use_opacity = !up.d_opacity.empty();
  const bool use_uncert = !up.d_uncertainty.empty() && cfg.uncertainty_full_gradient;
  if (use_uncert && !obs) throw std::invalid_argument("render_backward: uncertainty gradient needs observed depth");
  Grads bundle;
  bundle.init(prims);
  if (!(use_color || use_adepth || use_mdepth || use_opacity || use_uncert)) return bundle;

  const std::vector<PrimCache> cache = project_all(prims, pose, k, cfg);
  const int ts = cfg.tile_size;
  const int tiles_x = (w + ts - 1) / ts;
  const int tiles_y = (h + ts - 1) / ts;
  const size_t n_tiles = static_cast<size_t>(tiles_x) * tiles_y;
  struct TileGrads { std::vector<int32_t> ids; std::vector<ScreenGrad> grads; };
  std::vector<TileGrads> tiles(n_tiles);
  parallel_for(n_tiles, [&](size_t t_lo, size_t t_hi) {
  std::vector<int32_t> slot_of(prims.size(), -1);  // per thread, reset after every tile
  for (size_t t = t_lo; t < t_hi; ++t) {
    TileGrads& tg = tiles[t];
    const int tx = static_cast<int>(t) % tiles_x;
    const int ty = static_cast<int>(t) / tiles_x;
    const int x1 = std::min(w, (tx + 1) * ts);
    const int y1 = std::min(h, (ty + 1) * ts);
    for (int y = ty * ts; y < y1; ++y)
      for (int x = tx * ts; x < x1; ++x) {
        const size_t pi = static_cast<size_t>(y) * w + x;
        const uint32_t lo_e = rec.row_start[pi], hi_e = rec.row_start[pi + 1];
        if (lo_e == hi_e) continue;
        const V3 g_color = use_color ? up.d_color[pi] : V3();
        const double g_adepth = use_adepth ? up.d_alpha_depth[pi] : 0.0;
        const double g_opacity = use_opacity ? up.d_opacity[pi] : 0.0;
        double g_mdepth = use_mdepth ? up.d_median_depth[pi] : 0.0;
        double g_uncert = use_uncert ? up.d_uncertainty[pi] : 0.0;
        double obs_d = 0.0;
        if (obs) {
          obs_d = obs[pi];
          if (!depth_sample_valid(obs_d, k)) g_uncert = 0.0;
        } else {
          g_uncert = 0.0;
        }
        const int32_t median_id = rec.median_prim[pi];
        if (median_id < 0) g_mdepth = 0.0;
        if (zero3(g_color) && g_adepth == 0.0 && g_opacity == 0.0 && g_mdepth == 0.0 && g_uncert == 0.0) continue;
        const double px = x + 0.5, py = y + 0.5;
        double suffix = 0.0;
        for (uint32_t e = hi_e; e-- > lo_e;) {
          const int32_t id = rec.prim[e];
          const double alpha = rec.alpha[e];
          const double t_pre = rec.transmittance[e];
          const PrimCache& c = cache[id];
          const double depth_err = c.proj.depth - obs_d;
          const double q = dot(g_color, c.color) + g_adepth * c.proj.depth + g_opacity + g_uncert * depth_err * depth_err;
          const double d_alpha = t_pre * q - suffix / (1.0 - alpha);
          suffix += alpha * t_pre * q;
          int32_t slot = slot_of[id];
          if (slot < 0) {
            slot = static_cast<int32_t>(tg.ids.size());
            slot_of[id] = slot;
            tg.ids.push_back(id);
            tg.grads.emplace_back();
          }
          ScreenGrad& sg = tg.grads[slot];
          const double weight = alpha * t_pre;
          sg.d_color += weight * g_color;
          sg.d_depth += weight * (g_adepth + 2.0 * g_uncert * depth_err);
          if (id == median_id) sg.d_depth += g_mdepth;
          const double dx = px - c.proj.mean2d.x;
          const double dy = py - c.proj.mean2d.y;
          const double rho = c.proj.conic.m[0][0] * dx * dx + 2.0 * c.proj.conic.m[0][1] * dx * dy +
                             c.proj.conic.m[1][1] * dy * dy;
          const double g_val = std::exp(-0.5 * rho);
          if (c.sigma * g_val > cfg.alpha_clamp) continue;
          sg.d_sigma += d_alpha * g_val;
          const double d_g = d_alpha * c.sigma;
          const V2 u(c.proj.conic.m[0][0] * dx + c.proj.conic.m[0][1] * dy,
                     c.proj.conic.m[1][0] * dx + c.proj.conic.m[1][1] * dy);
          sg.d_mean2d.x += g_val * d_g * u.x;
          sg.d_mean2d.y += g_val * d_g * u.y;
          const double f = 0.5 * g_val * d_g;
          sg.c00 += f * (u.x * u.x);
          sg.c01 += f * (u.x * u.y);
          sg.c10 += f * (u.y * u.x);
          sg.c11 += f * (u.y * u.y);
        }
      }
    for (const int32_t id : tg.ids) slot_of[id] = -1;
  }
  });
  std::vector<ScreenGrad> screen(prims.size());
  for (const TileGrads& tg : tiles)
    for (size_t s = 0; s < tg.ids.size(); ++s) {
      ScreenGrad& dst = screen[tg.ids[s]];
      const ScreenGrad& src = tg.grads[s];
      dst.d_mean2d.x += src.d_mean2d.x; dst.d_mean2d.y += src.d_mean2d.y;
      dst.c00 += src.c00; dst.c01 += src.c01; dst.c10 += src.c10; dst.c11 += src.c11;
      dst.d_sigma += src.d_sigma;
      dst.d_color += src.d_color;
      dst.d_depth += src.d_depth;
    }

  const M3 w_rot = pose.rotation();
  const V3 cam_center = pose.center();
  std::vector<std::array<double, 6>> pose_contrib(prims.size(), std::array<double, 6>{0, 0, 0, 0, 0, 0});
  parallel_for(prims.size(), [&](size_t i_lo, size_t i_hi) {
  for (size_t i = i_lo; i < i_hi; ++i) {
    const ScreenGrad& sg = screen[i];
    if (sg.zero()) continue;
    const Prim& p = prims[i];
    double* d_pose = pose_contrib[i].data();
    bundle.d_mean2d[i] = sg.d_mean2d;
    const V3 p_cam = mul(w_rot, p.mean) + pose.trans;
    const M23 jac = projection_jacobian(p_cam, k);
    const M3 rot = p.rotation();
    const V3 s = p.scale();
    M3 rs2;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) rs2[a][b] = rot[a][b] * (s[b] * s[b]);
    const M3 cov_world = mul(rs2, tr(rot));
    const M3 cov_cam = mul(mul(w_rot, cov_world), tr(w_rot));
    // d_cov_cam = J^T d_cov2d J ; d_jac = 2 d_cov2d J cov_cam  (rasterizer.cpp:503-504)
    const double dc[2][2] = {{sg.c00, sg.c01}, {sg.c10, sg.c11}};
    double jtd[3][2];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 2; ++b) jtd[a][b] = jac.m[0][a] * dc[0][b] + jac.m[1][a] * dc[1][b];
    M3 d_cov_cam;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) d_cov_cam[a][b] = jtd[a][0] * jac.m[0][b] + jtd[a][1] * jac.m[1][b];
    M23 dcj;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) dcj.m[a][b] = (2.0 * dc[a][0]) * jac.m[0][b] + (2.0 * dc[a][1]) * jac.m[1][b];
    const M23 d_jac = mul(dcj, cov_cam);
    const double z = p_cam[2], iz2 = 1.0 / (z * z), iz3 = iz2 / z;
    V3 d_p_cam;
    d_p_cam[0] += d_jac.m[0][2] * (-k.fx * iz2);
    d_p_cam[1] += d_jac.m[1][2] * (-k.fy * iz2);
    d_p_cam[2] += d_jac.m[0][0] * (-k.fx * iz2) + d_jac.m[1][1] * (-k.fy * iz2) +
                  d_jac.m[0][2] * (2.0 * k.fx * p_cam[0] * iz3) + d_jac.m[1][2] * (2.0 * k.fy * p_cam[1] * iz3);
    for (int a = 0; a < 3; ++a) d_p_cam[a] += jac.m[0][a] * sg.d_mean2d.x + jac.m[1][a] * sg.d_mean2d.y;
    d_p_cam[2] += sg.d_depth;
    const V3 pc = cross(p_cam, d_p_cam);
    for (int a = 0; a < 3; ++a) { d_pose[a] += pc[a]; d_pose[3 + a] += d_p_cam[a]; }
    for (int j = 0; j < 3; ++j) {
      V3 unit;
      unit[j] = 1.0;
      const M3 e = skew(unit);
      const M3 ev = mul(e, cov_cam), ve = mul(cov_cam, e);
      double sum = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) sum += d_cov_cam[a][b] * (ev[a][b] - ve[a][b]);
      d_pose[j] += sum;
    }
    V3 d_mean = mul(tr(w_rot), d_p_cam);
    const M3 d_cov_world = mul(mul(tr(w_rot), d_cov_cam), w_rot);
    M3 m;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) m[a][b] = rot[a][b] * s[b];
    const M3 d_m = scale(2.0, mul(d_cov_world, m));
    const M3 rtdm = mul(tr(rot), d_m);
    bundle.d_log_scale[i] = V3(rtdm[0][0] * s[0], rtdm[1][1] * s[1], rtdm[2][2] * s[2]);
    M3 d_rot;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) d_rot[a][b] = d_m[a][b] * s[b];
    const V4 qn = p.qn();
    M3 jq[4];
    rotation_quat_jacobians(qn, jq);
    V4 d_qn;
    for (int kq = 0; kq < 4; ++kq) {
      double sum = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) sum += d_rot[a][b] * jq[kq][a][b];
      d_qn[kq] = sum;
    }
    const double qlen = p.qnorm();
    const double qd = qn[0] * d_qn[0] + qn[1] * d_qn[1] + qn[2] * d_qn[2] + qn[3] * d_qn[3];
    for (int a = 0; a < 4; ++a) bundle.d_quat[i][a] = (d_qn[a] - qn[a] * qd) / qlen;
    const double sig = p.opacity();
    bundle.d_opacity_logit[i] = sg.d_sigma * sig * (1.0 - sig);
    if (!p.sh.empty()) {
      V3 dir = p.mean - cam_center;
      const double len = norm(dir);
      if (len > 1e-12) {
        dir = dir / len;
        V3 d_dir;
        eval_sh_color_backward(p.sh, dir, sg.d_color, bundle.d_sh[i], d_dir);
        const V3 through = (d_dir - dot(dir, d_dir) * dir) / len;
        d_mean += through;
        const V3 wt = mul(w_rot, through);
        for (int a = 0; a < 3; ++a) d_pose[3 + a] += wt[a];
      } else {
        V3 d_dir;
        eval_sh_color_backward(p.sh, V3(0, 0, 1), sg.d_color, bundle.d_sh[i], d_dir);
      }
    }
    bundle.d_mean[i] = d_mean;
  }
  });
  // primitive-order pose sum (rasterizer.cpp:570): independent of the thread count
  for (const auto& c : pose_contrib)
    for (int a = 0; a < 6; ++a) bundle.d_pose[a] += c[a];
  return bundle;
}

// ---- losses.cpp ------------------------------------------------------------------------------
inline double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

void validate_weights(const gsf_loss_weights& w) {
  const double all[] = {w.w_color, w.w_ssim, w.w_geo, w.w_align, w.w_iso, w.w_var, w.t_color, w.t_geo};
  for (double v : all)
    if (!(v >= 0.0)) throw std::invalid_argument("loss weights must be non-negative");
  if (!(w.iso_epsilon >= 1.0)) throw std::invalid_argument("iso epsilon must be >= 1");
  if (!(w.opacity_floor >= 0.0 && w.opacity_floor <= 1.0))
    throw std::invalid_argument("opacity floor must lie in [0,1]");
}

struct TrackLoss {
  double color = 0, geo = 0, total = 0;
  int valid_color = 0, valid_geo = 0;
  Upstream up;
};

// losses.cpp:284-339
TrackLoss tracking_loss(const Result& rr, const double* target, const double* obs, const gsf_intrinsics& k,
                        const gsf_loss_weights& w, bool want) {
  validate_weights(w);
  const RenderOut& out = rr.out;
  const size_t n = static_cast<size_t>(out.width) * out.height;
  TrackLoss r;
  std::vector<uint8_t> op(n), geo(n);
  for (size_t i = 0; i < n; ++i) {
    op[i] = out.opacity[i] >= w.opacity_floor ? 1 : 0;
    geo[i] = (op[i] && depth_sample_valid(obs[i], k)) ? 1 : 0;
    r.valid_color += op[i];
    r.valid_geo += geo[i];
  }
  const int hw = static_cast<int>(n);
  const int m_color = w.normalize_by_valid ? r.valid_color : hw;
  const int m_geo = w.normalize_by_valid ? r.valid_geo : hw;
  // color_loss with mask (losses.cpp:58-72), geo_loss (:80-92)
  {
    int valid = 0;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      if (!op[i]) continue;
      ++valid;
      sum += std::abs(out.color[i][0] - target[3 * i]) + std::abs(out.color[i][1] - target[3 * i + 1]) +
             std::abs(out.color[i][2] - target[3 * i + 2]);
    }
    r.color = valid == 0 ? 0.0 : sum / (3.0 * (w.normalize_by_valid ? valid : hw));
  }
  {
    int valid = 0;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      if (!geo[i]) continue;
      ++valid;
      sum += std::abs(out.alpha_depth[i] - obs[i]);
    }
    r.geo = valid == 0 ? 0.0 : sum / (w.normalize_by_valid ? valid : hw);
  }
  r.total = w.t_color * r.color + w.t_geo * r.geo;
  if (!want) return r;
  if (w.t_color > 0.0 && m_color > 0) r.up.d_color.assign(n, V3());
  if (w.t_geo > 0.0 && m_geo > 0) r.up.d_alpha_depth.assign(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    if (!r.up.d_color.empty() && op[i]) {
      const double f = w.t_color / (3.0 * m_color);
      r.up.d_color[i] = V3(f * sgn(out.color[i][0] - target[3 * i]), f * sgn(out.color[i][1] - target[3 * i + 1]),
                           f * sgn(out.color[i][2] - target[3 * i + 2]));
    }
    if (!r.up.d_alpha_depth.empty() && geo[i]) r.up.d_alpha_depth[i] = w.t_geo * sgn(out.alpha_depth[i] - obs[i]) / m_geo;
  }
  return r;
}

// ---- ssim.cpp -----------------------------------------------------------------------------
constexpr int kRadius = 5;
constexpr double kSC1 = 0.01 * 0.01;
constexpr double kSC2 = 0.03 * 0.03;

const std::array<double, 11>& ssim_window() {
  static const auto w = [] {
    std::array<double, 11> a{};
    for (int i = 0; i <= 2 * kRadius; ++i) {
      const double d = i - kRadius;
      a[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    }
    return a;
  }();
  return w;
}
std::vector<double> axis_norms(int n) {
  const auto& w = ssim_window();
  std::vector<double> z(n, 0.0);
  for (int p = 0; p < n; ++p)
    for (int o = -kRadius; o <= kRadius; ++o)
      if (p + o >= 0 && p + o < n) z[p] += w[o + kRadius];
  return z;
}
using Img3 = std::vector<V3>;
Img3 blur(const Img3& in, int w, int h, const std::vector<double>& zx, const std::vector<double>& zy) {
  const auto& k = ssim_window();
  Img3 tmp(in.size()), out(in.size());
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      V3 acc;
      for (int o = -kRadius; o <= kRadius; ++o)
        if (x + o >= 0 && x + o < w) acc += k[o + kRadius] * in[static_cast<size_t>(y) * w + x + o];
      tmp[static_cast<size_t>(y) * w + x] = acc / zx[x];
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      V3 acc;
      for (int o = -kRadius; o <= kRadius; ++o)
        if (y + o >= 0 && y + o < h) acc += k[o + kRadius] * tmp[static_cast<size_t>(y + o) * w + x];
      out[static_cast<size_t>(y) * w + x] = acc / zy[y];
    }
  return out;
}
Img3 blur_adjoint(const Img3& u, int w, int h, const std::vector<double>& zx, const std::vector<double>& zy) {
  const auto& k = ssim_window();
  Img3 tmp(u.size()), out(u.size());
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      V3 acc;
      for (int o = -kRadius; o <= kRadius; ++o)
        if (y + o >= 0 && y + o < h) acc += k[o + kRadius] * (u[static_cast<size_t>(y + o) * w + x] / zy[y + o]);
      tmp[static_cast<size_t>(y) * w + x] = acc;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      V3 acc;
      for (int o = -kRadius; o <= kRadius; ++o)
        if (x + o >= 0 && x + o < w) acc += k[o + kRadius] * (tmp[static_cast<size_t>(y) * w + x + o] / zx[x + o]);
      out[static_cast<size_t>(y) * w + x] = acc;
    }
  return out;
}
struct Partials { V3 d_mu_x, d_ex2, d_exy; };
V3 ssim_value(const V3& mu_x, const V3& mu_y, const V3& ex2, const V3& ey2, const V3& exy, Partials* part) {
  V3 s;
  for (int c = 0; c < 3; ++c) {
    const double mx = mu_x[c], my = mu_y[c];
    const double a1 = 2.0 * mx * my + kSC1;
    const double a2 = 2.0 * (exy[c] - mx * my) + kSC2;
    const double b1 = mx * mx + my * my + kSC1;
    const double b2 = (ex2[c] - mx * mx) + (ey2[c] - my * my) + kSC2;
    const double denom = b1 * b2;
    s[c] = a1 * a2 / denom;
    if (part) {
      const double d_a1 = a2 / denom;
      const double d_a2 = a1 / denom;
      const double d_b1 = -s[c] / b1;
      const double d_b2 = -s[c] / b2;
      part->d_mu_x[c] = 2.0 * my * d_a1 - 2.0 * my * d_a2 + 2.0 * mx * d_b1 - 2.0 * mx * d_b2;
      part->d_ex2[c] = d_b2;
      part->d_exy[c] = 2.0 * d_a2;
    }
  }
  return s;
}
// ssim.cpp:110-187
double ssim_impl(const Img3& x, const Img3& y, int w, int h, Img3* d_x) {
  if (w == 0 || h == 0) throw std::invalid_argument("ssim: empty image");
  const size_t n = x.size();
  if (w < 2 * kRadius + 1 || h < 2 * kRadius + 1) {
    V3 mu_x, mu_y, ex2, ey2, exy;
    for (size_t i = 0; i < n; ++i) {
      mu_x += x[i]; mu_y += y[i];
      ex2 += V3(x[i][0] * x[i][0], x[i][1] * x[i][1], x[i][2] * x[i][2]);
      ey2 += V3(y[i][0] * y[i][0], y[i][1] * y[i][1], y[i][2] * y[i][2]);
      exy += V3(x[i][0] * y[i][0], x[i][1] * y[i][1], x[i][2] * y[i][2]);
    }
    const double inv = 1.0 / double(n);
    mu_x = inv * mu_x; mu_y = inv * mu_y; ex2 = inv * ex2; ey2 = inv * ey2; exy = inv * exy;
    Partials part;
    const V3 s = ssim_value(mu_x, mu_y, ex2, ey2, exy, d_x ? &part : nullptr);
    if (d_x) {
      d_x->assign(n, V3());
      for (size_t i = 0; i < n; ++i) {
        V3 g;
        for (int c = 0; c < 3; ++c) g[c] = part.d_mu_x[c] + 2.0 * part.d_ex2[c] * x[i][c] + part.d_exy[c] * y[i][c];
        (*d_x)[i] = (inv / 3.0) * g;
      }
    }
    return (s[0] + s[1] + s[2]) / 3.0;
  }
  const std::vector<double> zx = axis_norms(w), zy = axis_norms(h);
  const Img3 mu_x = blur(x, w, h, zx, zy), mu_y = blur(y, w, h, zx, zy);
  Img3 xx(n), yy(n), xy(n);
  for (size_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      xx[i][c] = x[i][c] * x[i][c];
      yy[i][c] = y[i][c] * y[i][c];
      xy[i][c] = x[i][c] * y[i][c];
    }
  const Img3 ex2 = blur(xx, w, h, zx, zy), ey2 = blur(yy, w, h, zx, zy), exy = blur(xy, w, h, zx, zy);
  double total = 0.0;
  Img3 u_mu, u_ex2, u_exy;
  if (d_x) { u_mu.assign(n, V3()); u_ex2.assign(n, V3()); u_exy.assign(n, V3()); }
  const double weight = 1.0 / (3.0 * double(n));
  for (size_t i = 0; i < n; ++i) {
    Partials part;
    const V3 s = ssim_value(mu_x[i], mu_y[i], ex2[i], ey2[i], exy[i], d_x ? &part : nullptr);
    total += s[0] + s[1] + s[2];
    if (d_x) {
      u_mu[i] = weight * part.d_mu_x;
      u_ex2[i] = weight * part.d_ex2;
      u_exy[i] = weight * part.d_exy;
    }
  }
  if (d_x) {
    const Img3 a_mu = blur_adjoint(u_mu, w, h, zx, zy);
    const Img3 a_ex2 = blur_adjoint(u_ex2, w, h, zx, zy);
    const Img3 a_exy = blur_adjoint(u_exy, w, h, zx, zy);
    d_x->assign(n, V3());
    for (size_t i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) (*d_x)[i][c] = a_mu[i][c] + 2.0 * a_ex2[i][c] * x[i][c] + a_exy[i][c] * y[i][c];
  }
  return total * weight;
}

struct MapLoss {
  double color = 0, ssim = 0, geo = 0, align = 0, iso = 0, var = 0, total = 0;
  bool any_empty = false;
  Upstream up;
  std::vector<V3> d_ls_direct;
};

// losses.cpp:156-282
MapLoss mapping_loss(const std::vector<Prim>& prims, const Result& rr, const double* target, const double* obs,
                     const gsf_intrinsics& k, const gsf_loss_weights& w, bool want) {
  validate_weights(w);
  const RenderOut& out = rr.out;
  const int width = out.width, height = out.height;
  const size_t n = static_cast<size_t>(width) * height;
  MapLoss r;
  std::vector<uint8_t> op(n), geo(n), align(n), var(n, 0);
  int c_geo = 0, c_align = 0, c_var = 0;
  for (size_t i = 0; i < n; ++i) {
    op[i] = out.opacity[i] >= w.opacity_floor ? 1 : 0;
    geo[i] = (op[i] && depth_sample_valid(obs[i], k)) ? 1 : 0;
    align[i] = (op[i] && out.median_valid[i]) ? 1 : 0;
    if (out.has_uncertainty) var[i] = geo[i];
    c_geo += geo[i]; c_align += align[i]; c_var += var[i];
  }
  const int hw = static_cast<int>(n);
  const int m_geo = w.normalize_by_valid ? c_geo : hw;
  const int m_align = w.normalize_by_valid ? c_align : hw;
  const int m_var = w.normalize_by_valid ? c_var : hw;
  bool warn = false;
  {  // color_loss, unmasked (losses.cpp:187)
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i)
      sum += std::abs(out.color[i][0] - target[3 * i]) + std::abs(out.color[i][1] - target[3 * i + 1]) +
             std::abs(out.color[i][2] - target[3 * i + 2]);
    r.color = n == 0 ? 0.0 : sum / (3.0 * hw);
    if (n == 0) warn = true;
  }
  auto masked_mean = [&](const std::vector<uint8_t>& m, const std::function<double(size_t)>& f) {
    int valid = 0;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      if (!m[i]) continue;
      ++valid;
      sum += f(i);
    }
    if (valid == 0) { warn = true; return 0.0; }
    return sum / (w.normalize_by_valid ? valid : hw);
  };
  r.geo = masked_mean(geo, [&](size_t i) { return std::abs(out.alpha_depth[i] - obs[i]); });
  r.align = masked_mean(align, [&](size_t i) { return std::abs(out.alpha_depth[i] - out.median_depth[i]); });
  if (out.has_uncertainty) r.var = masked_mean(var, [&](size_t i) { return std::abs(out.uncertainty[i]); });
  else { warn = true; r.var = 0.0; }
  Img3 xc(n), yc(n);
  for (size_t i = 0; i < n; ++i) { xc[i] = out.color[i]; yc[i] = V3(target[3 * i], target[3 * i + 1], target[3 * i + 2]); }
  if (w.w_ssim > 0.0 && !want) r.ssim = 1.0 - ssim_impl(xc, yc, width, height, nullptr);
  int iso_count = 0;
  double iso_sum = 0.0;
  std::vector<int> iso_hi(prims.size(), -1), iso_lo(prims.size(), -1);
  std::vector<double> iso_ratio(prims.size(), 0.0);
  for (size_t i = 0; i < prims.size(); ++i) {
    if (!rr.record.visible[i]) continue;
    ++iso_count;
    const V3 s = prims[i].scale();
    int a = 0, b = 0;
    for (int c = 1; c < 3; ++c) { if (s[c] > s[a]) a = c; if (s[c] < s[b]) b = c; }
    iso_hi[i] = a; iso_lo[i] = b;
    iso_ratio[i] = s[a] / s[b];
    iso_sum += std::max(iso_ratio[i], w.iso_epsilon) - w.iso_epsilon;
  }
  r.iso = iso_count == 0 ? 0.0 : iso_sum / iso_count;
  Img3 d_ssim;
  if (w.w_ssim > 0.0 && want) r.ssim = 1.0 - ssim_impl(xc, yc, width, height, &d_ssim);
  r.any_empty = warn;
  r.total = w.w_color * r.color + w.w_ssim * r.ssim + w.w_geo * r.geo + w.w_align * r.align + w.w_iso * r.iso + w.w_var * r.var;
  if (!want) return r;
  Upstream& up = r.up;
  const double c_norm = 3.0 * hw;
  if (w.w_color > 0.0 || w.w_ssim > 0.0) up.d_color.assign(n, V3());
  if (w.w_geo > 0.0 || w.w_align > 0.0) up.d_alpha_depth.assign(n, 0.0);
  if (w.w_align > 0.0) up.d_median_depth.assign(n, 0.0);
  if (w.w_var > 0.0 && out.has_uncertainty && m_var > 0) up.d_uncertainty.assign(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    if (!up.d_color.empty()) {
      V3 g;
      if (w.w_color > 0.0) {
        const double f = w.w_color / c_norm;
        g += V3(f * sgn(out.color[i][0] - target[3 * i]), f * sgn(out.color[i][1] - target[3 * i + 1]),
                f * sgn(out.color[i][2] - target[3 * i + 2]));
      }
      if (w.w_ssim > 0.0) g = g - w.w_ssim * d_ssim[i];
      up.d_color[i] = g;
    }
    if (!up.d_alpha_depth.empty()) {
      double g = 0.0;
      if (w.w_geo > 0.0 && geo[i] && m_geo > 0) g += w.w_geo * sgn(out.alpha_depth[i] - obs[i]) / m_geo;
      if (w.w_align > 0.0 && align[i] && m_align > 0) {
        const double s = sgn(out.alpha_depth[i] - out.median_depth[i]);
        g += w.w_align * s / m_align;
        up.d_median_depth[i] = -w.w_align * s / m_align;
      }
      up.d_alpha_depth[i] = g;
    }
    if (!up.d_uncertainty.empty() && var[i]) up.d_uncertainty[i] = w.w_var / m_var;
  }
  if (w.w_iso > 0.0 && iso_count > 0) {
    r.d_ls_direct.assign(prims.size(), V3());
    for (size_t i = 0; i < prims.size(); ++i) {
      if (iso_hi[i] < 0 || iso_ratio[i] <= w.iso_epsilon) continue;
      const double g = w.w_iso * iso_ratio[i] / iso_count;
      r.d_ls_direct[i][iso_hi[i]] += g;
      r.d_ls_direct[i][iso_lo[i]] -= g;
    }
  }
  return r;
}

// ---- adam.cpp:40-53 -------------------------------------------------------------------------
struct Adam {
  double lr;
  int stride;
  uint64_t t = 0;
  std::vector<double> m, v;
  Adam(double l, int s) : lr(l), stride(s) {
    if (s <= 0) throw std::invalid_argument("optimizer stride must be positive");
    if (!(l >= 0.0)) throw std::invalid_argument("learning rate must be non-negative");
  }
  void append(size_t e) { m.resize(m.size() + e * stride, 0.0); v.resize(v.size() + e * stride, 0.0); }
  void filter(const std::vector<uint8_t>& keep) {
    size_t out = 0;
    for (size_t i = 0; i < keep.size(); ++i) {
      if (!keep[i]) continue;
      for (int a = 0; a < stride; ++a) { m[out * stride + a] = m[i * stride + a]; v[out * stride + a] = v[i * stride + a]; }
      ++out;
    }
    m.resize(out * stride); v.resize(out * stride);
  }
  void step(double* params, const double* grads) {
    ++t;
    const double bc1 = 1.0 - std::pow(0.9, static_cast<double>(t));
    const double bc2 = 1.0 - std::pow(0.999, static_cast<double>(t));
    for (size_t i = 0; i < m.size(); ++i) {
      const double g = grads[i];
      m[i] = 0.9 * m[i] + (1.0 - 0.9) * g;
      v[i] = 0.999 * v[i] + (1.0 - 0.999) * g * g;
      const double m_hat = m[i] / bc1;
      const double v_hat = v[i] / bc2;
      params[i] -= lr * m_hat / (std::sqrt(v_hat) + 1e-8);
    }
  }
};

// mapper.cpp:48-117
struct PrimOpt {
  Adam mean, log_scale, quat, opacity, sh;
  int sh_dim;
  explicit PrimOpt(const gsf_mapper_cfg& c)
      : mean(c.lr_mean * c.scene_extent, 3), log_scale(c.lr_scale, 3), quat(c.lr_rotation, 4),
        opacity(c.lr_opacity, 1), sh(c.lr_sh, 3 * c.sh_coeffs), sh_dim(3 * c.sh_coeffs) {}
  void append(size_t n) { mean.append(n); log_scale.append(n); quat.append(n); opacity.append(n); sh.append(n); }
  void filter(const std::vector<uint8_t>& k) { mean.filter(k); log_scale.filter(k); quat.filter(k); opacity.filter(k); sh.filter(k); }
  size_t entries() const { return mean.m.size() / 3; }
  void step(std::vector<Prim>& prims, const Grads& g) {
    const size_t n = prims.size();
    if (n != entries() || g.d_mean.size() != n) throw std::invalid_argument("optimizer state out of sync with the primitive list");
    std::vector<double> x, gr;
    auto run = [&](Adam& opt, auto gx, auto gg, auto sc) {
      x.assign(n * opt.stride, 0.0);
      gr.assign(n * opt.stride, 0.0);
      for (size_t i = 0; i < n; ++i) { gx(i, &x[i * opt.stride]); gg(i, &gr[i * opt.stride]); }
      opt.step(x.data(), gr.data());
      for (size_t i = 0; i < n; ++i) sc(i, &x[i * opt.stride]);
    };
    run(mean, [&](size_t i, double* o) { for (int a = 0; a < 3; ++a) o[a] = prims[i].mean[a]; },
        [&](size_t i, double* o) { for (int a = 0; a < 3; ++a) o[a] = g.d_mean[i][a]; },
        [&](size_t i, const double* o) { for (int a = 0; a < 3; ++a) prims[i].mean[a] = o[a]; });
    run(log_scale, [&](size_t i, double* o) { for (int a = 0; a < 3; ++a) o[a] = prims[i].log_scale[a]; },
        [&](size_t i, double* o) { for (int a = 0; a < 3; ++a) o[a] = g.d_log_scale[i][a]; },
        [&](size_t i, const double* o) { for (int a = 0; a < 3; ++a) prims[i].log_scale[a] = o[a]; });
    run(quat, [&](size_t i, double* o) { for (int a = 0; a < 4; ++a) o[a] = prims[i].quat[a]; },
        [&](size_t i, double* o) { for (int a = 0; a < 4; ++a) o[a] = g.d_quat[i][a]; },
        [&](size_t i, const double* o) { for (int a = 0; a < 4; ++a) prims[i].quat[a] = o[a]; });
    run(opacity, [&](size_t i, double* o) { o[0] = prims[i].opacity_logit; },
        [&](size_t i, double* o) { o[0] = g.d_opacity_logit[i]; },
        [&](size_t i, const double* o) { prims[i].opacity_logit = o[0]; });
    run(sh, [&](size_t i, double* o) { for (int b = 0; b < sh_dim / 3; ++b) for (int c = 0; c < 3; ++c) o[3 * b + c] = prims[i].sh[b][c]; },
        [&](size_t i, double* o) { for (int b = 0; b < sh_dim / 3; ++b) for (int c = 0; c < 3; ++c) o[3 * b + c] = g.d_sh[i][b][c]; },
        [&](size_t i, const double* o) { for (int b = 0; b < sh_dim / 3; ++b) for (int c = 0; c < 3; ++c) prims[i].sh[b][c] = o[3 * b + c]; });
  }
};

Upstream to_upstream(const orc_upstream* up, size_t n) {
  Upstream u;
  if (!up) return u;
  if (up->d_color) { u.d_color.resize(n); for (size_t i = 0; i < n; ++i) u.d_color[i] = V3(up->d_color[3 * i], up->d_color[3 * i + 1], up->d_color[3 * i + 2]); }
  if (up->d_alpha_depth) u.d_alpha_depth.assign(up->d_alpha_depth, up->d_alpha_depth + n);
  if (up->d_median_depth) u.d_median_depth.assign(up->d_median_depth, up->d_median_depth + n);
  if (up->d_opacity) u.d_opacity.assign(up->d_opacity, up->d_opacity + n);
  if (up->d_uncertainty) u.d_uncertainty.assign(up->d_uncertainty, up->d_uncertainty + n);
  return u;
}

}  // namespace

struct orc_result {
  Result r;
};

struct orc_mapstate {
  std::vector<Prim> prims;
  PrimOpt opt;
  int iteration = 0;
  std::vector<double> grad_accum;
  std::vector<int> grad_count;
  std::mt19937_64 rng;
  explicit orc_mapstate(const gsf_mapper_cfg& c) : opt(c), rng(c.seed) {}
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GSF_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return std::string(e.what()).find("non-finite") != std::string::npos ? GSF_ENONFINITE : GSF_EINVAL;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return GSF_EDIVERGED;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GSF_EINVAL;
  }
}

void export_grads(const Grads& g, int K, orc_grads* out) {
  for (size_t i = 0; i < g.d_mean.size(); ++i) {
    if (out->d_mean) for (int a = 0; a < 3; ++a) out->d_mean[3 * i + a] = g.d_mean[i][a];
    if (out->d_log_scale) for (int a = 0; a < 3; ++a) out->d_log_scale[3 * i + a] = g.d_log_scale[i][a];
    if (out->d_quat) for (int a = 0; a < 4; ++a) out->d_quat[4 * i + a] = g.d_quat[i][a];
    if (out->d_opacity_logit) out->d_opacity_logit[i] = g.d_opacity_logit[i];
    if (out->d_sh)
      for (int b = 0; b < K; ++b)
        for (int c = 0; c < 3; ++c) out->d_sh[3 * K * i + 3 * b + c] = b < static_cast<int>(g.d_sh[i].size()) ? g.d_sh[i][b][c] : 0.0;
    if (out->d_mean2d) { out->d_mean2d[2 * i] = g.d_mean2d[i].x; out->d_mean2d[2 * i + 1] = g.d_mean2d[i].y; }
  }
  for (int a = 0; a < 6; ++a) out->d_pose[a] = g.d_pose[a];
}

// gradcheck.cpp:8-19
uint64_t fingerprint_record(const Record& rec, double alpha_clamp) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto fold = [&](uint64_t v) { h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); };
  for (const uint32_t v : rec.row_start) fold(v);
  for (size_t i = 0; i < rec.prim.size(); ++i) {
    fold(static_cast<uint64_t>(rec.prim[i]));
    fold(rec.alpha[i] >= alpha_clamp ? 1 : 0);
  }
  for (const int32_t m : rec.median_prim) fold(static_cast<uint64_t>(static_cast<int64_t>(m)));
  for (const uint8_t v : rec.visible) fold(v);
  return h;
}

struct DensifyCounts {
  int split, cloned, removed;
};

// mapper.cpp:172-230
DensifyCounts densify_and_cull(orc_mapstate& st, const gsf_mapper_cfg& cfg) {
  const size_t n = st.prims.size();
  const double size_boundary = cfg.densify_size_fraction * cfg.scene_extent;
  std::vector<uint8_t> keep(n, 1);
  std::vector<Prim> appended;
  int removed = 0, split = 0, cloned = 0;
  for (size_t i = 0; i < n; ++i) {
    const Prim& p = st.prims[i];
    if (p.opacity() < cfg.densify_cull_opacity) { keep[i] = 0; ++removed; continue; }
    if (st.grad_count[i] == 0) continue;
    const double mean_grad = st.grad_accum[i] / st.grad_count[i];
    if (mean_grad <= cfg.densify_grad_threshold) continue;
    const V3 s = p.scale();
    if (std::max({s[0], s[1], s[2]}) > size_boundary) {
      keep[i] = 0;
      ++split;
      std::normal_distribution<double> gauss(0.0, 1.0);
      const M3 rot = p.rotation();
      for (int child = 0; child < 2; ++child) {
        Prim c = p;
        const V3 z(gauss(st.rng), gauss(st.rng), gauss(st.rng));
        V3 bz;
        for (int a = 0; a < 3; ++a) bz[a] = rot[a][0] * s[0] * z[0] + rot[a][1] * s[1] * z[1] + rot[a][2] * s[2] * z[2];
        c.mean = p.mean + bz;
        const double ls = std::log(cfg.densify_split_factor);
        c.log_scale = p.log_scale - V3(ls, ls, ls);
        appended.push_back(c);
      }
    } else {
      ++cloned;
      appended.push_back(p);
    }
  }
  if (removed == 0 && split == 0 && cloned == 0) {
    st.grad_accum.assign(n, 0.0);
    st.grad_count.assign(n, 0);
    return DensifyCounts{0, 0, 0};
  }
  std::vector<Prim> next;
  for (size_t i = 0; i < n; ++i)
    if (keep[i]) next.push_back(st.prims[i]);
  next.insert(next.end(), appended.begin(), appended.end());
  st.opt.filter(keep);
  st.opt.append(appended.size());
  st.prims = std::move(next);
  st.grad_accum.assign(st.prims.size(), 0.0);
  st.grad_count.assign(st.prims.size(), 0);
  return DensifyCounts{split, cloned, removed};
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_threads(void) { return oracle_threads(); }

int orc_render(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
               const double* observed_depth, const gsf_raster_cfg* cfg, int brute_force, orc_result** out) {
  return guarded([&] {
    const std::vector<Prim> prims = load_map(map);
    auto* res = new orc_result;
    try {
      res->r = render(prims, to_pose(pose), *K, observed_depth, *cfg, brute_force != 0);
    } catch (...) {
      delete res;
      throw;
    }
    *out = res;
  });
}

void orc_result_free(orc_result* r) { delete r; }

int orc_result_maps(const orc_result* res, orc_maps* o) {
  const RenderOut& out = res->r.out;
  const Record& rec = res->r.record;
  const size_t n = static_cast<size_t>(out.width) * out.height;
  for (size_t i = 0; i < n; ++i) {
    if (o->color) for (int c = 0; c < 3; ++c) o->color[3 * i + c] = out.color[i][c];
    if (o->alpha_depth) o->alpha_depth[i] = out.alpha_depth[i];
    if (o->median_depth) o->median_depth[i] = out.median_depth[i];
    if (o->median_valid) o->median_valid[i] = out.median_valid[i];
    if (o->opacity) o->opacity[i] = out.opacity[i];
    if (o->uncertainty) o->uncertainty[i] = out.uncertainty[i];
    if (o->final_transmittance) o->final_transmittance[i] = out.final_t[i];
    if (o->per_pixel_count) o->per_pixel_count[i] = out.count[i];
    if (o->dominant) o->dominant[i] = rec.dominant[i];
    if (o->median_prim) o->median_prim[i] = rec.median_prim[i];
    if (o->dominant_weight) o->dominant_weight[i] = out.dom_w[i];
  }
  if (o->visible) for (size_t i = 0; i < rec.visible.size(); ++i) o->visible[i] = rec.visible[i];
  o->has_uncertainty = out.has_uncertainty ? 1 : 0;
  return GSF_OK;
}

int64_t orc_result_record_total(const orc_result* r) { return static_cast<int64_t>(r->r.record.prim.size()); }

int orc_result_record(const orc_result* res, uint32_t* row_start, int32_t* prim, double* alpha, double* transmittance) {
  const Record& rec = res->r.record;
  if (row_start) std::memcpy(row_start, rec.row_start.data(), rec.row_start.size() * sizeof(uint32_t));
  if (prim) std::memcpy(prim, rec.prim.data(), rec.prim.size() * sizeof(int32_t));
  if (alpha) std::memcpy(alpha, rec.alpha.data(), rec.alpha.size() * sizeof(double));
  if (transmittance) std::memcpy(transmittance, rec.transmittance.data(), rec.transmittance.size() * sizeof(double));
  return GSF_OK;
}

int orc_render_backward(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K, const orc_result* r,
                        const orc_upstream* up, const double* observed_depth, const gsf_raster_cfg* cfg, orc_grads* out) {
  return guarded([&] {
    const std::vector<Prim> prims = load_map(map);
    const size_t n = static_cast<size_t>(K->width) * K->height;
    const Grads g = render_backward(prims, to_pose(pose), *K, r->r.record, to_upstream(up, n), observed_depth, *cfg);
    export_grads(g, map->sh_coeffs, out);
  });
}

int orc_tracking_loss(const orc_result* r, const double* target, const double* obs, const gsf_intrinsics* K,
                      const gsf_loss_weights* w, gsf_loss_terms* out, double* d_color, double* d_alpha_depth) {
  return guarded([&] {
    const TrackLoss l = tracking_loss(r->r, target, obs, *K, *w, true);
    *out = gsf_loss_terms{};
    out->color = l.color; out->geo = l.geo; out->total = l.total;
    out->valid_color = l.valid_color; out->valid_geo = l.valid_geo;
    const size_t n = static_cast<size_t>(K->width) * K->height;
    for (size_t i = 0; i < n; ++i) {
      if (d_color) for (int c = 0; c < 3; ++c) d_color[3 * i + c] = l.up.d_color.empty() ? 0.0 : l.up.d_color[i][c];
      if (d_alpha_depth) d_alpha_depth[i] = l.up.d_alpha_depth.empty() ? 0.0 : l.up.d_alpha_depth[i];
    }
  });
}

int orc_mapping_loss(const gsf_map_host* map, const orc_result* r, const double* target, const double* obs,
                     const gsf_intrinsics* K, const gsf_loss_weights* w, gsf_loss_terms* out, double* d_color,
                     double* d_alpha_depth, double* d_median_depth, double* d_uncertainty, double* d_ls_direct) {
  return guarded([&] {
    const std::vector<Prim> prims = load_map(map);
    const MapLoss l = mapping_loss(prims, r->r, target, obs, *K, *w, true);
    *out = gsf_loss_terms{};
    out->color = l.color; out->ssim = l.ssim; out->geo = l.geo; out->align = l.align; out->iso = l.iso;
    out->var = l.var; out->total = l.total; out->any_empty_mask = l.any_empty ? 1 : 0;
    const size_t n = static_cast<size_t>(K->width) * K->height;
    for (size_t i = 0; i < n; ++i) {
      if (d_color) for (int c = 0; c < 3; ++c) d_color[3 * i + c] = l.up.d_color.empty() ? 0.0 : l.up.d_color[i][c];
      if (d_alpha_depth) d_alpha_depth[i] = l.up.d_alpha_depth.empty() ? 0.0 : l.up.d_alpha_depth[i];
      if (d_median_depth) d_median_depth[i] = l.up.d_median_depth.empty() ? 0.0 : l.up.d_median_depth[i];
      if (d_uncertainty) d_uncertainty[i] = l.up.d_uncertainty.empty() ? 0.0 : l.up.d_uncertainty[i];
    }
    if (d_ls_direct)
      for (size_t i = 0; i < prims.size(); ++i)
        for (int a = 0; a < 3; ++a) d_ls_direct[3 * i + a] = l.d_ls_direct.empty() ? 0.0 : l.d_ls_direct[i][a];
  });
}

int orc_ssim(const double* x, const double* y, int w, int h, double* value, double* d_x) {
  return guarded([&] {
    const size_t n = static_cast<size_t>(w) * h;
    Img3 xi(n), yi(n);
    for (size_t i = 0; i < n; ++i) {
      xi[i] = V3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
      yi[i] = V3(y[3 * i], y[3 * i + 1], y[3 * i + 2]);
    }
    Img3 g;
    *value = ssim_impl(xi, yi, w, h, d_x ? &g : nullptr);
    if (d_x)
      for (size_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) d_x[3 * i + c] = g[i][c];
  });
}

void orc_adam_step(double* params, const double* grads, double* m, double* v, int64_t n, uint64_t* t, double lr,
                   double beta1, double beta2, double eps) {
  ++*t;
  const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(*t));
  const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(*t));
  for (int64_t i = 0; i < n; ++i) {
    const double g = grads[i];
    m[i] = beta1 * m[i] + (1.0 - beta1) * g;
    v[i] = beta2 * v[i] + (1.0 - beta2) * g * g;
    params[i] -= lr * (m[i] / bc1) / (std::sqrt(v[i] / bc2) + eps);
  }
}

// tracker.cpp:30-84
int orc_track_frame(const gsf_map_host* map, const double* rgb, const double* depth, const gsf_pose* initial,
                    const gsf_intrinsics* K, const gsf_tracker_cfg* cfg, const gsf_loss_weights* w,
                    const gsf_raster_cfg* raster, gsf_track_result* out) {
  return guarded([&] {
    const std::vector<Prim> prims = load_map(map);
    Pose pose = to_pose(initial);
    *out = gsf_track_result{};
    Adam rot_opt(cfg->lr_rotation, 3), trans_opt(cfg->lr_translation, 3);
    rot_opt.append(1);
    trans_opt.append(1);
    double initial_loss = 0.0;
    for (int it = 0; it < cfg->iterations; ++it) {
      const Result rr = render(prims, pose, *K, nullptr, *raster, false);
      const TrackLoss loss = tracking_loss(rr, rgb, depth, *K, *w, true);
      if (it == 0) {
        initial_loss = loss.total;
        out->initial_loss = initial_loss;
        if (loss.valid_color == 0 && loss.valid_geo == 0) {
          out->degraded = 1;
          out->final_loss = loss.total;
          from_pose(pose, &out->pose);
          return;
        }
      }
      if (!std::isfinite(loss.total)) {
        std::ostringstream msg;
        msg << "tracking diverged at iteration " << it << ": total=" << loss.total << " color=" << loss.color
            << " geo=" << loss.geo;
        throw std::runtime_error(msg.str());
      }
      const Grads g = render_backward(prims, pose, *K, rr.record, loss.up, nullptr, *raster);
      double step_rot[3] = {0, 0, 0}, step_trans[3] = {0, 0, 0};
      rot_opt.step(step_rot, &g.d_pose[0]);
      trans_opt.step(step_trans, &g.d_pose[3]);
      const double delta[6] = {step_rot[0], step_rot[1], step_rot[2], step_trans[0], step_trans[1], step_trans[2]};
      pose = pose.perturbed(delta);
      ++out->iterations_run;
    }
    const Result rr = render(prims, pose, *K, nullptr, *raster, false);
    const TrackLoss fin = tracking_loss(rr, rgb, depth, *K, *w, false);
    out->final_loss = fin.total;
    if (cfg->iterations == 0) out->degraded = (fin.valid_color == 0 && fin.valid_geo == 0) ? 1 : 0;
    else if (fin.total > cfg->degraded_loss_ratio * initial_loss) out->degraded = 1;
    from_pose(pose, &out->pose);
  });
}

int orc_mapstate_create(const gsf_map_host* map, const gsf_mapper_cfg* mcfg, orc_mapstate** out) {
  return guarded([&] {
    auto* s = new orc_mapstate(*mcfg);
    s->prims = load_map(map);
    s->opt.append(s->prims.size());
    s->grad_accum.assign(s->prims.size(), 0.0);
    s->grad_count.assign(s->prims.size(), 0);
    *out = s;
  });
}
void orc_mapstate_free(orc_mapstate* s) { delete s; }
int64_t orc_mapstate_count(const orc_mapstate* s) { return static_cast<int64_t>(s->prims.size()); }
int orc_mapstate_get(const orc_mapstate* s, gsf_map_host* out) {
  if (out->count != static_cast<int64_t>(s->prims.size())) { g_err = "count mismatch"; return GSF_EINVAL; }
  store_map(s->prims, out);
  return GSF_OK;
}

// Overwrite the primitives of a MapState (same count): what accumulate_uncertainty / prune_unreliable
// do to MapState::primitives in place (system.cpp:130-132).
int orc_mapstate_put(orc_mapstate* s, const gsf_map_host* map) {
  return guarded([&] {
    if (map->count != static_cast<int64_t>(s->prims.size())) throw std::invalid_argument("count mismatch");
    s->prims = load_map(map);
  });
}

// spawn_gaussians' tail (mapper.cpp:163-169): append primitives, zero Adam moments and statistics.
int orc_mapstate_append(orc_mapstate* s, const gsf_map_host* map) {
  return guarded([&] {
    const std::vector<Prim> add = load_map(map);
    s->prims.insert(s->prims.end(), add.begin(), add.end());
    s->opt.append(add.size());
    s->grad_accum.resize(s->prims.size(), 0.0);
    s->grad_count.resize(s->prims.size(), 0);
  });
}

// mapper.cpp:232-281
int orc_map_step(orc_mapstate* st, int n, const double* const* rgbs, const double* const* depths, const gsf_pose* poses,
                 const gsf_intrinsics* K, const gsf_mapper_cfg* cfg, int iterations, double* trace) {
  return guarded([&] {
    if (n <= 0) throw std::invalid_argument("mapping window is empty");
    for (int i = 0; i < n; ++i)
      if (!rgbs[i] || !depths[i]) throw std::invalid_argument("mapping window observation missing rgb or depth");
    for (int it = 0; it < iterations; ++it) {
      const int o = it % n;
      const Pose pose = to_pose(&poses[o]);
      const Result rr = render(st->prims, pose, *K, depths[o], cfg->raster, false);
      const MapLoss loss = mapping_loss(st->prims, rr, rgbs[o], depths[o], *K, cfg->weights, true);
      if (!std::isfinite(loss.total)) {
        std::ostringstream msg;
        msg << "mapping diverged at iteration " << st->iteration << ": total=" << loss.total << " color=" << loss.color
            << " ssim=" << loss.ssim << " geo=" << loss.geo << " align=" << loss.align << " iso=" << loss.iso
            << " var=" << loss.var;
        throw std::runtime_error(msg.str());
      }
      Grads g = render_backward(st->prims, pose, *K, rr.record, loss.up, depths[o], cfg->raster);
      for (size_t i = 0; i < loss.d_ls_direct.size(); ++i) g.d_log_scale[i] += loss.d_ls_direct[i];
      for (size_t i = 0; i < st->prims.size(); ++i) {
        if (!rr.record.visible[i]) continue;
        const double nx = g.d_mean2d[i].x * 0.5 * K->width, ny = g.d_mean2d[i].y * 0.5 * K->height;
        st->grad_accum[i] += std::sqrt(nx * nx + ny * ny);
        ++st->grad_count[i];
      }
      st->opt.step(st->prims, g);
      ++st->iteration;
      if (trace) trace[it] = loss.total;
      if (cfg->densify_interval > 0 && st->iteration % cfg->densify_interval == 0) densify_and_cull(*st, *cfg);
    }
  });
}

// tracker.cpp:119-183
int orc_sliding_ba(orc_mapstate* st, int n, const double* const* rgbs, const double* const* depths, gsf_pose* poses,
                   const int32_t* frame_ids, const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg,
                   const gsf_mapper_cfg* mcfg, int iterations, double* trace) {
  return guarded([&] {
    if (n <= 0) throw std::invalid_argument("adjustment window is empty");
    int anchor = -1;
    if (tcfg->freeze_oldest_pose) {
      anchor = 0;
      for (int i = 1; i < n; ++i)
        if (frame_ids[i] < frame_ids[anchor]) anchor = i;
    }
    std::vector<Adam> rot_opts, trans_opts;
    for (int i = 0; i < n; ++i) {
      rot_opts.emplace_back(tcfg->lr_rotation, 3);
      rot_opts.back().append(1);
      trans_opts.emplace_back(tcfg->lr_translation, 3);
      trans_opts.back().append(1);
    }
    for (int it = 0; it < iterations; ++it) {
      Grads total;
      total.init(st->prims);
      std::vector<std::array<double, 6>> pose_grads(n);
      double loss_sum = 0.0;
      for (int wi = 0; wi < n; ++wi) {
        const Pose pose = to_pose(&poses[wi]);
        const Result rr = render(st->prims, pose, *K, depths[wi], mcfg->raster, false);
        const MapLoss loss = mapping_loss(st->prims, rr, rgbs[wi], depths[wi], *K, mcfg->weights, true);
        if (!std::isfinite(loss.total)) {
          std::ostringstream msg;
          msg << "bundle adjustment diverged at iteration " << it << " keyframe " << frame_ids[wi] << ": total=" << loss.total;
          throw std::runtime_error(msg.str());
        }
        Grads b = render_backward(st->prims, pose, *K, rr.record, loss.up, depths[wi], mcfg->raster);
        for (size_t i = 0; i < loss.d_ls_direct.size(); ++i) b.d_log_scale[i] += loss.d_ls_direct[i];
        for (int a = 0; a < 6; ++a) pose_grads[wi][a] = b.d_pose[a];
        total.add(b);
        loss_sum += loss.total;
      }
      st->opt.step(st->prims, total);
      for (int wi = 0; wi < n; ++wi) {
        if (wi == anchor) continue;
        double step_rot[3] = {0, 0, 0}, step_trans[3] = {0, 0, 0};
        rot_opts[wi].step(step_rot, &pose_grads[wi][0]);
        trans_opts[wi].step(step_trans, &pose_grads[wi][3]);
        const double delta[6] = {step_rot[0], step_rot[1], step_rot[2], step_trans[0], step_trans[1], step_trans[2]};
        from_pose(to_pose(&poses[wi]).perturbed(delta), &poses[wi]);
      }
      if (trace) trace[it] = loss_sum;
    }
  });
}

// mapper.cpp:12-26 (backprojected_primitive) over the loops of initialize_map (:125-148) and
// spawn_gaussians (:150-170): stride-sampled pixels in row-major order, sensor_valid_mask
// (losses.cpp:141-148), and for spawn rendered.opacity < spawn_opacity_threshold (opacity != NULL).
// Writes the new primitives (capacity out->count) and their number.
int orc_backproject(const double* rgb, const double* depth, const double* opacity, const gsf_pose* pose,
                    const gsf_intrinsics* K, const gsf_mapper_cfg* cfg, int stride, gsf_map_host* out, int64_t* count) {
  return guarded([&] {
    const Pose ps = to_pose(pose);
    const M3 rinv = exp_map(V3(-ps.rot[0], -ps.rot[1], -ps.rot[2]));     // pose.inverse(): exp(-rot)
    const M3 rt = tr(ps.rotation());
    const V3 tinv = -(mul(rt, ps.trans));                                 // -(R^T t)
    const double kC0 = 0.28209479177387814;
    std::vector<Prim> made;
    for (int y = 0; y < K->height; y += stride)
      for (int x = 0; x < K->width; x += stride) {
        const size_t pi = static_cast<size_t>(y) * K->width + x;
        const double d = depth[pi];
        if (!(std::isfinite(d) && d > K->near_plane && d < K->far_plane)) continue;
        if (opacity && opacity[pi] >= cfg->spawn_opacity_threshold) continue;
        Prim p;
        const V3 pc((x + 0.5 - K->cx) / K->fx * d, (y + 0.5 - K->cy) / K->fy * d, d);   // camera.hpp:33-35
        p.mean = mul(rinv, pc) + tinv;
        const double ls = std::log((d / K->fx) * stride * 0.5);
        p.log_scale = V3(ls, ls, ls);
        p.quat = V4(1, 0, 0, 0);
        p.opacity_logit = std::log(cfg->init_opacity / (1.0 - cfg->init_opacity));
        p.sh.assign(cfg->sh_coeffs, V3(0, 0, 0));
        for (int c = 0; c < 3; ++c) p.sh[0][c] = (rgb[3 * pi + c] - 0.5) / kC0;
        p.uncertainty = 0.0;
        p.observed = true;
        made.push_back(p);
      }
    *count = static_cast<int64_t>(made.size());
    if (out && out->mean && static_cast<int64_t>(made.size()) <= out->count) store_map(made, out);
  });
}

int orc_mapstate_set_stats(orc_mapstate* st, const double* accum, const int32_t* count) {
  return guarded([&] {
    for (size_t i = 0; i < st->prims.size(); ++i) { st->grad_accum[i] = accum[i]; st->grad_count[i] = count[i]; }
  });
}

int orc_mapstate_densify(orc_mapstate* st, const gsf_mapper_cfg* cfg, int32_t* change /*split, cloned, removed*/) {
  return guarded([&] {
    const size_t before = st->prims.size();
    (void)before;
    const DensifyCounts c = densify_and_cull(*st, *cfg);
    change[0] = c.split;
    change[1] = c.cloned;
    change[2] = c.removed;
  });
}

// uncertainty.cpp:35-73: per-view (sum, count) partials of Eq. 13 reduced in window order
static void uncertainty_partials(const std::vector<Prim>& prims, int n, const orc_result* const* records,
                                 const double* const* depths, const gsf_pose* poses, const gsf_intrinsics* K,
                                 std::vector<double>& total, std::vector<int>& pixels) {
  const size_t np = prims.size();
  total.assign(np, 0.0);
  pixels.assign(np, 0);
  for (int v = 0; v < n; ++v) {
    const Record& rec = records[v]->r.record;
    if (rec.num_primitives != static_cast<int>(np))
      throw std::invalid_argument("uncertainty view was rendered from a different primitive set");
    const M3 rot = to_pose(&poses[v]).rotation();
    const V3 t = to_pose(&poses[v]).trans;
    std::vector<double> depth_in_view(np);
    for (size_t i = 0; i < np; ++i) depth_in_view[i] = (mul(rot, prims[i].mean) + t)[2];
    std::vector<double> sum(np, 0.0);
    std::vector<int> count(np, 0);
    for (int y = 0; y < rec.height; ++y)
      for (int x = 0; x < rec.width; ++x) {
        const size_t pi = static_cast<size_t>(y) * rec.width + x;
        const int32_t owner = rec.dominant[pi];
        if (owner < 0) continue;
        const double d_obs = depths[v][pi];
        if (!std::isfinite(d_obs) || d_obs <= K->near_plane || d_obs >= K->far_plane) continue;
        for (uint32_t e = rec.row_start[pi]; e < rec.row_start[pi + 1]; ++e) {
          if (rec.prim[e] != owner) continue;
          const double resid = d_obs - depth_in_view[owner];
          sum[owner] += rec.alpha[e] * rec.transmittance[e] * resid * resid;
          ++count[owner];
          break;
        }
      }
    for (size_t i = 0; i < np; ++i) { total[i] += sum[i]; pixels[i] += count[i]; }
  }
}

int orc_uncertainty_partials(const gsf_map_host* map, int n, const orc_result* const* records, const double* const* depths,
                             const gsf_pose* poses, const gsf_intrinsics* K, double* sum_out, int32_t* count_out) {
  return guarded([&] {
    const std::vector<Prim> prims = load_map(map);
    std::vector<double> total;
    std::vector<int> pixels;
    uncertainty_partials(prims, n, records, depths, poses, K, total, pixels);
    for (size_t i = 0; i < prims.size(); ++i) { sum_out[i] = total[i]; count_out[i] = pixels[i]; }
  });
}

// uncertainty.cpp:17-87
int orc_accumulate_uncertainty(gsf_map_host* map, int n, const orc_result* const* records, const double* const* depths,
                               const gsf_pose* poses, const gsf_intrinsics* K, int32_t* observed_count) {
  return guarded([&] {
    *observed_count = 0;
    if (n == 0) return;
    std::vector<Prim> prims = load_map(map);
    const size_t np = prims.size();
    std::vector<double> total;
    std::vector<int> pixels;
    uncertainty_partials(prims, n, records, depths, poses, K, total, pixels);
    int observed = 0;
    for (size_t i = 0; i < np; ++i) {
      if (pixels[i] > 0) {
        prims[i].uncertainty = total[i] / pixels[i];
        prims[i].observed = true;
        ++observed;
      } else {
        prims[i].observed = false;
      }
    }
    *observed_count = observed;
    for (size_t i = 0; i < np; ++i) {
      if (map->uncertainty) map->uncertainty[i] = prims[i].uncertainty;
      if (map->observed) map->observed[i] = prims[i].observed ? 1 : 0;
    }
  });
}

// uncertainty.cpp:89-100
int orc_prune_unreliable(gsf_map_host* map, double tau, double reduced_opacity, int32_t* reduced) {
  return guarded([&] {
    if (!(tau > 0.0)) throw std::invalid_argument("uncertainty threshold must be positive");
    if (!(reduced_opacity > 0.0 && reduced_opacity < 0.1)) throw std::invalid_argument("reduced opacity must lie in (0, 0.1)");
    const double target = logit(reduced_opacity);
    int r = 0;
    for (int64_t i = 0; i < map->count; ++i) {
      const double u = map->uncertainty ? map->uncertainty[i] : 0.0;
      if (u > tau && map->opacity_logit[i] != target) {
        map->opacity_logit[i] = target;
        ++r;
      }
    }
    *reduced = r;
  });
}

// gradcheck.cpp:47-128 with the LinearProbe objective of test_gradients.cpp:17-61
int orc_gradcheck_linear(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K, const gsf_raster_cfg* cfg,
                         const double* obs, const double* a_color, const double* a_depth, const double* a_opacity,
                         const double* a_uncert, const double* a_median, double step, double denom_floor,
                         orc_gradcheck_report* rep) {
  return guarded([&] {
    *rep = orc_gradcheck_report{};
    rep->worst_index = -1;
    const std::vector<Prim> base_prims = load_map(map);
    const Pose base_pose = to_pose(pose);
    const size_t n = static_cast<size_t>(K->width) * K->height;
    auto value = [&](const RenderOut& out) {
      double v = 0.0;
      for (size_t i = 0; i < n; ++i) {
        v += a_color[3 * i] * out.color[i][0] + a_color[3 * i + 1] * out.color[i][1] + a_color[3 * i + 2] * out.color[i][2];
        v += a_depth[i] * out.alpha_depth[i];
        v += a_opacity[i] * out.opacity[i];
        if (a_uncert) v += a_uncert[i] * out.uncertainty[i];
        if (out.median_valid[i]) v += a_median[i] * out.median_depth[i];
      }
      return v;
    };
    struct Ev { double value; uint64_t fp; };
    auto evaluate = [&](const std::vector<Prim>& prims, const Pose& ps) {
      const Result rr = render(prims, ps, *K, obs, *cfg, false);
      return Ev{value(rr.out), fingerprint_record(rr.record, cfg->alpha_clamp)};
    };
    const Result base = render(base_prims, base_pose, *K, obs, *cfg, false);
    Upstream up;
    up.d_color.resize(n);
    for (size_t i = 0; i < n; ++i) up.d_color[i] = V3(a_color[3 * i], a_color[3 * i + 1], a_color[3 * i + 2]);
    up.d_alpha_depth.assign(a_depth, a_depth + n);
    up.d_opacity.assign(a_opacity, a_opacity + n);
    if (a_uncert) up.d_uncertainty.assign(a_uncert, a_uncert + n);
    up.d_median_depth.assign(a_median, a_median + n);
    const Grads an = render_backward(base_prims, base_pose, *K, base.record, up, obs, *cfg);
    int idx = 0;
    auto probe = [&](double analytic, const std::function<void(std::vector<Prim>&, Pose&, double)>& apply) {
      ++rep->total;
      const double offsets[4] = {step, -step, 0.5 * step, -0.5 * step};
      Ev ev[4];
      for (int s = 0; s < 4; ++s) {
        std::vector<Prim> p = base_prims;
        Pose ps = base_pose;
        apply(p, ps, offsets[s]);
        ev[s] = evaluate(p, ps);
      }
      const int my = idx++;
      if (ev[0].fp != ev[1].fp || ev[0].fp != ev[2].fp || ev[0].fp != ev[3].fp) { ++rep->skipped; return; }
      ++rep->checked;
      const double fd = (8.0 * (ev[2].value - ev[3].value) - (ev[0].value - ev[1].value)) / (6.0 * step);
      const double denom = std::max({std::abs(analytic), std::abs(fd), denom_floor});
      const double rel = std::abs(analytic - fd) / denom;
      if (rel > rep->max_rel_err) {
        rep->max_rel_err = rel;
        rep->worst_analytic = analytic;
        rep->worst_fd = fd;
        rep->worst_index = my;
      }
    };
    for (size_t i = 0; i < base_prims.size(); ++i) {
      for (int a = 0; a < 3; ++a) probe(an.d_mean[i][a], [i, a](std::vector<Prim>& g, Pose&, double h) { g[i].mean[a] += h; });
      for (int a = 0; a < 3; ++a) probe(an.d_log_scale[i][a], [i, a](std::vector<Prim>& g, Pose&, double h) { g[i].log_scale[a] += h; });
      for (int a = 0; a < 4; ++a) probe(an.d_quat[i][a], [i, a](std::vector<Prim>& g, Pose&, double h) { g[i].quat[a] += h; });
      probe(an.d_opacity_logit[i], [i](std::vector<Prim>& g, Pose&, double h) { g[i].opacity_logit += h; });
      for (size_t b = 0; b < base_prims[i].sh.size(); ++b)
        for (int c = 0; c < 3; ++c)
          probe(an.d_sh[i][b][c], [i, b, c](std::vector<Prim>& g, Pose&, double h) { g[i].sh[b][c] += h; });
    }
    for (int a = 0; a < 6; ++a)
      probe(an.d_pose[a], [a](std::vector<Prim>&, Pose& ps, double h) {
        double d[6] = {0, 0, 0, 0, 0, 0};
        d[a] = h;
        ps = ps.perturbed(d);
      });
  });
}

// test_utils.hpp:27-53 (argument evaluation order as compiled by the same gcc)
int orc_random_scene(uint32_t seed, int count, int sh_coeffs, double max_opacity, double min_scale, double max_scale,
                     gsf_map_host* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uz(1.2, 5.0);
  std::uniform_real_distribution<double> uxy(-0.4, 0.4);
  std::uniform_real_distribution<double> uls(std::log(min_scale), std::log(max_scale));
  std::uniform_real_distribution<double> uop(0.05, max_opacity);
  std::uniform_real_distribution<double> ush(-0.8, 0.8);
  std::uniform_real_distribution<double> ush_hi(-0.15, 0.15);
  std::normal_distribution<double> n(0.0, 1.0);
  std::vector<Prim> prims(count);
  for (auto& p : prims) {
    const double z = uz(rng);
    p.mean = V3(uxy(rng) * z, uxy(rng) * z, z);
    p.log_scale = V3(uls(rng), uls(rng), uls(rng));
    V4 q(n(rng), n(rng), n(rng), n(rng));
    const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (qn < 1e-3) q = V4(1, 0, 0, 0);
    const double qn2 = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    p.quat = V4(q[0] / qn2, q[1] / qn2, q[2] / qn2, q[3] / qn2);
    p.opacity_logit = logit(uop(rng));
    p.sh.resize(sh_coeffs);
    p.sh[0] = V3(ush(rng), ush(rng), ush(rng));
    for (int b = 1; b < sh_coeffs; ++b) p.sh[b] = V3(ush_hi(rng), ush_hi(rng), ush_hi(rng));
  }
  out->count = count;
  out->sh_coeffs = sh_coeffs;
  if (out->mean) store_map(prims, out);
  return GSF_OK;
}

// test_utils.hpp:56-65
void orc_wavy_depth(int w, int h, double base, int hole_every, double* out) {
  int i = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x, ++i) {
      out[static_cast<size_t>(y) * w + x] = 0.0;
      if (hole_every > 0 && i % hole_every == 3) continue;
      out[static_cast<size_t>(y) * w + x] = base + 0.4 * std::sin(0.31 * x) + 0.3 * std::cos(0.23 * y);
    }
}

void orc_default_raster(gsf_raster_cfg* c) {
  *c = gsf_raster_cfg{0.99, 1.0 / 255.0, 1e-8, 3.0, 0.3, 16, 1, 0};
}
void orc_default_weights(gsf_loss_weights* w, int handheld_real) {
  *w = gsf_loss_weights{0.7, 0.1, 0.25, 0.25, 0.1, 0.15, 0.2, 1.0, 1.0, 0.1, 1};
  if (handheld_real) {  // losses.cpp:35-46
    w->w_color = 1.0; w->w_ssim = 0.1; w->w_geo = 0.8; w->w_align = 0.5; w->w_iso = 0.1; w->w_var = 0.5;
    w->t_color = 1.0; w->t_geo = 0.6;
  }
}
void orc_default_tracker(gsf_tracker_cfg* c) { *c = gsf_tracker_cfg{0.0015, 0.00215, 15, 4, 10, 30, 2, 1, 2.0}; }
void orc_default_mapper(gsf_mapper_cfg* c) {
  *c = gsf_mapper_cfg{};
  c->sh_coeffs = 1;
  c->scene_extent = 4.0;
  c->lr_mean = 1.6e-4;
  c->lr_sh = 2.5e-3;
  c->lr_opacity = 5e-2;
  c->lr_scale = 5e-3;
  c->lr_rotation = 1e-3;
  c->densify_interval = 100;
  c->densify_grad_threshold = 2e-4;
  c->densify_split_factor = 1.6;
  c->densify_size_fraction = 0.01;
  c->densify_cull_opacity = 0.005;
  c->uncertainty_tau = 0.025;
  c->uncertainty_reduced_opacity = 0.005;
  c->seed = 0;
  orc_default_raster(&c->raster);
  orc_default_weights(&c->weights, 0);
  c->init_stride = 2;
  c->spawn_stride = 2;
  c->spawn_opacity_threshold = 0.5;
  c->init_opacity = 0.5;
}

}  // extern "C"
