// integration/rasterizer_b200.cpp — the reference-side drop-in for raster/rasterizer.cpp.
//
// Implements the three functions declared by the reference's own header
// (gsfield/raster/rasterizer.hpp:19-35: render, render_reference, render_backward) on top of the
// C-ABI in include/gsf_cuda.h (libgsf_cuda.so), so a maintainer compiles this file INSTEAD of
// src/raster/rasterizer.cpp and every caller (tracker, mapper, uncertainty, gradcheck, the tests)
// runs on the B200 unchanged.  Nothing here is compute: the host side converts the reference's
// AoS doubles / Image<> containers to the flat fp32 buffers of the C-ABI and back, and repeats the
// reference's argument checks (rasterizer.cpp:339-365) at the boundary so the same
// std::invalid_argument is thrown before any device work.
//
// render_backward accepts ANY BlendRecord produced by render on identical inputs (the reference's
// contract, rasterizer.hpp:29-31), while the device backward is bound to the context's most recent
// render: the drop-in keeps a key of that render (inputs + the record it returned) and re-renders
// first whenever the record handed in is not the latest one.
//
// Built (not shipped) by integration/Makefile against /root/reference/proj/include with
// oracle/eigen_lite standing in for Eigen; integration/_build/ then links the reference's own
// tests/test_rasterizer.cpp and tests/test_gradients.cpp against this file (tests/test_gpu_integration.py).
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gsf_cuda.h"
#include "gsfield/raster/rasterizer.hpp"

namespace gsf {
namespace {

struct DropIn {
  gsf_ctx ctx = nullptr;
  // key of the most recent device render: its inputs and the record it returned
  std::vector<double> key;
  const BlendRecord* record = nullptr;
  ~DropIn() {
    if (ctx) gsf_ctx_destroy(ctx);
  }
};

DropIn& state() {
  thread_local DropIn s;   // one context per host thread, like the reference's per-call state
  if (!s.ctx && gsf_ctx_create(0, &s.ctx) != GSF_OK) throw std::runtime_error("gsf: no CUDA device for the B200 path");
  return s;
}

void raise(int rc) {   // the reference's exception types; messages come from the library
  if (rc == GSF_OK) return;
  const std::string msg = gsf_last_error(state().ctx);
  if (rc == GSF_EINVAL || rc == GSF_ENONFINITE) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

gsf_pose to_pose(const CameraPose& p) {
  return gsf_pose{{p.rotation_tangent.x(), p.rotation_tangent.y(), p.rotation_tangent.z()},
                  {p.translation.x(), p.translation.y(), p.translation.z()}};
}

gsf_intrinsics to_k(const CameraIntrinsics& k) {
  return gsf_intrinsics{k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale, k.near_plane, k.far_plane};
}

gsf_raster_cfg to_cfg(const RasterConfig& c) {
  return gsf_raster_cfg{c.alpha_clamp, c.alpha_skip, c.termination_threshold, c.footprint_sigma, c.dilation,
                        c.tile_size, c.uncertainty_full_gradient ? 1 : 0, c.threads};
}

// std::vector<GaussianPrimitive> -> the device map (every call: the caller may have edited it)
void upload(const std::vector<GaussianPrimitive>& prims, std::vector<double>* key) {
  const size_t P = prims.size();
  const int K = P ? static_cast<int>(prims[0].sh.size()) : 1;
  std::vector<double> mean(3 * P), ls(3 * P), q(4 * P), op(P), sh(3 * static_cast<size_t>(K) * P), nu(P);
  std::vector<uint8_t> obs(P);
  for (size_t i = 0; i < P; ++i) {
    const GaussianPrimitive& p = prims[i];
    if (static_cast<int>(p.sh.size()) != K) throw std::invalid_argument("render: primitives disagree on the SH count");
    for (int a = 0; a < 3; ++a) {
      mean[3 * i + a] = p.mean(a);
      ls[3 * i + a] = p.log_scale(a);
    }
    for (int a = 0; a < 4; ++a) q[4 * i + a] = p.quat(a);
    op[i] = p.opacity_logit;
    for (int c = 0; c < K; ++c)
      for (int a = 0; a < 3; ++a) sh[(i * K + c) * 3 + a] = p.sh[c](a);
    nu[i] = p.uncertainty;
    obs[i] = p.observed ? 1 : 0;
  }
  gsf_map_host m{static_cast<int64_t>(P), K, mean.data(), ls.data(), q.data(), op.data(), sh.data(), nu.data(), obs.data()};
  raise(gsf_map_upload(state().ctx, &m));
  if (key) {
    key->insert(key->end(), mean.begin(), mean.end());
    key->insert(key->end(), ls.begin(), ls.end());
    key->insert(key->end(), q.begin(), q.end());
    key->insert(key->end(), op.begin(), op.end());
    key->insert(key->end(), sh.begin(), sh.end());
  }
}

std::vector<float> depth_f32(const ImageD* d) {
  std::vector<float> out;
  if (d) out.assign(d->data().begin(), d->data().end());
  return out;
}

// validate_primitives (rasterizer.cpp:34-44) at the boundary, for the calls that may return before
// any device work (render_backward with no upstream gradient)
void validate_host(const std::vector<GaussianPrimitive>& prims) {
  for (size_t i = 0; i < prims.size(); ++i) {
    const GaussianPrimitive& p = prims[i];
    bool ok = p.mean.allFinite() && p.log_scale.allFinite() && p.quat.allFinite() && std::isfinite(p.opacity_logit) &&
              p.quat.norm() > 1e-12;
    for (const Vec3& c : p.sh) ok = ok && c.allFinite();
    if (!ok) throw std::invalid_argument("render: primitive " + std::to_string(i) + " has non-finite parameters");
  }
}

void check_observed(const ImageD* d, const CameraIntrinsics& k) {   // rasterizer.cpp:141-145
  if (d && (d->width() != k.width || d->height() != k.height))
    throw std::invalid_argument("render: observed depth dimensions do not match intrinsics");
}

std::vector<double> render_key(const std::vector<GaussianPrimitive>& prims, const CameraPose& pose,
                               const CameraIntrinsics& k, const ImageD* observed_depth, const RasterConfig& cfg) {
  std::vector<double> key = {pose.rotation_tangent.x(), pose.rotation_tangent.y(), pose.rotation_tangent.z(),
                             pose.translation.x(), pose.translation.y(), pose.translation.z(), k.fx, k.fy, k.cx, k.cy,
                             static_cast<double>(k.width), static_cast<double>(k.height), k.depth_scale, k.near_plane,
                             k.far_plane, cfg.alpha_clamp, cfg.alpha_skip, cfg.termination_threshold, cfg.footprint_sigma,
                             cfg.dilation, static_cast<double>(cfg.tile_size), cfg.uncertainty_full_gradient ? 1.0 : 0.0,
                             static_cast<double>(prims.size()), observed_depth ? 1.0 : 0.0};
  if (observed_depth) key.insert(key.end(), observed_depth->data().begin(), observed_depth->data().end());
  return key;
}

// One device render of (prims, pose, k, observed_depth, cfg) into `rr` (maps + the full CSR record).
void device_render(const std::vector<GaussianPrimitive>& prims, const CameraPose& pose, const CameraIntrinsics& k,
                   const ImageD* observed_depth, const RasterConfig& cfg, RenderResult* rr, bool reference,
                   std::vector<double>* key) {
  k.validate();
  check_observed(observed_depth, k);
  DropIn& s = state();
  upload(prims, key);
  const gsf_pose p = to_pose(pose);
  const gsf_intrinsics K = to_k(k);
  const gsf_raster_cfg c = to_cfg(cfg);
  const std::vector<float> obs = depth_f32(observed_depth);
  const size_t n = static_cast<size_t>(k.width) * k.height;
  std::vector<float> color(3 * n), ad(n), md(n), op(n), u(n), T(n), dw(n);
  std::vector<uint8_t> mv(n), vis(prims.size() + 1);
  std::vector<int32_t> cnt(n), dom(n), med(n);
  gsf_render_out o{color.data(), ad.data(), md.data(), mv.data(), op.data(), u.data(), T.data(), cnt.data(),
                   dom.data(), med.data(), dw.data(), vis.data(), 0, 0, 0};
  const float* od = observed_depth ? obs.data() : nullptr;
  raise(reference ? gsf_render_reference(s.ctx, &p, &K, od, &c, &o) : gsf_render(s.ctx, &p, &K, od, &c, &o));
  RenderOutput& out = rr->out;
  out.init(k.width, k.height);
  out.has_uncertainty = o.has_uncertainty != 0;
  for (size_t i = 0; i < n; ++i) {
    out.color[i] = Vec3(color[3 * i], color[3 * i + 1], color[3 * i + 2]);
    out.alpha_depth[i] = ad[i];
    out.median_depth[i] = md[i];
    out.median_valid[i] = mv[i];
    out.opacity[i] = op[i];
    out.uncertainty[i] = out.has_uncertainty ? u[i] : 0.0;
    out.final_transmittance[i] = T[i];
    out.per_pixel_count[i] = cnt[i];
  }
  if (reference) return;
  BlendRecord& r = rr->record;
  r.width = k.width;
  r.height = k.height;
  r.num_primitives = static_cast<int>(prims.size());
  r.dominant.resize(k.width, k.height);
  r.median_prim.resize(k.width, k.height);
  for (size_t i = 0; i < n; ++i) {
    r.dominant[i] = dom[i];
    r.median_prim[i] = med[i];
  }
  r.visible.assign(vis.begin(), vis.begin() + static_cast<std::ptrdiff_t>(prims.size()));
  int64_t total = 0;
  raise(gsf_render_record(s.ctx, nullptr, nullptr, nullptr, nullptr, &total));
  r.row_start.assign(n + 1, 0u);
  r.prim.assign(static_cast<size_t>(total), 0);
  std::vector<float> a(static_cast<size_t>(total)), t(static_cast<size_t>(total));
  raise(gsf_render_record(s.ctx, r.row_start.data(), r.prim.data(), a.data(), t.data(), &total));
  r.alpha.assign(a.begin(), a.end());
  r.transmittance.assign(t.begin(), t.end());
}

}  // namespace

RenderResult render(const std::vector<GaussianPrimitive>& primitives, const CameraPose& pose,
                    const CameraIntrinsics& intrinsics, const ImageD* observed_depth, const RasterConfig& config) {
  RenderResult rr;
  std::vector<double> key = render_key(primitives, pose, intrinsics, observed_depth, config);
  device_render(primitives, pose, intrinsics, observed_depth, config, &rr, false, &key);
  DropIn& s = state();
  s.key = std::move(key);
  s.record = nullptr;   // the caller's copy of rr.record is not addressable from here: match by key
  return rr;
}

RenderOutput render_reference(const std::vector<GaussianPrimitive>& primitives, const CameraPose& pose,
                              const CameraIntrinsics& intrinsics, const ImageD* observed_depth,
                              const RasterConfig& config) {
  RenderResult rr;
  device_render(primitives, pose, intrinsics, observed_depth, config, &rr, true, nullptr);
  state().key.clear();   // the device's latest render is now a reference render
  return rr.out;
}

GradientBundle render_backward(const std::vector<GaussianPrimitive>& prims, const CameraPose& pose,
                               const CameraIntrinsics& k, const BlendRecord& rec, const UpstreamGradients& up,
                               const ImageD* observed_depth, const RasterConfig& cfg) {
  // the reference's checks, in its order (rasterizer.cpp:343-365)
  k.validate();
  validate_host(prims);
  check_observed(observed_depth, k);
  if (rec.num_primitives != static_cast<int>(prims.size()))
    throw std::invalid_argument("render_backward: record does not match the primitive list");
  if (rec.width != k.width || rec.height != k.height)
    throw std::invalid_argument("render_backward: record dimensions do not match intrinsics");
  const int w = k.width, h = k.height;
  auto check_map = [&](const auto& img, const char* name) {
    if (!img.empty() && (img.width() != w || img.height() != h))
      throw std::invalid_argument(std::string("render_backward: upstream gradient ") + name + " has wrong dimensions");
    return !img.empty();
  };
  const bool use_color = check_map(up.d_color, "color");
  const bool use_adepth = check_map(up.d_alpha_depth, "alpha_depth");
  const bool use_mdepth = check_map(up.d_median_depth, "median_depth");
  const bool use_opacity = check_map(up.d_opacity, "opacity");
  const bool use_uncert = check_map(up.d_uncertainty, "uncertainty") && cfg.uncertainty_full_gradient;
  if (use_uncert && !observed_depth)
    throw std::invalid_argument("render_backward: uncertainty gradient needs observed depth");

  GradientBundle bundle;
  bundle.init(prims);
  const size_t P = prims.size();
  if (!(use_color || use_adepth || use_mdepth || use_opacity || use_uncert) || P == 0) return bundle;
  // the device backward runs over the context's latest render: re-render unless it is this one
  DropIn& s = state();
  std::vector<double> key = render_key(prims, pose, k, observed_depth, cfg);
  std::vector<double> probe = key;
  {
    // the map contents are part of the key (the caller may have stepped an optimizer in between)
    const int K = static_cast<int>(prims[0].sh.size());
    for (const GaussianPrimitive& p : prims)
      for (int a = 0; a < 3; ++a) probe.push_back(p.mean(a));
    for (const GaussianPrimitive& p : prims)
      for (int a = 0; a < 3; ++a) probe.push_back(p.log_scale(a));
    for (const GaussianPrimitive& p : prims)
      for (int a = 0; a < 4; ++a) probe.push_back(p.quat(a));
    for (const GaussianPrimitive& p : prims) probe.push_back(p.opacity_logit);
    for (const GaussianPrimitive& p : prims)
      for (int c = 0; c < K; ++c)
        for (int a = 0; a < 3; ++a) probe.push_back(p.sh[c](a));
  }
  if (s.key.empty() || s.key != probe) {
    RenderResult tmp;
    device_render(prims, pose, k, observed_depth, cfg, &tmp, false, &key);
    s.key = std::move(key);
  }
  const size_t n = static_cast<size_t>(w) * h;
  std::vector<float> dc, dad, dmd, dop, du;
  auto flat1 = [&](const ImageD& img, std::vector<float>& v) {
    v.assign(img.data().begin(), img.data().end());
    return v.data();
  };
  if (use_color) {
    dc.resize(3 * n);
    for (size_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) dc[3 * i + a] = static_cast<float>(up.d_color[i](a));
  }
  gsf_upstream u{use_color ? dc.data() : nullptr, use_adepth ? flat1(up.d_alpha_depth, dad) : nullptr,
                 use_mdepth ? flat1(up.d_median_depth, dmd) : nullptr, use_opacity ? flat1(up.d_opacity, dop) : nullptr,
                 use_uncert ? flat1(up.d_uncertainty, du) : nullptr};
  const int K = static_cast<int>(prims[0].sh.size());
  std::vector<float> gm(3 * P), gls(3 * P), gq(4 * P), gop(P), gsh(3 * static_cast<size_t>(K) * P), gm2(2 * P);
  gsf_grads_out g{gm.data(), gls.data(), gq.data(), gop.data(), gsh.data(), gm2.data(), {0, 0, 0, 0, 0, 0}};
  const std::vector<float> obs = depth_f32(observed_depth);
  raise(gsf_render_backward(s.ctx, &u, observed_depth ? obs.data() : nullptr, &g));
  for (size_t i = 0; i < P; ++i) {
    bundle.d_mean[i] = Vec3(gm[3 * i], gm[3 * i + 1], gm[3 * i + 2]);
    bundle.d_log_scale[i] = Vec3(gls[3 * i], gls[3 * i + 1], gls[3 * i + 2]);
    bundle.d_quat[i] = Vec4(gq[4 * i], gq[4 * i + 1], gq[4 * i + 2], gq[4 * i + 3]);
    bundle.d_opacity_logit[i] = gop[i];
    for (int c = 0; c < K; ++c)
      bundle.d_sh[i][c] = Vec3(gsh[(i * K + c) * 3], gsh[(i * K + c) * 3 + 1], gsh[(i * K + c) * 3 + 2]);
    bundle.d_mean2d[i] = Vec2(gm2[2 * i], gm2[2 * i + 1]);
  }
  for (int a = 0; a < 6; ++a) bundle.d_pose(a) = g.d_pose[a];
  return bundle;
}

}  // namespace gsf
