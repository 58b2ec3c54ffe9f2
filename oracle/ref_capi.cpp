// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// The C surface of oracle/_ref/libgsfref.so: the UNMODIFIED reference sources
// (/root/reference/proj/src/{geometry,raster,loss,map,track,io/synthetic,verify}/*.cpp, compiled in
// place by oracle/Makefile.ref against oracle/eigen_lite) behind the same orc_* entry points as the
// restatement (oracle/gsf_oracle.h), so the Python checker can run either backend on identical
// inputs.  This file only converts between the flat C layout of include/gsf_cuda.h and the
// reference's own types; every computation is the reference's.
//
// Built only where /root/reference exists (this container); the .so travels to the GPU box in the
// gpurun snapshot (oracle/_ref/ is git-ignored, not gpurun-ignored).
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gsf_oracle.h"
#include "gsfield/io/synthetic.hpp"
#include "gsfield/loss/losses.hpp"
#include "gsfield/loss/ssim.hpp"
#include "gsfield/map/mapper.hpp"
#include "gsfield/map/uncertainty.hpp"
#include "gsfield/raster/rasterizer.hpp"
#include "gsfield/track/tracker.hpp"
#include "gsfield/verify/gradcheck.hpp"

namespace {

thread_local std::string g_err;

gsf::CameraPose to_pose(const gsf_pose* p) {
  gsf::CameraPose o;
  o.rotation_tangent = gsf::Vec3(p->rotation_tangent[0], p->rotation_tangent[1], p->rotation_tangent[2]);
  o.translation = gsf::Vec3(p->translation[0], p->translation[1], p->translation[2]);
  return o;
}
void from_pose(const gsf::CameraPose& p, gsf_pose* o) {
  for (int a = 0; a < 3; ++a) {
    o->rotation_tangent[a] = p.rotation_tangent(a);
    o->translation[a] = p.translation(a);
  }
}
gsf::CameraIntrinsics to_k(const gsf_intrinsics* k) {
  gsf::CameraIntrinsics o;
  o.fx = k->fx; o.fy = k->fy; o.cx = k->cx; o.cy = k->cy;
  o.width = k->width; o.height = k->height;
  o.depth_scale = k->depth_scale; o.near_plane = k->near_plane; o.far_plane = k->far_plane;
  return o;
}
gsf::RasterConfig to_raster(const gsf_raster_cfg* c) {
  gsf::RasterConfig o;
  o.alpha_clamp = c->alpha_clamp; o.alpha_skip = c->alpha_skip; o.termination_threshold = c->termination_threshold;
  o.footprint_sigma = c->footprint_sigma; o.dilation = c->dilation; o.tile_size = c->tile_size;
  o.uncertainty_full_gradient = c->uncertainty_full_gradient != 0; o.threads = c->threads;
  return o;
}
void from_raster(const gsf::RasterConfig& o, gsf_raster_cfg* c) {
  c->alpha_clamp = o.alpha_clamp; c->alpha_skip = o.alpha_skip; c->termination_threshold = o.termination_threshold;
  c->footprint_sigma = o.footprint_sigma; c->dilation = o.dilation; c->tile_size = o.tile_size;
  c->uncertainty_full_gradient = o.uncertainty_full_gradient ? 1 : 0; c->threads = o.threads;
}
gsf::LossWeights to_w(const gsf_loss_weights* w) {
  gsf::LossWeights o;
  o.w_color = w->w_color; o.w_ssim = w->w_ssim; o.w_geo = w->w_geo; o.w_align = w->w_align; o.w_iso = w->w_iso;
  o.w_var = w->w_var; o.t_color = w->t_color; o.t_geo = w->t_geo; o.iso_epsilon = w->iso_epsilon;
  o.opacity_floor = w->opacity_floor; o.normalize_by_valid = w->normalize_by_valid != 0;
  return o;
}
void from_w(const gsf::LossWeights& o, gsf_loss_weights* w) {
  w->w_color = o.w_color; w->w_ssim = o.w_ssim; w->w_geo = o.w_geo; w->w_align = o.w_align; w->w_iso = o.w_iso;
  w->w_var = o.w_var; w->t_color = o.t_color; w->t_geo = o.t_geo; w->iso_epsilon = o.iso_epsilon;
  w->opacity_floor = o.opacity_floor; w->normalize_by_valid = o.normalize_by_valid ? 1 : 0;
}
gsf::TrackerConfig to_t(const gsf_tracker_cfg* t) {
  gsf::TrackerConfig o;
  o.lr_rotation = t->lr_rotation; o.lr_translation = t->lr_translation; o.iterations = t->iterations;
  o.ba_window = t->ba_window; o.ba_iterations = t->ba_iterations; o.keyframe_interval = t->keyframe_interval;
  o.recent_keyframes = t->recent_keyframes; o.freeze_oldest_pose = t->freeze_oldest_pose != 0;
  o.degraded_loss_ratio = t->degraded_loss_ratio;
  return o;
}
gsf::MapperConfig to_m(const gsf_mapper_cfg* m) {
  gsf::MapperConfig o;
  o.sh_coeffs = m->sh_coeffs; o.scene_extent = m->scene_extent; o.lr_mean = m->lr_mean; o.lr_sh = m->lr_sh;
  o.lr_opacity = m->lr_opacity; o.lr_scale = m->lr_scale; o.lr_rotation = m->lr_rotation;
  o.densify.interval = m->densify_interval; o.densify.grad_threshold = m->densify_grad_threshold;
  o.densify.split_factor = m->densify_split_factor; o.densify.size_fraction = m->densify_size_fraction;
  o.densify.cull_opacity = m->densify_cull_opacity;
  o.uncertainty.tau = m->uncertainty_tau; o.uncertainty.reduced_opacity = m->uncertainty_reduced_opacity;
  o.seed = m->seed; o.raster = to_raster(&m->raster); o.weights = to_w(&m->weights);
  o.init_stride = m->init_stride; o.spawn_stride = m->spawn_stride;
  o.spawn_opacity_threshold = m->spawn_opacity_threshold; o.init_opacity = m->init_opacity;
  return o;
}

std::vector<gsf::GaussianPrimitive> load_map(const gsf_map_host* m) {
  std::vector<gsf::GaussianPrimitive> p(static_cast<size_t>(m->count));
  const int K = m->sh_coeffs;
  for (int64_t i = 0; i < m->count; ++i) {
    gsf::GaussianPrimitive& g = p[i];
    g.mean = gsf::Vec3(m->mean[3 * i], m->mean[3 * i + 1], m->mean[3 * i + 2]);
    g.log_scale = gsf::Vec3(m->log_scale[3 * i], m->log_scale[3 * i + 1], m->log_scale[3 * i + 2]);
    g.quat = gsf::Vec4(m->quat[4 * i], m->quat[4 * i + 1], m->quat[4 * i + 2], m->quat[4 * i + 3]);
    g.opacity_logit = m->opacity_logit[i];
    g.sh.resize(K);
    for (int b = 0; b < K; ++b)
      g.sh[b] = gsf::Vec3(m->sh[3 * K * i + 3 * b], m->sh[3 * K * i + 3 * b + 1], m->sh[3 * K * i + 3 * b + 2]);
    if (m->uncertainty) g.uncertainty = m->uncertainty[i];
    if (m->observed) g.observed = m->observed[i] != 0;
  }
  return p;
}
void store_map(const std::vector<gsf::GaussianPrimitive>& p, gsf_map_host* m) {
  const int K = m->sh_coeffs;
  for (size_t i = 0; i < p.size(); ++i) {
    for (int a = 0; a < 3; ++a) { m->mean[3 * i + a] = p[i].mean(a); m->log_scale[3 * i + a] = p[i].log_scale(a); }
    for (int a = 0; a < 4; ++a) m->quat[4 * i + a] = p[i].quat(a);
    m->opacity_logit[i] = p[i].opacity_logit;
    for (int b = 0; b < K; ++b)
      for (int c = 0; c < 3; ++c) m->sh[3 * K * i + 3 * b + c] = b < static_cast<int>(p[i].sh.size()) ? p[i].sh[b](c) : 0.0;
    if (m->uncertainty) m->uncertainty[i] = p[i].uncertainty;
    if (m->observed) m->observed[i] = p[i].observed ? 1 : 0;
  }
}
gsf::ImageD image_d(const double* d, int w, int h) {
  gsf::ImageD o(w, h);
  std::memcpy(o.data().data(), d, sizeof(double) * static_cast<size_t>(w) * h);
  return o;
}
gsf::ImageRGB image_rgb(const double* d, int w, int h) {
  gsf::ImageRGB o(w, h);
  for (size_t i = 0; i < o.size(); ++i) o[i] = gsf::Vec3(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
  return o;
}

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

void export_grads(const gsf::GradientBundle& g, int K, orc_grads* out) {
  for (size_t i = 0; i < g.d_mean.size(); ++i) {
    if (out->d_mean) for (int a = 0; a < 3; ++a) out->d_mean[3 * i + a] = g.d_mean[i](a);
    if (out->d_log_scale) for (int a = 0; a < 3; ++a) out->d_log_scale[3 * i + a] = g.d_log_scale[i](a);
    if (out->d_quat) for (int a = 0; a < 4; ++a) out->d_quat[4 * i + a] = g.d_quat[i](a);
    if (out->d_opacity_logit) out->d_opacity_logit[i] = g.d_opacity_logit[i];
    if (out->d_sh)
      for (int b = 0; b < K; ++b)
        for (int c = 0; c < 3; ++c)
          out->d_sh[3 * K * i + 3 * b + c] = b < static_cast<int>(g.d_sh[i].size()) ? g.d_sh[i][b](c) : 0.0;
    if (out->d_mean2d) { out->d_mean2d[2 * i] = g.d_mean2d[i](0); out->d_mean2d[2 * i + 1] = g.d_mean2d[i](1); }
  }
  for (int a = 0; a < 6; ++a) out->d_pose[a] = g.d_pose(a);
}

gsf::UpstreamGradients to_upstream(const orc_upstream* up, int w, int h) {
  gsf::UpstreamGradients u;
  if (!up) return u;
  if (up->d_color) u.d_color = image_rgb(up->d_color, w, h);
  if (up->d_alpha_depth) u.d_alpha_depth = image_d(up->d_alpha_depth, w, h);
  if (up->d_median_depth) u.d_median_depth = image_d(up->d_median_depth, w, h);
  if (up->d_opacity) u.d_opacity = image_d(up->d_opacity, w, h);
  if (up->d_uncertainty) u.d_uncertainty = image_d(up->d_uncertainty, w, h);
  return u;
}

void export_upstream(const gsf::UpstreamGradients& u, size_t n, double* d_color, double* d_ad, double* d_md,
                     double* d_u) {
  for (size_t i = 0; i < n; ++i) {
    if (d_color) for (int c = 0; c < 3; ++c) d_color[3 * i + c] = u.d_color.empty() ? 0.0 : u.d_color[i](c);
    if (d_ad) d_ad[i] = u.d_alpha_depth.empty() ? 0.0 : u.d_alpha_depth[i];
    if (d_md) d_md[i] = u.d_median_depth.empty() ? 0.0 : u.d_median_depth[i];
    if (d_u) d_u[i] = u.d_uncertainty.empty() ? 0.0 : u.d_uncertainty[i];
  }
}

}  // namespace

struct orc_result {
  gsf::RenderResult r;   // render_reference fills r.out only (no record)
};

struct orc_mapstate {
  gsf::MapState st;
  explicit orc_mapstate(const gsf::MapperConfig& c) : st(c) {}
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_threads(void) { return gsf::resolve_threads(0); }

int orc_render(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K, const double* observed_depth,
               const gsf_raster_cfg* cfg, int brute_force, orc_result** out) {
  return guarded([&] {
    const auto prims = load_map(map);
    const gsf::CameraIntrinsics k = to_k(K);
    gsf::ImageD obs;
    if (observed_depth) obs = image_d(observed_depth, k.width, k.height);
    auto res = std::make_unique<orc_result>();
    if (brute_force) {
      res->r.out = gsf::render_reference(prims, to_pose(pose), k, observed_depth ? &obs : nullptr, to_raster(cfg));
    } else {
      res->r = gsf::render(prims, to_pose(pose), k, observed_depth ? &obs : nullptr, to_raster(cfg));
    }
    *out = res.release();
  });
}

void orc_result_free(orc_result* r) { delete r; }

// RenderOutput + BlendRecord's per-pixel parts.  The reference keeps no dominant weight map; it is
// recovered from the record (alpha * T of the dominant contributor, the weight rasterizer.cpp:124-127
// maximises), 0 where no contributor.
int orc_result_maps(const orc_result* res, orc_maps* o) {
  const gsf::RenderOutput& out = res->r.out;
  const gsf::BlendRecord& rec = res->r.record;
  const bool have_rec = !rec.row_start.empty();
  const size_t n = static_cast<size_t>(out.width) * out.height;
  for (size_t i = 0; i < n; ++i) {
    if (o->color) for (int c = 0; c < 3; ++c) o->color[3 * i + c] = out.color[i](c);
    if (o->alpha_depth) o->alpha_depth[i] = out.alpha_depth[i];
    if (o->median_depth) o->median_depth[i] = out.median_depth[i];
    if (o->median_valid) o->median_valid[i] = out.median_valid[i];
    if (o->opacity) o->opacity[i] = out.opacity[i];
    if (o->uncertainty) o->uncertainty[i] = out.uncertainty[i];
    if (o->final_transmittance) o->final_transmittance[i] = out.final_transmittance[i];
    if (o->per_pixel_count) o->per_pixel_count[i] = out.per_pixel_count[i];
    if (o->dominant) o->dominant[i] = have_rec ? rec.dominant[i] : -1;
    if (o->median_prim) o->median_prim[i] = have_rec ? rec.median_prim[i] : -1;
    if (o->dominant_weight) {
      double dw = 0.0;
      if (have_rec && rec.dominant[i] >= 0)
        for (uint32_t e = rec.row_start[i]; e < rec.row_start[i + 1]; ++e)
          if (rec.prim[e] == rec.dominant[i]) { dw = rec.alpha[e] * rec.transmittance[e]; break; }
      o->dominant_weight[i] = dw;
    }
  }
  if (o->visible) for (size_t i = 0; i < rec.visible.size(); ++i) o->visible[i] = rec.visible[i];
  o->has_uncertainty = out.has_uncertainty ? 1 : 0;
  return GSF_OK;
}

int64_t orc_result_record_total(const orc_result* r) { return static_cast<int64_t>(r->r.record.prim.size()); }

int orc_result_record(const orc_result* res, uint32_t* row_start, int32_t* prim, double* alpha, double* transmittance) {
  const gsf::BlendRecord& rec = res->r.record;
  if (row_start) std::memcpy(row_start, rec.row_start.data(), rec.row_start.size() * sizeof(uint32_t));
  if (prim) std::memcpy(prim, rec.prim.data(), rec.prim.size() * sizeof(int32_t));
  if (alpha) std::memcpy(alpha, rec.alpha.data(), rec.alpha.size() * sizeof(double));
  if (transmittance) std::memcpy(transmittance, rec.transmittance.data(), rec.transmittance.size() * sizeof(double));
  return GSF_OK;
}

int orc_render_backward(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K, const orc_result* r,
                        const orc_upstream* up, const double* observed_depth, const gsf_raster_cfg* cfg, orc_grads* out) {
  return guarded([&] {
    const auto prims = load_map(map);
    gsf::ImageD obs;
    if (observed_depth) obs = image_d(observed_depth, K->width, K->height);
    const gsf::GradientBundle g = gsf::render_backward(prims, to_pose(pose), to_k(K), r->r.record,
                                                       to_upstream(up, K->width, K->height),
                                                       observed_depth ? &obs : nullptr, to_raster(cfg));
    export_grads(g, map->sh_coeffs, out);
  });
}

int orc_tracking_loss(const orc_result* r, const double* target, const double* obs, const gsf_intrinsics* K,
                      const gsf_loss_weights* w, gsf_loss_terms* out, double* d_color, double* d_alpha_depth) {
  return guarded([&] {
    const gsf::TrackingLossResult l = gsf::evaluate_tracking_loss(
        r->r, image_rgb(target, K->width, K->height), image_d(obs, K->width, K->height), to_k(K), to_w(w), true);
    *out = gsf_loss_terms{};
    out->color = l.color; out->geo = l.geo; out->total = l.total;
    out->valid_color = l.valid_color; out->valid_geo = l.valid_geo;
    export_upstream(l.upstream, static_cast<size_t>(K->width) * K->height, d_color, d_alpha_depth, nullptr, nullptr);
  });
}

int orc_mapping_loss(const gsf_map_host* map, const orc_result* r, const double* target, const double* obs,
                     const gsf_intrinsics* K, const gsf_loss_weights* w, gsf_loss_terms* out, double* d_color,
                     double* d_alpha_depth, double* d_median_depth, double* d_uncertainty, double* d_ls_direct) {
  return guarded([&] {
    const auto prims = load_map(map);
    const gsf::MappingLossResult l = gsf::evaluate_mapping_loss(
        prims, r->r, image_rgb(target, K->width, K->height), image_d(obs, K->width, K->height), to_k(K), to_w(w), true);
    *out = gsf_loss_terms{};
    out->color = l.color; out->ssim = l.ssim; out->geo = l.geo; out->align = l.align; out->iso = l.iso;
    out->var = l.var; out->total = l.total; out->any_empty_mask = l.any_empty_mask ? 1 : 0;
    export_upstream(l.upstream, static_cast<size_t>(K->width) * K->height, d_color, d_alpha_depth, d_median_depth,
                    d_uncertainty);
    if (d_ls_direct)
      for (size_t i = 0; i < prims.size(); ++i)
        for (int a = 0; a < 3; ++a) d_ls_direct[3 * i + a] = l.d_log_scale_direct.empty() ? 0.0 : l.d_log_scale_direct[i](a);
  });
}

int orc_ssim(const double* x, const double* y, int w, int h, double* value, double* d_x) {
  return guarded([&] {
    const gsf::ImageRGB xi = image_rgb(x, w, h), yi = image_rgb(y, w, h);
    if (!d_x) {
      *value = gsf::ssim(xi, yi);
      return;
    }
    gsf::ImageRGB g;
    *value = gsf::ssim_with_gradient(xi, yi, g);
    for (size_t i = 0; i < g.size(); ++i)
      for (int c = 0; c < 3; ++c) d_x[3 * i + c] = g[i](c);
  });
}

int orc_track_frame(const gsf_map_host* map, const double* rgb, const double* depth, const gsf_pose* initial,
                    const gsf_intrinsics* K, const gsf_tracker_cfg* cfg, const gsf_loss_weights* w,
                    const gsf_raster_cfg* raster, gsf_track_result* out) {
  return guarded([&] {
    const auto prims = load_map(map);
    const gsf::TrackResult r = gsf::track_frame(prims, image_rgb(rgb, K->width, K->height),
                                                image_d(depth, K->width, K->height), to_pose(initial), to_k(K),
                                                to_t(cfg), to_w(w), to_raster(raster));
    *out = gsf_track_result{};
    from_pose(r.pose, &out->pose);
    out->final_loss = r.final_loss;
    out->degraded = r.degraded ? 1 : 0;
    out->iterations_run = r.iterations_run;
    out->initial_loss = 0.0;   // TrackResult carries no initial loss (tracker.hpp:28-33)
  });
}

int orc_mapstate_create(const gsf_map_host* map, const gsf_mapper_cfg* mcfg, orc_mapstate** out) {
  return guarded([&] {
    auto s = std::make_unique<orc_mapstate>(to_m(mcfg));
    s->st.primitives = load_map(map);
    s->st.optimizer.append(s->st.primitives.size());
    s->st.grad_accum.assign(s->st.primitives.size(), 0.0);
    s->st.grad_count.assign(s->st.primitives.size(), 0);
    *out = s.release();
  });
}
void orc_mapstate_free(orc_mapstate* s) { delete s; }
int64_t orc_mapstate_count(const orc_mapstate* s) { return static_cast<int64_t>(s->st.primitives.size()); }
int orc_mapstate_get(const orc_mapstate* s, gsf_map_host* out) {
  if (out->count != static_cast<int64_t>(s->st.primitives.size())) { g_err = "count mismatch"; return GSF_EINVAL; }
  store_map(s->st.primitives, out);
  return GSF_OK;
}
int orc_mapstate_put(orc_mapstate* s, const gsf_map_host* map) {
  return guarded([&] {
    if (map->count != static_cast<int64_t>(s->st.primitives.size())) throw std::invalid_argument("count mismatch");
    s->st.primitives = load_map(map);
  });
}

// spawn_gaussians' tail (mapper.cpp:163-169) as MapState edits: append primitives with fresh moments.
int orc_mapstate_append(orc_mapstate* s, const gsf_map_host* map) {
  return guarded([&] {
    const auto add = load_map(map);
    s->st.primitives.insert(s->st.primitives.end(), add.begin(), add.end());
    s->st.optimizer.append(add.size());
    s->st.grad_accum.resize(s->st.primitives.size(), 0.0);
    s->st.grad_count.resize(s->st.primitives.size(), 0);
  });
}
int orc_mapstate_set_stats(orc_mapstate* s, const double* accum, const int32_t* count) {
  for (size_t i = 0; i < s->st.primitives.size(); ++i) {
    s->st.grad_accum[i] = accum[i];
    s->st.grad_count[i] = count[i];
  }
  return GSF_OK;
}
int orc_mapstate_densify(orc_mapstate* s, const gsf_mapper_cfg* cfg, int32_t* change /*split, cloned, removed*/) {
  return guarded([&] {
    const gsf::StructuralChange c = gsf::densify_and_cull(s->st, to_m(cfg));
    change[0] = c.split;
    change[1] = c.cloned;
    change[2] = c.removed;
  });
}

int orc_map_step(orc_mapstate* s, int n, const double* const* rgbs, const double* const* depths, const gsf_pose* poses,
                 const gsf_intrinsics* K, const gsf_mapper_cfg* mcfg, int iterations, double* trace) {
  return guarded([&] {
    std::vector<gsf::ImageRGB> rgb(n);
    std::vector<gsf::ImageD> dep(n);
    std::vector<gsf::MapObservation> win(n);
    for (int i = 0; i < n; ++i) {
      if (rgbs[i]) rgb[i] = image_rgb(rgbs[i], K->width, K->height);
      if (depths[i]) dep[i] = image_d(depths[i], K->width, K->height);
      win[i].rgb = rgbs[i] ? &rgb[i] : nullptr;
      win[i].depth = depths[i] ? &dep[i] : nullptr;
      win[i].pose = to_pose(&poses[i]);
    }
    const std::vector<double> t = gsf::map_step(s->st, win, to_k(K), to_m(mcfg), iterations);
    if (trace) for (size_t i = 0; i < t.size(); ++i) trace[i] = t[i];
  });
}

int orc_sliding_ba(orc_mapstate* s, int n, const double* const* rgbs, const double* const* depths, gsf_pose* poses,
                   const int32_t* frame_ids, const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg,
                   const gsf_mapper_cfg* mcfg, int iterations, double* trace) {
  return guarded([&] {
    std::vector<gsf::KeyframeRecord> kf(n);
    std::vector<gsf::KeyframeRecord*> win(n);
    for (int i = 0; i < n; ++i) {
      kf[i].frame_id = frame_ids[i];
      kf[i].rgb = image_rgb(rgbs[i], K->width, K->height);
      kf[i].depth = image_d(depths[i], K->width, K->height);
      kf[i].pose = to_pose(&poses[i]);
      win[i] = &kf[i];
    }
    const std::vector<double> t = gsf::sliding_ba(s->st, win, to_k(K), to_t(tcfg), to_m(mcfg), iterations);
    for (int i = 0; i < n; ++i) from_pose(kf[i].pose, &poses[i]);
    if (trace) for (size_t i = 0; i < t.size(); ++i) trace[i] = t[i];
  });
}

int orc_accumulate_uncertainty(gsf_map_host* map, int n, const orc_result* const* records, const double* const* depths,
                               const gsf_pose* poses, const gsf_intrinsics* K, int32_t* observed_count) {
  return guarded([&] {
    auto prims = load_map(map);
    std::vector<gsf::ImageD> dep(n);
    std::vector<gsf::UncertaintyView> win(n);
    for (int i = 0; i < n; ++i) {
      dep[i] = image_d(depths[i], K->width, K->height);
      win[i].record = &records[i]->r.record;
      win[i].observed_depth = &dep[i];
      win[i].pose = to_pose(&poses[i]);
      win[i].intrinsics = to_k(K);
    }
    const int obs = gsf::accumulate_uncertainty(prims, win, 0);
    if (observed_count) *observed_count = obs;
    store_map(prims, map);
  });
}

int orc_prune_unreliable(gsf_map_host* map, double tau, double reduced_opacity, int32_t* reduced) {
  return guarded([&] {
    auto prims = load_map(map);
    gsf::UncertaintyConfig c;
    c.tau = tau;
    c.reduced_opacity = reduced_opacity;
    const int r = gsf::prune_unreliable(prims, c);
    if (reduced) *reduced = r;
    store_map(prims, map);
  });
}

// Config defaults straight from the reference structs (config.hpp, losses.cpp:33-46, tracker.hpp, mapper.hpp).
void orc_default_raster(gsf_raster_cfg* c) { from_raster(gsf::RasterConfig{}, c); }
void orc_default_weights(gsf_loss_weights* w, int handheld_real) {
  from_w(handheld_real ? gsf::LossWeights::handheld_real() : gsf::LossWeights::indoor_synthetic(), w);
}
void orc_default_tracker(gsf_tracker_cfg* c) {
  const gsf::TrackerConfig t;
  *c = gsf_tracker_cfg{t.lr_rotation, t.lr_translation, t.iterations, t.ba_window, t.ba_iterations,
                       t.keyframe_interval, t.recent_keyframes, t.freeze_oldest_pose ? 1 : 0, t.degraded_loss_ratio};
}
void orc_default_mapper(gsf_mapper_cfg* c) {
  const gsf::MapperConfig m;
  *c = gsf_mapper_cfg{};
  c->sh_coeffs = m.sh_coeffs; c->scene_extent = m.scene_extent; c->lr_mean = m.lr_mean; c->lr_sh = m.lr_sh;
  c->lr_opacity = m.lr_opacity; c->lr_scale = m.lr_scale; c->lr_rotation = m.lr_rotation;
  c->densify_interval = m.densify.interval; c->densify_grad_threshold = m.densify.grad_threshold;
  c->densify_split_factor = m.densify.split_factor; c->densify_size_fraction = m.densify.size_fraction;
  c->densify_cull_opacity = m.densify.cull_opacity; c->uncertainty_tau = m.uncertainty.tau;
  c->uncertainty_reduced_opacity = m.uncertainty.reduced_opacity; c->seed = m.seed;
  from_raster(m.raster, &c->raster);
  from_w(m.weights, &c->weights);
  c->init_stride = m.init_stride; c->spawn_stride = m.spawn_stride;
  c->spawn_opacity_threshold = m.spawn_opacity_threshold; c->init_opacity = m.init_opacity;
}
void orc_smooth_raster(gsf_raster_cfg* c) { from_raster(gsf::smooth_raster_config(), c); }

// The reference's synthetic scene + trajectory (io/synthetic.cpp:199-211; frames are not rendered).
// Writes up to out->count primitives (sh_coeffs 1) and returns the true count in *count; poses up to
// max_poses.  kind 0 room / 1 flat wall.
int ref_synth_scene(int kind, int primitive_count, double extent, int wall_layers, int frames, double radius,
                    uint64_t seed, const gsf_intrinsics* K, gsf_map_host* out, int64_t* count, gsf_pose* poses,
                    int max_poses) {
  return guarded([&] {
    gsf::SceneSpec sc;
    sc.kind = kind == 0 ? gsf::SceneKind::room : gsf::SceneKind::flat_wall;
    sc.primitive_count = primitive_count;
    sc.extent = extent;
    sc.wall_layers = wall_layers;
    gsf::TrajectorySpec tr;
    tr.frames = frames;
    tr.radius = radius;
    const gsf::SyntheticSource src(sc, tr, gsf::NoiseSpec{}, to_k(K), seed);
    const auto& gt = src.ground_truth();
    *count = static_cast<int64_t>(gt.size());
    if (out && out->count >= static_cast<int64_t>(gt.size())) {
      gsf_map_host o = *out;
      o.count = static_cast<int64_t>(gt.size());
      store_map(gt, &o);
    }
    for (int i = 0; i < max_poses && i < static_cast<int>(src.poses().size()); ++i) from_pose(src.poses()[i], &poses[i]);
  });
}

}  // extern "C"
