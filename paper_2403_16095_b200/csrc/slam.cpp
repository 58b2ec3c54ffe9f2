// slam.cpp — SlamSystem (slam/system.cpp:31-154) on the device map, written against the public
// C-ABI only (include/gsf_cuda.h): tracking per frame, and per keyframe map_step over the selected
// window, sliding_ba, uncertainty accumulation + pruning and spawning.  The host keeps what the
// reference keeps on the host: keyframe records (pose, frame id, timestamp, appearance
// descriptor), the trajectory, the velocity model and the per-frame logs.  Frames live in device
// slots of the context: slot 0 is the frame being tracked, keyframe k owns slot 1 + k.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <utility>
#include <vector>

#include "../../include/gsf_cuda.h"

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); }

// ---- SO(3) / SE(3) helpers (geometry/lie.cpp:7-52, geometry/pose.hpp:13-49), fp64 ---------------
struct M3 {
  double a[9];
};

M3 exp_map(const double* v) {
  const double th2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  const double th = std::sqrt(th2);
  double a, b;
  if (th < 1e-8) {
    a = 1.0 - th2 / 6.0;
    b = 0.5 - th2 / 24.0;
  } else {
    a = std::sin(th) / th;
    b = (1.0 - std::cos(th)) / th2;
  }
  const double k[9] = {0.0, -v[2], v[1], v[2], 0.0, -v[0], -v[1], v[0], 0.0};
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double kk = k[3 * i] * k[j] + k[3 * i + 1] * k[3 + j] + k[3 * i + 2] * k[6 + j];
      r.a[3 * i + j] = (i == j ? 1.0 : 0.0) + a * k[3 * i + j] + b * kk;
    }
  return r;
}

void log_map(const M3& R, double* out) {
  const double* r = R.a;
  const double ct = std::clamp((r[0] + r[4] + r[8] - 1.0) * 0.5, -1.0, 1.0);
  const double theta = std::acos(ct);
  const double vee[3] = {r[7] - r[5], r[2] - r[6], r[3] - r[1]};
  if (theta < 1e-8) {
    const double f = 0.5 * (1.0 + theta * theta / 6.0);
    for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
    return;
  }
  if (theta > 3.14159265358979323846 - 1e-3) {
    double outer[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) outer[3 * i + j] = (0.5 * (r[3 * i + j] + r[3 * j + i]) - ct * (i == j ? 1.0 : 0.0)) / (1.0 - ct);
    int a = 0;
    for (int i = 1; i < 3; ++i)
      if (outer[4 * i] > outer[4 * a]) a = i;
    const double sq = std::sqrt(outer[4 * a]);
    double ax[3] = {outer[a] / sq, outer[3 + a] / sq, outer[6 + a] / sq};
    if (ax[0] * vee[0] + ax[1] * vee[1] + ax[2] * vee[2] < 0.0)
      for (double& x : ax) x = -x;
    for (int i = 0; i < 3; ++i) out[i] = theta * ax[i];
    return;
  }
  const double f = theta / (2.0 * std::sin(theta));
  for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
}

M3 mul(const M3& x, const M3& y) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[3 * i + j] = x.a[3 * i] * y.a[j] + x.a[3 * i + 1] * y.a[3 + j] + x.a[3 * i + 2] * y.a[6 + j];
  return r;
}

// this o other: apply other first (pose.hpp:29-33)
gsf_pose compose(const gsf_pose& self, const gsf_pose& other) {
  const M3 r1 = exp_map(self.rotation_tangent), r2 = exp_map(other.rotation_tangent);
  gsf_pose out{};
  log_map(mul(r1, r2), out.rotation_tangent);
  for (int i = 0; i < 3; ++i)
    out.translation[i] = r1.a[3 * i] * other.translation[0] + r1.a[3 * i + 1] * other.translation[1] +
                         r1.a[3 * i + 2] * other.translation[2] + self.translation[i];
  return out;
}

gsf_pose inverse(const gsf_pose& p) {   // pose.hpp:35-38
  const M3 r = exp_map(p.rotation_tangent);
  gsf_pose out{};
  for (int i = 0; i < 3; ++i) {
    out.rotation_tangent[i] = -p.rotation_tangent[i];
    out.translation[i] = -(r.a[i] * p.translation[0] + r.a[3 + i] * p.translation[1] + r.a[6 + i] * p.translation[2]);
  }
  return out;
}

// constant-velocity prediction (tracker.cpp:26-28)
gsf_pose predict_pose(const gsf_pose& prev, const gsf_pose& before) { return compose(prev, compose(inverse(before), prev)); }

// ---- appearance descriptor (track/descriptor.cpp:9-43) -----------------------------------------
constexpr int kDescriptorLength = 8 * 8 + 3 * 16;

std::vector<double> compute_descriptor(const float* rgb, int w, int h) {
  std::vector<double> d(kDescriptorLength, 0.0);
  for (int gy = 0; gy < 8; ++gy)
    for (int gx = 0; gx < 8; ++gx) {   // 8x8 grid of mean luminance
      const int x0 = w * gx / 8, x1 = std::max(w * (gx + 1) / 8, x0 + 1);
      const int y0 = h * gy / 8, y1 = std::max(h * (gy + 1) / 8, y0 + 1);
      double acc = 0.0;
      int n = 0;
      for (int y = y0; y < y1 && y < h; ++y)
        for (int x = x0; x < x1 && x < w; ++x) {
          const float* p = rgb + 3 * (static_cast<size_t>(y) * w + x);
          acc += 0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2];
          ++n;
        }
      if (n > 0) d[gy * 8 + gx] = acc / n;
    }
  const size_t npix = static_cast<size_t>(w) * h;
  const double inv_n = 1.0 / static_cast<double>(npix);
  for (size_t i = 0; i < npix; ++i)   // per-channel 16-bin colour histograms
    for (int c = 0; c < 3; ++c) {
      const double v = std::clamp(static_cast<double>(rgb[3 * i + c]), 0.0, 1.0);
      d[64 + c * 16 + std::min(15, static_cast<int>(v * 16.0))] += inv_n;
    }
  double nrm = 0.0;
  for (double x : d) nrm += x * x;
  nrm = std::sqrt(nrm);
  if (nrm > 0.0)
    for (double& x : d) x /= nrm;
  return d;
}

double cosine_similarity(const std::vector<double>& a, const std::vector<double>& b) {
  double na = 0.0, nb = 0.0, dot = 0.0;
  for (size_t i = 0; i < a.size(); ++i) { na += a[i] * a[i]; nb += b[i] * b[i]; dot += a[i] * b[i]; }
  na = std::sqrt(na);
  nb = std::sqrt(nb);
  return (na == 0.0 || nb == 0.0) ? 0.0 : dot / (na * nb);
}

// ---- quality metrics (eval/metrics.cpp:72-96) ----------------------------------------------------
double psnr_db(const std::vector<float>& a, const float* b) {
  double sum = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = static_cast<double>(a[i]) - b[i];
    sum += d * d;
  }
  const double mse = sum / static_cast<double>(a.size());
  return mse == 0.0 ? std::numeric_limits<double>::infinity() : -10.0 * std::log10(mse);
}

double depth_l1_cm(const std::vector<float>& rendered, const float* sensor, const gsf_intrinsics& K) {
  double sum = 0.0;
  int n = 0;
  for (size_t i = 0; i < rendered.size(); ++i) {
    const double s = sensor[i];
    if (!(s > K.near_plane && s < K.far_plane)) continue;
    if (!(rendered[i] > 0.0f)) continue;
    sum += std::abs(static_cast<double>(rendered[i]) - s);
    ++n;
  }
  return n == 0 ? 0.0 : 100.0 * sum / n;
}

struct Keyframe {
  int32_t frame_id;
  double timestamp;
  gsf_pose pose;
  std::vector<double> descriptor;
  int32_t slot;
};

}  // namespace

struct gsf_slam_s {
  gsf_ctx ctx = nullptr;
  gsf_slam_cfg cfg{};
  bool have_map = false;
  std::vector<Keyframe> keyframes;
  std::vector<gsf_pose> trajectory;
  gsf_pose prev{}, prev_prev{};
  int32_t degraded = 0;
};

namespace {

// Window selection (tracker.cpp:86-117): the newest keyframe, up to recent_keyframes before it,
// then the most similar remaining ones (ties favour the newer keyframe), ba_window in total.
std::vector<int> select_window(const std::vector<Keyframe>& pool, const gsf_tracker_cfg& cfg) {
  const int n = static_cast<int>(pool.size());
  const int current = n - 1;
  std::vector<int> window = {current};
  std::vector<uint8_t> taken(n, 0);
  taken[current] = 1;
  for (int i = current - 1; i >= 0 && static_cast<int>(window.size()) < cfg.ba_window && current - i <= cfg.recent_keyframes;
       --i) {
    window.push_back(i);
    taken[i] = 1;
  }
  std::vector<std::pair<double, int>> rest;
  for (int i = 0; i < n; ++i)
    if (!taken[i]) rest.emplace_back(cosine_similarity(pool[i].descriptor, pool[current].descriptor), i);
  std::sort(rest.begin(), rest.end(), [](const auto& a, const auto& b) {
    return a.first != b.first ? a.first > b.first : a.second > b.second;
  });
  for (const auto& r : rest) {
    if (static_cast<int>(window.size()) >= cfg.ba_window) break;
    window.push_back(r.second);
  }
  return window;
}

// Render at `pose` against the keyframe's depth and score colour / depth (system.cpp:87-91).
int score_view(gsf_slam_s* s, const gsf_pose& pose, const float* rgb, const float* depth, double* psnr, double* l1) {
  const gsf_intrinsics& K = s->cfg.intrinsics;
  const size_t npix = static_cast<size_t>(K.width) * K.height;
  std::vector<float> color(3 * npix), ad(npix);
  gsf_render_out out{};
  out.color = color.data();
  out.alpha_depth = ad.data();
  const int rc = gsf_render(s->ctx, &pose, &K, depth, &s->cfg.mapper.raster, &out);
  if (rc != GSF_OK) return rc;
  *psnr = psnr_db(color, rgb);
  *l1 = depth_l1_cm(ad, depth, K);
  return GSF_OK;
}

#define SLAM_TRY(call)               \
  do {                               \
    const int rc_ = (call);          \
    if (rc_ != GSF_OK) return rc_;   \
  } while (0)

int add_keyframe(gsf_slam_s* s, int32_t index, double timestamp, const gsf_pose& pose, const float* rgb, const float* depth) {
  const gsf_intrinsics& K = s->cfg.intrinsics;
  Keyframe kf{index, timestamp, pose, compute_descriptor(rgb, K.width, K.height),
              1 + static_cast<int32_t>(s->keyframes.size())};
  SLAM_TRY(gsf_frame_upload(s->ctx, kf.slot, rgb, depth, K.width, K.height));
  s->keyframes.push_back(std::move(kf));
  return GSF_OK;
}

int bootstrap(gsf_slam_s* s, int32_t index, double timestamp, const float* rgb, const float* depth, gsf_frame_log* log) {
  const auto t0 = Clock::now();
  const gsf_pose origin{};   // the first camera anchors the world frame
  SLAM_TRY(add_keyframe(s, index, timestamp, origin, rgb, depth));
  int64_t count = 0;
  SLAM_TRY(gsf_initialize_map(s->ctx, s->keyframes[0].slot, &origin, &s->cfg.intrinsics, &s->cfg.mapper, &count));
  s->have_map = true;
  const int32_t slot = s->keyframes[0].slot;
  SLAM_TRY(gsf_map_step(s->ctx, &slot, &origin, 1, &s->cfg.intrinsics, &s->cfg.mapper, s->cfg.init_iterations, nullptr));
  log->map_ms = ms_since(t0);
  log->keyframe = 1;
  s->prev = s->prev_prev = origin;
  s->trajectory.push_back(origin);
  log->pose = origin;
  return score_view(s, origin, rgb, depth, &log->kf_psnr_db, &log->kf_depth_l1_cm);
}

int keyframe_cycle(gsf_slam_s* s, int32_t index, double timestamp, const float* rgb, const float* depth, gsf_frame_log* log) {
  const gsf_slam_cfg& cfg = s->cfg;
  log->keyframe = 1;
  SLAM_TRY(add_keyframe(s, index, timestamp, s->trajectory.back(), rgb, depth));
  const std::vector<int> win = select_window(s->keyframes, cfg.tracker);
  std::vector<int32_t> slots, ids;
  std::vector<gsf_pose> poses;
  for (int k : win) {
    slots.push_back(s->keyframes[k].slot);
    ids.push_back(s->keyframes[k].frame_id);
    poses.push_back(s->keyframes[k].pose);
  }
  const int32_t n = static_cast<int32_t>(win.size());
  auto t0 = Clock::now();
  SLAM_TRY(gsf_map_step(s->ctx, slots.data(), poses.data(), n, &cfg.intrinsics, &cfg.mapper, cfg.map_iterations, nullptr));
  log->map_ms = ms_since(t0);
  t0 = Clock::now();
  SLAM_TRY(gsf_sliding_ba(s->ctx, slots.data(), poses.data(), ids.data(), n, &cfg.intrinsics, &cfg.tracker, &cfg.mapper,
                          cfg.tracker.ba_iterations, nullptr));
  log->ba_ms = ms_since(t0);
  for (int i = 0; i < n; ++i) s->keyframes[win[i]].pose = poses[i];
  // the adjustment may have moved the incoming keyframe: trajectory and velocity model follow it
  s->trajectory.back() = s->keyframes.back().pose;
  s->prev = s->keyframes.back().pose;
  t0 = Clock::now();
  int32_t observed = 0, reduced = 0;
  SLAM_TRY(gsf_accumulate_uncertainty(s->ctx, slots.data(), poses.data(), n, &cfg.intrinsics, &cfg.mapper.raster, &observed));
  SLAM_TRY(gsf_prune_unreliable(s->ctx, cfg.mapper.uncertainty_tau, cfg.mapper.uncertainty_reduced_opacity, &reduced));
  log->uncertainty_ms = ms_since(t0);
  t0 = Clock::now();
  const Keyframe& cur = s->keyframes.back();
  SLAM_TRY(score_view(s, cur.pose, rgb, depth, &log->kf_psnr_db, &log->kf_depth_l1_cm));   // leaves the render for spawn
  int32_t spawned = 0;
  SLAM_TRY(gsf_spawn_gaussians(s->ctx, cur.slot, &cur.pose, &cfg.intrinsics, &cfg.mapper, &spawned));
  log->spawn_ms = ms_since(t0);
  log->pose = s->trajectory.back();
  return GSF_OK;
}

}  // namespace

extern "C" {

int gsf_slam_create(gsf_ctx ctx, const gsf_slam_cfg* cfg, gsf_slam* out) {
  if (!ctx || !cfg || !out) return GSF_EINVAL;
  const gsf_tracker_cfg& t = cfg->tracker;
  if (!(t.lr_rotation > 0.0) || !(t.lr_translation > 0.0) || t.iterations <= 0 || t.ba_window < 2 || t.ba_iterations < 0 || t.keyframe_interval < 1 || t.recent_keyframes < 0 ||
      !(t.degraded_loss_ratio > 1.0) || cfg->map_iterations < 0 || cfg->init_iterations < 0)
    return GSF_EINVAL;   // TrackerConfig::validate / MapperConfig::validate (tracker.cpp:12-24)
  auto* s = new gsf_slam_s;
  s->ctx = ctx;
  s->cfg = *cfg;
  s->cfg.mapper.seed = cfg->seed;   // the run seed drives every stochastic choice (system.cpp:20-24)
  *out = s;
  return GSF_OK;
}

int gsf_slam_destroy(gsf_slam s) {
  delete s;
  return GSF_OK;
}

int gsf_slam_process(gsf_slam s, int32_t index, double timestamp, const float* rgb, const float* depth, gsf_frame_log* log) {
  if (!s || !rgb || !depth || !log) return GSF_EINVAL;
  std::memset(log, 0, sizeof(*log));
  log->frame = index;
  log->timestamp = timestamp;
  const gsf_slam_cfg& cfg = s->cfg;
  if (!s->have_map) {
    SLAM_TRY(bootstrap(s, index, timestamp, rgb, depth, log));
  } else {
    const auto t0 = Clock::now();
    const gsf_pose predicted = s->trajectory.size() < 2 ? s->prev : predict_pose(s->prev, s->prev_prev);
    SLAM_TRY(gsf_frame_upload(s->ctx, 0, rgb, depth, cfg.intrinsics.width, cfg.intrinsics.height));
    gsf_track_result r{};
    SLAM_TRY(gsf_track_frame(s->ctx, 0, &predicted, &cfg.intrinsics, &cfg.tracker, &cfg.mapper.weights, &cfg.mapper.raster, &r));
    log->track_ms = ms_since(t0);
    log->track_loss = r.final_loss;
    log->track_iterations = r.iterations_run;
    log->track_degraded = r.degraded;
    if (r.degraded) ++s->degraded;
    s->prev_prev = s->prev;
    s->prev = r.pose;
    s->trajectory.push_back(r.pose);
    log->pose = r.pose;
    if (index % cfg.tracker.keyframe_interval == 0) SLAM_TRY(keyframe_cycle(s, index, timestamp, rgb, depth, log));
  }
  log->primitives = gsf_map_count(s->ctx);
  return GSF_OK;
}

int32_t gsf_slam_keyframes(gsf_slam s) { return s ? static_cast<int32_t>(s->keyframes.size()) : -1; }
int32_t gsf_slam_degraded_frames(gsf_slam s) { return s ? s->degraded : -1; }

}  // extern "C"
