// mirror.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain sequential CPU restatement of the device forward path, written in the structure of
// the reference (rasterizer.cpp:168-261: project_all -> global (depth, id) sort -> per-tile
// lists -> per-pixel front-to-back blend), but computing each per-primitive and per-pair
// value with the same explicitly-rounded arithmetic the sm_100a kernels use
// (paper_2403_16095_b200/csrc/gsf_shared.cuh).  It is therefore the bit-exact reference for
// the discrete outputs of the GPU pipeline (visible flags, depth order, tile lists/ranges,
// per-pixel counts, dominant/median ids) and for its fp32 pixel maps.  It shares arithmetic
// with the kernels, not structure: the kernels use a radix sort, a parallel scan/duplicate
// and a tile-CTA blend; the mirror uses std::sort and nested loops.
//
// The mirror is itself checked against the fp64 oracle (gsf_oracle.cpp) at tolerance in
// tests/test_oracle_mirror.py.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../paper_2403_16095_b200/csrc/gsf_shared.cuh"
#include "gsf_oracle.h"

using namespace gsfk;

extern "C" int mir_render(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
                          const float* obs, const gsf_raster_cfg* cfg, mir_out* out) {
  const int64_t P = map->count;
  const int Ks = map->sh_coeffs;
  const int D = 11 + 3 * Ks;
  // SoA fp32 [field][P], converted exactly as the device upload does.
  std::vector<float> soa(static_cast<size_t>(D) * P);
  for (int64_t i = 0; i < P; ++i) {
    for (int a = 0; a < 3; ++a) soa[a * P + i] = static_cast<float>(map->mean[3 * i + a]);
    for (int a = 0; a < 3; ++a) soa[(3 + a) * P + i] = static_cast<float>(map->log_scale[3 * i + a]);
    for (int a = 0; a < 4; ++a) soa[(6 + a) * P + i] = static_cast<float>(map->quat[4 * i + a]);
    soa[10 * P + i] = static_cast<float>(map->opacity_logit[i]);
    for (int b = 0; b < 3 * Ks; ++b) soa[(11 + b) * P + i] = static_cast<float>(map->sh[3 * Ks * i + b]);
  }
  const int W = K->width, H = K->height, ts = cfg->tile_size;
  RasterParams rp;
  rp.footprint_sigma = cfg->footprint_sigma;
  rp.dilation = cfg->dilation;
  rp.alpha_clamp = cfg->alpha_clamp;
  rp.alpha_skip = cfg->alpha_skip;
  rp.termination = cfg->termination_threshold;
  rp.tile = ts;
  rp.tiles_x = (W + ts - 1) / ts;
  rp.tiles_y = (H + ts - 1) / ts;
  rp.sh_coeffs = Ks;
  const Cam cam = make_cam(pose->rotation_tangent, pose->translation, K->fx, K->fy, K->cx, K->cy, W, H,
                           K->near_plane, K->far_plane);
  std::vector<PreOut> pre(P);
  std::vector<int32_t> vis;
  for (int64_t i = 0; i < P; ++i) {
    pre[i] = preprocess_one(&soa[i], P, cam, rp);
    if (out->visible) out->visible[i] = pre[i].visible ? 1 : 0;
    if (pre[i].visible) vis.push_back(static_cast<int32_t>(i));
  }
  std::sort(vis.begin(), vis.end(), [&](int32_t a, int32_t b) {
    return pre[a].depth < pre[b].depth || (pre[a].depth == pre[b].depth && a < b);
  });
  const int V = static_cast<int>(vis.size());
  out->num_visible = V;
  if (out->rank_to_id) std::memcpy(out->rank_to_id, vis.data(), sizeof(int32_t) * V);
  const int ntiles = rp.tiles_x * rp.tiles_y;
  std::vector<std::vector<int32_t>> lists(ntiles);
  for (int r = 0; r < V; ++r) {
    const PreOut& o = pre[vis[r]];
    for (int ty = o.ty0; ty <= o.ty1; ++ty)
      for (int tx = o.tx0; tx <= o.tx1; ++tx) lists[ty * rp.tiles_x + tx].push_back(r);
  }
  int64_t total = 0;
  for (int t = 0; t < ntiles; ++t) {
    if (out->tile_range) {   // empty tiles are [0, 0), as the device's memset leaves them
      out->tile_range[2 * t] = lists[t].empty() ? 0 : static_cast<int32_t>(total);
      out->tile_range[2 * t + 1] = lists[t].empty() ? 0 : static_cast<int32_t>(total + lists[t].size());
    }
    for (size_t j = 0; j < lists[t].size(); ++j) {
      if (out->pair_rank && total + static_cast<int64_t>(j) < out->pair_capacity) out->pair_rank[total + j] = lists[t][j];
    }
    total += static_cast<int64_t>(lists[t].size());
  }
  out->num_pairs = total;
  std::vector<BlendG> bg(V);
  std::vector<GuardG> gg(V);
  const BlendConsts kc = make_blend_consts(rp);
  for (int r = 0; r < V; ++r) {
    bg[r] = make_blend_g(pre[vis[r]]);
    blend_rho_bounds(bg[r], kc);
    gg[r] = make_guard_g(pre[vis[r]]);
  }
  int64_t flagged = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int tx = t % rp.tiles_x, ty = t / rp.tiles_x;
    for (int y = ty * ts; y < std::min(H, (ty + 1) * ts); ++y)
      for (int x = tx * ts; x < std::min(W, (tx + 1) * ts); ++x) {
        const size_t pi = static_cast<size_t>(y) * W + x;
        bool obs_valid = false;
        float ov = 0.0f;
        if (obs) {
          ov = obs[pi];
          const double d = ov;
          obs_valid = std::isfinite(d) && d > K->near_plane && d < K->far_plane;
        }
        PixelState s;
        pixel_init(s);
        const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
        for (size_t j = 0; j < lists[t].size() && !s.done; ++j) {
          const int r = lists[t][j];
          const PairEval e = eval_pair(px, py, bg[r], &gg[r], kc);
          if (!e.code) continue;
          pixel_accumulate(s, bg[r], e, vis[r], static_cast<int32_t>(j), obs_valid, ov, kc, true);
        }
        if (s.flag) {   // exact-decision fix-up: the pixel re-blended in fp64 (k_pixel_fixup)
          ExactPixel q;
          exact_init(q);
          for (size_t j = 0; j < lists[t].size() && !q.done; ++j) {
            const int r = lists[t][j];
            double a = 0.0;
            if (exact_alpha(static_cast<double>(px), static_cast<double>(py), gg[r], kc, &a))
              exact_accumulate(q, a, bg[r], vis[r], static_cast<int32_t>(j), obs_valid, static_cast<double>(ov), kc);
          }
          s.cr = static_cast<float>(q.cr); s.cg = static_cast<float>(q.cg); s.cb = static_cast<float>(q.cb);
          s.ad = static_cast<float>(q.ad); s.op = static_cast<float>(q.op); s.unc = static_cast<float>(q.unc);
          s.T = static_cast<float>(q.T); s.best = static_cast<float>(q.best);
          s.med_depth = static_cast<float>(q.med_depth);
          s.count = q.count; s.dominant = q.dominant; s.median = q.median; s.last = q.last;
          ++flagged;
        }
        if (out->color) { out->color[3 * pi] = s.cr; out->color[3 * pi + 1] = s.cg; out->color[3 * pi + 2] = s.cb; }
        if (out->alpha_depth) out->alpha_depth[pi] = s.ad;
        if (out->median_depth) out->median_depth[pi] = s.med_depth;
        if (out->median_valid) out->median_valid[pi] = s.median >= 0 ? 1 : 0;
        if (out->opacity) out->opacity[pi] = s.op;
        if (out->uncertainty) out->uncertainty[pi] = s.unc;
        if (out->final_transmittance) out->final_transmittance[pi] = s.T;
        if (out->per_pixel_count) out->per_pixel_count[pi] = s.count;
        if (out->dominant) out->dominant[pi] = s.dominant;
        if (out->median_prim) out->median_prim[pi] = s.median;
        if (out->dominant_weight) out->dominant_weight[pi] = s.best;
        if (out->last_index) out->last_index[pi] = s.last;
      }
  }
  out->num_flagged = flagged;
  return GSF_OK;
}

// Stress check of blend_rho_bounds (gsf_shared.cuh): n random primitives (fp64 mean2d anywhere in
// [-4000, 6000]^2 px, screen sigmas 0.3-300 px, any orientation, conditioning down to 1e-4, plus
// the reference's 0.3 px^2 dilation), every pixel centre of the bounding box of the cutoff ellipse
// (grown by 2 px; boxes wider than 600 px are row-sampled).  For each pixel the fp32 rho of the
// kernels is compared with the fp64 rho of the guard: a fast-path rho (< rho_fast) must be an fp64
// contribution, a rho above rho_hi an fp64 skip.  out[0] = violations, out[1] = max |rho_f - rho_d|
// / band_i where band_i is the primitive's own bound, out[2] = pixels tested, out[3] = pixels on the
// guard path, out[4] = max ratio where band_i is capped at the global band (far off-image means).
extern "C" int mir_band_check(int n, uint64_t seed, double* out) {
  uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  auto rnd = [&s]() {   // splitmix64 -> [0, 1)
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return static_cast<double>((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
  };
  RasterParams rp{};   // RasterConfig defaults (raster/config.hpp:5-16)
  rp.footprint_sigma = 3.0;
  rp.dilation = 0.3;
  rp.alpha_skip = 1.0 / 255.0;
  rp.alpha_clamp = 0.99;
  rp.termination = 1e-8;
  const BlendConsts kc = make_blend_consts(rp);
  double viol = 0, worst = 0, worst_capped = 0, tested = 0, guarded = 0;
  for (int i = 0; i < n; ++i) {
    const double mx = -4000.0 + 10000.0 * rnd(), my = -4000.0 + 10000.0 * rnd();
    const double s1 = 0.3 * std::pow(1000.0, rnd()), s2 = s1 * std::pow(1e-2, rnd()), th = 3.14159265358979 * rnd();
    const double cs = std::cos(th), sn = std::sin(th);
    const double cxx = cs * cs * s1 * s1 + sn * sn * s2 * s2 + 0.3, cyy = sn * sn * s1 * s1 + cs * cs * s2 * s2 + 0.3,
                 cxy = cs * sn * (s1 * s1 - s2 * s2);
    const double det = cxx * cyy - cxy * cxy;
    GuardG gg{mx, my, cyy / det, -cxy / det, cxx / det, 0.98};
    BlendG g{};
    g.mx = static_cast<float>(mx);
    g.my = static_cast<float>(my);
    g.sigma = 0.98f;
    g.c00 = static_cast<float>(gg.c00);
    g.c01x2 = static_cast<float>(2.0 * gg.c01);
    g.c11 = static_cast<float>(gg.c11);
    blend_rho_bounds(g, kc);
    const double band = static_cast<double>(g.rho_hi) - kc.cutoff_d;
    const bool capped = !(band < 0.999 * kc.rho_band);
    const double rx = std::sqrt(kc.cutoff_d * cxx) + 2.0, ry = std::sqrt(kc.cutoff_d * cyy) + 2.0;
    const int x0 = static_cast<int>(std::floor(mx - rx)), x1 = static_cast<int>(std::ceil(mx + rx));
    const int y0 = static_cast<int>(std::floor(my - ry)), y1 = static_cast<int>(std::ceil(my + ry));
    const int ystep = std::max(1, (y1 - y0) / 600), xstep = std::max(1, (x1 - x0) / 600);
    for (int y = y0; y <= y1; y += ystep)
      for (int x = x0; x <= x1; x += xstep) {
        const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
        const float rho = pair_rho(fsub(px, g.mx), fsub(py, g.my), g);
        const double rd = guard_rho(static_cast<double>(px), static_cast<double>(py), gg);
        tested += 1;
        if (std::fabs(rd - kc.cutoff_d) < 2.0 * band) {
          double& w = capped ? worst_capped : worst;
          w = std::max(w, std::fabs(rho - rd) / band);
        }
        if (rho > g.rho_hi) {
          if (!(rd > kc.cutoff_d || rd < 0.0)) viol += 1;
        } else if (rho < g.rho_fast) {
          if (!(rd <= kc.cutoff_d && rd >= 0.0)) viol += 1;
        } else {
          guarded += 1;
        }
      }
  }
  out[0] = viol;
  out[1] = worst;
  out[2] = tested;
  out[3] = guarded;
  out[4] = worst_capped;
  return 0;
}
