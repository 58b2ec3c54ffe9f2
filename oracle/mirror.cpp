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
    bg[r].rho_fast = blend_rho_fast(bg[r], kc);
    gg[r] = make_guard_g(pre[vis[r]]);
  }
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
          pixel_accumulate(s, bg[r], e, vis[r], static_cast<int32_t>(j), obs_valid, ov, kc);
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
  return GSF_OK;
}
