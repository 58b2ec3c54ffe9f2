// abi.cu — the C-ABI (include/gsf_cuda.h): context, map residency, and the device-resident
// render / render_backward / losses / track_frame / map_step / sliding_ba / uncertainty loops.
//
// Host responsibilities only: argument validation with the reference's exception messages,
// buffer residency, kernel sequencing on one stream, and turning device-side status flags
// (DevState) back into the reference's error semantics.  Every number is computed on the device.
#include <dlfcn.h>

#include <cstddef>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gsf_cuda.h"
#include "kernels.h"

using namespace gsfk;

namespace {

struct EInval : std::invalid_argument {
  explicit EInval(const std::string& s) : std::invalid_argument(s) {}
};
struct ENonFinite : std::invalid_argument {
  int64_t index;
  ENonFinite(const std::string& s, int64_t i) : std::invalid_argument(s), index(i) {}
};
struct EDiverged : std::runtime_error {
  explicit EDiverged(const std::string& s) : std::runtime_error(s) {}
};
struct ERuntime : std::runtime_error {
  explicit ERuntime(const std::string& s) : std::runtime_error(s) {}
};
struct EUnsupported : std::runtime_error {
  explicit EUnsupported(const std::string& s) : std::runtime_error(s) {}
};

// NCCL is opened at run time so the library has no link-time dependency on it.
struct NcclApi {
  void* h = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, const void*, int) = nullptr;  // ncclUniqueId passed by value (128 B)
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*get_error)(int) = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
    all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclAllReduce"));
    comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    get_error = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    group_start = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
    group_end = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
    return get_unique_id && all_reduce && comm_destroy;
  }
};
NcclApi g_nccl;
struct NcclUid { char b[128]; };
typedef int (*nccl_init_fn)(void**, int, NcclUid, int);

struct Frame {
  float* rgb = nullptr;
  float* depth = nullptr;
  int w = 0, h = 0;
};

// Per-keyframe pose + Adam state for sliding_ba / map_step, device resident.

}  // namespace

// A captured track_frame (all iterations + the final render) replayed while its inputs match.
struct TrackGraphKey {
  const float* rgb;
  const float* depth;
  const float* params;
  gsf_intrinsics K;
  gsf_raster_cfg rcfg;
  gsf_loss_weights w;
  int32_t iterations;
  int64_t P;
  int32_t sh;
  int64_t alloc_gen;
};
struct TrackGraph {
  bool valid = false;
  TrackGraphKey key{};
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;   // kernel launches one replay performs
};

struct gsf_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t err_index = -1;
  int64_t launches = 0;
  // map
  int64_t P = 0;
  int K = 1;
  int D = 14;
  int64_t map_cap = 0;
  int64_t map_gen = 0;
  float* params = nullptr;
  float* grads = nullptr;
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  double adam_step = 0.0;
  double* nu = nullptr;   // per-primitive uncertainty (fp64: prune compares it with tau exactly as the reference)
  uint8_t* observed = nullptr;
  float* d_mean2d = nullptr;
  double* grad_accum = nullptr;   // MapState::grad_accum (fp64 like the reference)
  int32_t* grad_count = nullptr;
  std::mt19937_64 rng;            // MapState::rng, seeded with the mapper seed at the first densify
  bool rng_seeded = false;
  int64_t map_iteration = 0;
  // device workspace + scalars
  Workspace ws;
  DevState* ds = nullptr;
  DevState* ds_host = nullptr;   // pinned shadow for staging / readback
  KfPose* kf = nullptr;
  KfPose* kf_host = nullptr;
  int kf_cap = 0;
  double* trace_dev = nullptr;
  int trace_cap = 0;
  double* unc_sum = nullptr;
  uint32_t* unc_cnt = nullptr;
  uint32_t* counters = nullptr;
  int64_t unc_cap = 0;
  std::vector<Frame> frames;
  // last render (for render_backward / loss API)
  bool have_render = false;
  int64_t render_gen = -1;
  gsf_intrinsics rK{};
  gsf_raster_cfg rcfg{};
  bool render_obs = false;
  // initialize / spawn scratch (per-CTA candidate counts and offsets + total)
  uint32_t* bp_scratch = nullptr;
  int64_t bp_cap = 0;
  // captured track_frame graphs (small round-robin cache)
  TrackGraph track_graphs[8];
  Frame track_in;   // graph-owned copy of the frame being tracked (one graph serves every frame slot)
  int track_graph_next = 0;
  bool use_graphs = true;
  // staging for host inputs
  float* stage = nullptr;
  size_t stage_bytes = 0;
  // comm: an NCCL communicator (gsf_comm_init) or a host-staged one (gsf_comm_init_host: the
  // caller's all-reduce over host memory, e.g. a gloo/MPI process group)
  void* comm = nullptr;
  gsf_host_allreduce_fn host_ar = nullptr;
  void* host_ar_user = nullptr;
  void* host_stage = nullptr;   // pinned staging of the host-staged all-reduce
  size_t host_stage_bytes = 0;
  cudaStream_t comm_stream = nullptr;   // NCCL buckets run here, overlapping the per-group Adam
  cudaEvent_t ev_grads = nullptr, ev_bucket[8] = {nullptr};
  double* ba_pack = nullptr;    // [loss sum, halt flag, 6 pose-gradient doubles per window keyframe]
  int ba_pack_cap = 0;
  int nranks = 1, rank = 0;
  float* red_f = nullptr;   // allreduce scratch for the loss sum
  Profiler prof;
  cudaEvent_t ev[8] = {nullptr};
};

namespace {

// Device buffers come from the device's stream-ordered memory pool (cudaMallocAsync on the calling
// context's stream, release threshold unlimited): a map that grows by spawning or densification
// re-uses freed blocks instead of paying cudaMalloc/cudaFree (and cudaFree's device-wide sync) for
// every buffer.  dalloc waits for its stream so the new block is usable from any stream at once.
thread_local cudaStream_t g_alloc_stream = nullptr;

template <class T>
void dfree(T*& p) {
  if (p) cudaFreeAsync(p, g_alloc_stream);
  p = nullptr;
}

// Bumped by every device (re)allocation: captured CUDA graphs hold raw buffer pointers.
int64_t g_alloc_gen = 0;

template <class T>
void dalloc(T*& p, size_t count) {
  dfree(p);
  if (count == 0) count = 1;
  GSF_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, g_alloc_stream));
  GSF_CUDA_CHECK(cudaStreamSynchronize(g_alloc_stream));
  ++g_alloc_gen;
}

void keep_pool_memory(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
  uint64_t threshold = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
}

void check_intrinsics(const gsf_intrinsics& k) {   // camera.hpp:20-26
  if (!(k.fx > 0.0) || !(k.fy > 0.0)) throw EInval("intrinsics: focal lengths must be positive");
  if (k.width <= 0 || k.height <= 0) throw EInval("intrinsics: image size must be positive");
  if (!(k.depth_scale > 0.0)) throw EInval("intrinsics: depth_scale must be positive");
  if (!(k.near_plane > 0.0) || !(k.far_plane > k.near_plane)) throw EInval("intrinsics: need 0 < near < far");
}

void check_raster(const gsf_raster_cfg& c) {
  if (c.tile_size != kTile)
    throw EUnsupported("raster.tile_size " + std::to_string(c.tile_size) + " is not supported on the device path (16 only)");
}

void check_weights(const gsf_loss_weights& w) {   // losses.cpp:49-56
  const double all[] = {w.w_color, w.w_ssim, w.w_geo, w.w_align, w.w_iso, w.w_var, w.t_color, w.t_geo};
  for (double v : all)
    if (!(v >= 0.0)) throw EInval("loss weights must be non-negative");
  if (!(w.iso_epsilon >= 1.0)) throw EInval("iso epsilon must be >= 1");
  if (!(w.opacity_floor >= 0.0 && w.opacity_floor <= 1.0)) throw EInval("opacity floor must lie in [0,1]");
}

RasterParams make_rp(const gsf_ctx_s* c, const gsf_intrinsics& k, const gsf_raster_cfg& cfg) {
  RasterParams rp;
  rp.footprint_sigma = cfg.footprint_sigma;
  rp.dilation = cfg.dilation;
  rp.alpha_clamp = cfg.alpha_clamp;
  rp.alpha_skip = cfg.alpha_skip;
  rp.termination = cfg.termination_threshold;
  rp.tile = kTile;
  rp.tiles_x = (k.width + kTile - 1) / kTile;
  rp.tiles_y = (k.height + kTile - 1) / kTile;
  rp.sh_coeffs = c->K;
  return rp;
}

LossParams make_lp(int mode, const gsf_loss_weights* w, const gsf_raster_cfg& cfg) {
  LossParams lp{};
  lp.mode = mode;
  lp.uncertainty_full_gradient = cfg.uncertainty_full_gradient;
  if (w) {
    lp.opacity_floor = static_cast<float>(w->opacity_floor);
    lp.normalize_by_valid = w->normalize_by_valid;
    lp.w_color = w->w_color; lp.w_ssim = w->w_ssim; lp.w_geo = w->w_geo; lp.w_align = w->w_align;
    lp.w_iso = w->w_iso; lp.w_var = w->w_var; lp.t_color = w->t_color; lp.t_geo = w->t_geo;
    lp.iso_epsilon = w->iso_epsilon;
  }
  return lp;
}

Cam host_cam(const gsf_pose& p, const gsf_intrinsics& k) {
  return make_cam(p.rotation_tangent, p.translation, k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.near_plane, k.far_plane);
}

void* stage(gsf_ctx_s* c, size_t bytes) {
  if (bytes > c->stage_bytes) {
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    GSF_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&c->stage), bytes));
    c->stage_bytes = bytes;
  }
  return c->stage;
}

void sync(gsf_ctx_s* c) {
  GSF_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->prof.resolve();
}

void read_state(gsf_ctx_s* c) {
  GSF_CUDA_CHECK(cudaMemcpyAsync(c->ds_host, c->ds, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// Reset the per-call scalars; cam is written from the host shadow.
void reset_state(gsf_ctx_s* c, const Cam* cam) {
  DevState& h = *c->ds_host;
  std::memset(&h, 0, sizeof(DevState));
  h.bad_index = std::numeric_limits<int32_t>::max();
  if (cam) h.cam = *cam;
  GSF_CUDA_CHECK(cudaMemcpyAsync(c->ds, &h, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
}

void ensure_map(gsf_ctx_s* c, int64_t P, int K) {
  const int D = kFieldsBase + 3 * K;
  if (P * D > c->map_cap * c->D || P > c->map_cap || !c->params) {
    const int64_t cap = std::max<int64_t>(P, 1);
    dalloc(c->params, static_cast<size_t>(cap) * D);
    dalloc(c->grads, static_cast<size_t>(cap) * D);
    dalloc(c->adam_m, static_cast<size_t>(cap) * D);
    dalloc(c->adam_v, static_cast<size_t>(cap) * D);
    dalloc(c->nu, cap);
    dalloc(c->observed, cap);
    dalloc(c->d_mean2d, 2 * cap);
    dalloc(c->grad_accum, cap);
    dalloc(c->grad_count, cap);
    c->map_cap = cap;
  }
  c->P = P;
  c->K = K;
  c->D = D;
}

void alloc_pairs(Workspace& ws) {

  dalloc(ws.skey, ws.pair_cap); dalloc(ws.sid, ws.pair_cap);
  dalloc(ws.sslot, ws.pair_cap); dalloc(ws.qlist, 4 * ws.pair_cap);
  dalloc(ws.partials, ws.pair_cap * 10);
  // [pair][4 quadrants][10] (k_backward_q) + a written-flag byte per (pair, quadrant): k_pair_combine
  // reads the flagged slots and clears the flags, so they start cleared
  dalloc(ws.qpart, ws.pair_cap * 40);
  dalloc(ws.qflag, ws.pair_cap);
  GSF_CUDA_CHECK(cudaMemset(ws.qflag, 0, sizeof(uint32_t) * ws.pair_cap));
}

void ensure_ws(gsf_ctx_s* c, int W, int H) {
  Workspace& ws = c->ws;
  const int64_t P = std::max<int64_t>(c->P, 1);
  const int64_t npix = static_cast<int64_t>(W) * H;
  const int64_t tiles = static_cast<int64_t>((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile);
  if (P > ws.P_cap) {
    const int64_t Pc = P + P / 4 + 4096;   // headroom: a growing map (spawn, densify) rarely reallocates
    dalloc(ws.bg_id, Pc); dalloc(ws.gg_id, Pc); dalloc(ws.bg_slot, Pc); dalloc(ws.gg_slot, Pc); dalloc(ws.cand, Pc); dalloc(ws.depth_id, Pc); dalloc(ws.rect_id, Pc); dalloc(ws.visible, Pc);
    dalloc(ws.pj_id, static_cast<size_t>(Pc) * kPjFloats);
    dalloc(ws.big_ids, Pc);
    dalloc(ws.vis_list, Pc);
    dalloc(ws.pair_base, Pc);
    dalloc(ws.pj_slot, Pc);
    dalloc(ws.world, Pc);
    dalloc(ws.support, Pc);
    ws.P_cap = Pc;
    dfree(ws.pose_part);
  }
  if (ws.pair_cap == 0) ws.pair_cap = std::max<int64_t>(1 << 20, 4 * P);
  if (!ws.skey) alloc_pairs(ws);
  if (npix > ws.npix_cap) {
    dalloc(ws.color, 3 * npix); dalloc(ws.alpha_depth, npix); dalloc(ws.median_depth, npix); dalloc(ws.median_valid, npix);
    dalloc(ws.opacity, npix); dalloc(ws.uncertainty, npix); dalloc(ws.final_T, npix); dalloc(ws.count, npix);
    dalloc(ws.dominant, npix); dalloc(ws.median_prim, npix); dalloc(ws.dominant_w, npix); dalloc(ws.last, npix); dalloc(ws.lastc, npix);
    dalloc(ws.pxcode, npix);
    dalloc(ws.fix_list, npix);
    dalloc(ws.obs, npix); dalloc(ws.upstream, 7 * npix); dalloc(ws.dssim, 3 * npix); dalloc(ws.ssim_tmp, 9 * npix);
    ws.npix_cap = npix;
  }
  if (tiles > ws.tiles_cap) {
    dalloc(ws.ranges, tiles);
    dalloc(ws.bins, tiles * kBinStride + kCntNum);
    ws.tile_fill = ws.bins;
    ws.bin_counters = ws.bins + tiles * kBinStride;
    dfree(ws.bucket);
    dalloc(ws.loss_part, (5 * tiles + 64) * LS_NUM);
    dalloc(ws.order, 2 * (1 + 5 * tiles));
    dalloc(ws.qstat, 4 * tiles);
    GSF_CUDA_CHECK(cudaMemsetAsync(ws.order, 0, sizeof(uint32_t) * 2 * (1 + 5 * tiles), c->stream));
    ws.tiles_cap = tiles;
    dfree(ws.pose_part);
  }
  if (ws.bucket_cap == 0) ws.bucket_cap = 2048;
  if (!ws.bucket) dalloc(ws.bucket, static_cast<size_t>(ws.tiles_cap) * ws.bucket_cap);
  if (!ws.pose_part) {
    dalloc(ws.pose_part, static_cast<size_t>(std::max<int64_t>(div_up(ws.P_cap, 256), 5 * ws.tiles_cap + 64)) * 6);
    ws.wtickets_half = ws.tiles_cap / 8 + 8;   // groups of 32 rows over 4 rows per tile, + the top ticket
    dalloc(ws.wtickets, 2 * ws.wtickets_half);
    GSF_CUDA_CHECK(cudaMemsetAsync(ws.wtickets, 0, sizeof(uint32_t) * 2 * ws.wtickets_half, c->stream));
  }
  const int64_t red = 2 * std::max<int64_t>(div_up(npix, 256), div_up(P, 256)) + 64;
  if (!ws.red_part || ws.red_iso_offset * 2 < red) {
    dalloc(ws.red_part, red);
    ws.red_iso_offset = red / 2;
  }
  if (!c->counters) dalloc(c->counters, 16);
}

// After an overflow: grow the pair lists and/or the per-tile buckets to fit the largest render
// since the last reset (DevState::M_max / max_tile are maxima over a whole loop's renders).
void grow_pairs(gsf_ctx_s* c, uint32_t needed) {
  Workspace& ws = c->ws;
  if (needed > ws.pair_cap) {
    ws.pair_cap = static_cast<int64_t>(needed) + needed / 4 + 1024;
    alloc_pairs(ws);
  }
  const int64_t longest = c->ds_host->max_tile;
  if (longest > ws.bucket_cap) {
    while (ws.bucket_cap < longest + longest / 4) ws.bucket_cap *= 2;
    dalloc(ws.bucket, static_cast<size_t>(ws.tiles_cap) * ws.bucket_cap);
  }
}

// Still overflowed after the growth retries: the tile lists were truncated, so no result is returned.
void check_overflow(gsf_ctx_s* c, const char* what) {
  if (c->ds_host->overflow)
    throw EUnsupported(std::string(what) + ": pair capacity still exceeded after growing (" +
                       std::to_string(c->ds_host->M_max) + " pairs, longest tile list " +
                       std::to_string(c->ds_host->max_tile) + ")");
}

FwdArgs fwd_args(gsf_ctx_s* c, const gsf_intrinsics& k, const gsf_raster_cfg& cfg, const float* obs, const float* loss_rgb,
                 const float* loss_depth, const LossParams& lp, int iteration) {
  FwdArgs a;
  a.params = c->params;
  a.P = c->P;
  a.K = c->K;
  a.rp = make_rp(c, k, cfg);
  a.kc = make_blend_consts(a.rp);
  a.W = k.width;
  a.H = k.height;
  a.near_plane = k.near_plane;
  a.far_plane = k.far_plane;
  a.obs = obs;
  a.loss_rgb = loss_rgb;
  a.loss_depth = loss_depth;
  a.lp = lp;
  a.iteration = iteration;
  return a;
}

BwdArgs bwd_args(gsf_ctx_s* c, const gsf_intrinsics& k, const gsf_raster_cfg& cfg, const float* obs, const float* target,
                 const LossParams& lp, int seed_mode, bool pose_only) {
  BwdArgs b{};
  b.params = c->params;
  b.P = c->P;
  b.K = c->K;
  b.rp = make_rp(c, k, cfg);
  b.kc = make_blend_consts(b.rp);
  b.W = k.width;
  b.H = k.height;
  b.near_plane = k.near_plane;
  b.far_plane = k.far_plane;
  b.obs = obs;
  b.target_rgb = target;
  b.lp = lp;
  b.seed_mode = seed_mode;
  b.pose_only = pose_only;
  b.grads = c->grads;
  b.d_mean2d = c->d_mean2d;
  return b;
}

void throw_nonfinite(int32_t idx) {
  throw ENonFinite("render: primitive " + std::to_string(idx) + " has non-finite parameters", idx);
}

// One device render with the overflow-retry protocol (API path, synchronous).
void render_sync(gsf_ctx_s* c, const gsf_pose& pose, const gsf_intrinsics& k, const gsf_raster_cfg& cfg, const float* obs_dev) {
  ensure_ws(c, k.width, k.height);
  const Cam cam = host_cam(pose, k);
  for (int attempt = 0; attempt < 3; ++attempt) {
    reset_state(c, &cam);
    c->ds_host->has_obs = obs_dev ? 1 : 0;
    GSF_CUDA_CHECK(cudaMemcpyAsync(&c->ds->has_obs, &c->ds_host->has_obs, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    run_forward(c->ws, c->ds, fwd_args(c, k, cfg, obs_dev, nullptr, nullptr, make_lp(0, nullptr, cfg), -1), c->stream, &c->launches);
    read_state(c);
    if (c->ds_host->bad_index != std::numeric_limits<int32_t>::max()) throw_nonfinite(c->ds_host->bad_index);
    if (!c->ds_host->overflow) break;
    grow_pairs(c, c->ds_host->M_max);
  }
  check_overflow(c, "render");
  c->have_render = true;
  c->render_gen = c->map_gen;
  c->rK = k;
  c->rcfg = cfg;
  c->render_obs = obs_dev != nullptr;
}

void upload_floats(gsf_ctx_s* c, float* dst, const float* src, size_t n) {
  GSF_CUDA_CHECK(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
}

template <class F>
int guard(gsf_ctx c, F&& f) {
  if (!c) return GSF_EINVAL;
  c->err.clear();
  c->err_index = -1;
  try {
    cudaSetDevice(c->device);
    g_alloc_stream = c->stream;
    f();
    return GSF_OK;
  } catch (const ENonFinite& e) {
    c->err = e.what();
    c->err_index = e.index;
    return GSF_ENONFINITE;
  } catch (const EInval& e) {
    c->err = e.what();
    return GSF_EINVAL;
  } catch (const EDiverged& e) {
    c->err = e.what();
    return GSF_EDIVERGED;
  } catch (const EUnsupported& e) {
    c->err = e.what();
    return GSF_EUNSUPPORTED;
  } catch (const ERuntime& e) {
    c->err = e.what();
    return GSF_ERUNTIME;
  } catch (const CudaError& e) {
    std::ostringstream m;
    m << "CUDA error " << cudaGetErrorName(e.code) << " (" << cudaGetErrorString(e.code) << ") at " << e.file << ":"
      << e.line << " in " << e.expr;
    c->err = m.str();
    return GSF_ECUDA;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return GSF_ENOMEM;
  } catch (const std::exception& e) {
    c->err = e.what();
    return GSF_EINVAL;
  }
}

const Frame& get_frame(gsf_ctx_s* c, int slot, const gsf_intrinsics& k) {
  if (slot < 0 || slot >= static_cast<int>(c->frames.size()) || !c->frames[slot].rgb)
    throw EInval("frame slot " + std::to_string(slot) + " is empty");
  const Frame& f = c->frames[slot];
  if (f.w != k.width || f.h != k.height) throw EInval("loss: target rgb dimensions mismatch");
  return f;
}

void ensure_kf(gsf_ctx_s* c, int n) {
  if (n <= c->kf_cap) return;
  dfree(c->kf);
  if (c->kf_host) cudaFreeHost(c->kf_host);
  dalloc(c->kf, n);
  GSF_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&c->kf_host), sizeof(KfPose) * n));
  c->kf_cap = n;
}

void ensure_trace(gsf_ctx_s* c, int n) {
  if (n <= c->trace_cap) return;
  dalloc(c->trace_dev, n);
  c->trace_cap = n;
}

}  // namespace

// ---- small device helpers used by the loops ---------------------------------------------------
namespace {

__global__ void k_set_cam_from_kf(DevState* ds, const KfPose* kf, int k, int has_obs) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  const Cam old = ds->cam;
  ds->cam = make_cam(kf[k].rot, kf[k].trans, old.fx, old.fy, old.cx, old.cy, old.width, old.height, old.near_plane,
                     old.far_plane);
  ds->has_obs = has_obs;
}


__global__ void k_store(const double* src, double* dst) { *dst = *src; }

// Sharded sliding_ba: everything a rank contributes besides the Gaussian gradients, packed into one
// fp64 buffer for a single all-reduce — the window loss sum, a divergence flag (so every rank halts
// at the same iteration) and the six pose-gradient components of each window keyframe (zero for
// keyframes another rank owns).
__global__ void k_ba_pack(const DevState* ds, const KfPose* kf, int n, const double* loss_acc, double* pack) {
  for (int i = threadIdx.x; i < 6 * n; i += blockDim.x) pack[2 + i] = kf[i / 6].grad[i % 6];
  if (threadIdx.x == 0) {
    pack[0] = *loss_acc;
    pack[1] = ds->halt == 2 ? 1.0 : 0.0;
  }
}
__global__ void k_ba_unpack(DevState* ds, KfPose* kf, int n, double* loss_acc, const double* pack, int it) {
  for (int i = threadIdx.x; i < 6 * n; i += blockDim.x) kf[i / 6].grad[i % 6] = pack[2 + i];
  if (threadIdx.x == 0) {
    *loss_acc = pack[0];
    if (pack[1] > 0.0 && ds->halt != 2) {
      ds->halt = 2;
      ds->halt_iter = it;
      ds->loss_total = pack[0];
    }
  }
}

// Pose Adam + perturbed for every non-anchor keyframe (tracker.cpp:168-179).
__global__ void k_kf_update(DevState* ds, KfPose* kf, int n, int anchor, double lr_rot, double lr_trans) {
  const int k = threadIdx.x;
  if (k >= n || k == anchor || ds->halt) return;
  KfPose& p = kf[k];
  p.t += 1.0;
  const double bc1 = 1.0 - pow(0.9, p.t), bc2 = 1.0 - pow(0.999, p.t);
  double delta[6];
  for (int a = 0; a < 6; ++a) {
    const double g = p.grad[a];
    p.m[a] = 0.9 * p.m[a] + (1.0 - 0.9) * g;
    p.v[a] = 0.999 * p.v[a] + (1.0 - 0.999) * g * g;
    delta[a] = 0.0 - (a < 3 ? lr_rot : lr_trans) * (p.m[a] / bc1) / (sqrt(p.v[a] / bc2) + 1e-8);
  }
  double dR[9], Rc[9], Rn[9];
  exp_map_d(delta, dR);
  exp_map_d(p.rot, Rc);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rn[3 * i + j] = dR[3 * i] * Rc[j] + dR[3 * i + 1] * Rc[3 + j] + dR[3 * i + 2] * Rc[6 + j];
  double tn[3];
  for (int i = 0; i < 3; ++i) tn[i] = dR[3 * i] * p.trans[0] + dR[3 * i + 1] * p.trans[1] + dR[3 * i + 2] * p.trans[2] + delta[3 + i];
  // log_map (lie.cpp:30-52)
  const double trace = Rn[0] + Rn[4] + Rn[8];
  double ct = (trace - 1.0) * 0.5;
  ct = ct < -1.0 ? -1.0 : (ct > 1.0 ? 1.0 : ct);
  const double th = acos(ct);
  const double vee[3] = {Rn[7] - Rn[5], Rn[2] - Rn[6], Rn[3] - Rn[1]};
  double out[3];
  if (th < 1e-8) {
    const double f = 0.5 * (1.0 + th * th / 6.0);
    for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
  } else if (th > M_PI - 1e-3) {
    double o[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) o[3 * i + j] = (0.5 * (Rn[3 * i + j] + Rn[3 * j + i]) - ct * (i == j ? 1.0 : 0.0)) / (1.0 - ct);
    int a = 0;
    for (int i = 1; i < 3; ++i)
      if (o[4 * i] > o[4 * a]) a = i;
    const double sq = sqrt(o[4 * a]);
    double ax[3] = {o[a] / sq, o[3 + a] / sq, o[6 + a] / sq};
    if (ax[0] * vee[0] + ax[1] * vee[1] + ax[2] * vee[2] < 0.0)
      for (int i = 0; i < 3; ++i) ax[i] = -ax[i];
    for (int i = 0; i < 3; ++i) out[i] = th * ax[i];
  } else {
    const double f = th / (2.0 * sin(th));
    for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
  }
  for (int i = 0; i < 3; ++i) { p.rot[i] = out[i]; p.trans[i] = tn[i]; }
}

__global__ void k_gather_grads_aos(const float* __restrict__ g, int64_t P, int K, const float* __restrict__ m2d,
                                   float* __restrict__ out) {
  // out: per primitive [mean3, ls3, quat4, op1, sh 3K, mean2d 2] contiguous (AoS, for download)
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int D = kFieldsBase + 3 * K;
  float* o = out + i * (D + 2);
  for (int f = 0; f < D; ++f) o[f] = g[f * P + i];
  o[D] = m2d[i];
  o[D + 1] = m2d[P + i];
}

__global__ void k_scatter_map_soa(const double* __restrict__ in, int64_t P, int K, float* __restrict__ params) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int D = kFieldsBase + 3 * K;
  for (int f = 0; f < D; ++f) params[f * P + i] = static_cast<float>(in[i * D + f]);
}

__global__ void k_gather_map_aos(const float* __restrict__ params, int64_t P, int K, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int D = kFieldsBase + 3 * K;
  for (int f = 0; f < D; ++f) out[i * D + f] = params[f * P + i];
}

__global__ void k_add_d(double* acc, const double* v) { *acc += *v; }

// CSR record of the last render (rasterizer.cpp:240-259): per-pixel contributors front to back.
__global__ void k_record(const int2* __restrict__ ranges, const uint32_t* __restrict__ sid,
                         const BlendG* __restrict__ bg, const GuardG* __restrict__ gg, const int32_t* __restrict__ last, const uint32_t* __restrict__ row_start, int W, int H, int tiles_x,
                         BlendConsts kc, int32_t* __restrict__ prim, float* __restrict__ alpha, float* __restrict__ trans) {
  const int64_t pi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pi >= static_cast<int64_t>(W) * H) return;
  const int x = static_cast<int>(pi % W), y = static_cast<int>(pi / W);
  const int tile = (y / kTile) * tiles_x + (x / kTile);
  const int2 rg = ranges[tile];
  const int lim = last[pi];
  const float px = x + 0.5f, py = y + 0.5f;
  uint32_t out = row_start[pi];
  float T = 1.0f;
  for (int j = 0; j < lim; ++j) {
    const int id = static_cast<int>(sid[rg.x + j]);
    const PairEval e = eval_pair(px, py, bg[id], gg + id, kc);
    if (!e.code) continue;
    prim[out] = id;
    alpha[out] = e.alpha;
    trans[out] = T;
    ++out;
    T = fmul(T, fsub(1.0f, e.alpha));
  }
}

}  // namespace

// =================================================================================================
extern "C" {

int gsf_abi_version(void) { return GSF_ABI_VERSION; }

int gsf_ctx_create(int device, gsf_ctx* out) {
  if (!out) return GSF_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) return GSF_ECUDA;
  auto* c = new gsf_ctx_s;
  c->device = device;
  c->use_graphs = std::getenv("GSF_NO_GRAPHS") == nullptr;   // eager launches for debugging
  const int rc = guard(c, [&] {
    GSF_CUDA_CHECK(cudaSetDevice(device));
    GSF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    GSF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->ws.side, cudaStreamNonBlocking));
    GSF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ws.ev_fork, cudaEventDisableTiming));
    GSF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ws.ev_join, cudaEventDisableTiming));
    GSF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->ws.side2, cudaStreamNonBlocking));
    GSF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ws.ev_lfork, cudaEventDisableTiming));
    GSF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ws.ev_ljoin, cudaEventDisableTiming));
    g_alloc_stream = c->stream;
    keep_pool_memory(device);
    dalloc(c->ds, 1);
    GSF_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&c->ds_host), sizeof(DevState)));
    reset_state(c, nullptr);
    sync(c);
  });
  if (rc != GSF_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return GSF_OK;
}

int gsf_ctx_destroy(gsf_ctx c) {
  if (!c) return GSF_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (TrackGraph& g : c->track_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->comm && g_nccl.comm_destroy) g_nccl.comm_destroy(c->comm);
  Workspace& ws = c->ws;
  void* bufs[] = {ws.bg_id, ws.gg_id, ws.bg_slot, ws.gg_slot, ws.sslot, ws.qlist, ws.lastc, ws.cand, ws.depth_id, ws.rect_id, ws.visible, ws.bins,
                  ws.bucket, ws.skey, ws.sid, ws.big_ids, ws.vis_list, ws.pair_base, ws.pj_slot, ws.world, ws.support, ws.partials, ws.ranges, ws.loss_part, ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid,
                  ws.opacity, ws.uncertainty, ws.final_T, ws.count, ws.dominant, ws.median_prim, ws.dominant_w,
                  ws.last, ws.pxcode, ws.fix_list, ws.order, ws.qstat, ws.obs, ws.upstream, ws.dssim, ws.ssim_tmp, ws.pose_part, ws.wtickets, ws.pj_id, ws.qflag, ws.qpart,
                  ws.red_part, c->bp_scratch, c->params, c->grads, c->adam_m, c->adam_v, c->nu, c->observed, c->d_mean2d,
                  c->grad_accum, c->grad_count, c->ds, c->kf, c->trace_dev, c->unc_sum, c->unc_cnt, c->counters,
                  c->red_f, c->ba_pack};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, c->stream);
  if (c->track_in.rgb) cudaFreeAsync(c->track_in.rgb, c->stream);
  if (c->track_in.depth) cudaFreeAsync(c->track_in.depth, c->stream);
  for (Frame& f : c->frames) {
    if (f.rgb) cudaFreeAsync(f.rgb, c->stream);
    if (f.depth) cudaFreeAsync(f.depth, c->stream);
  }
  cudaStreamSynchronize(c->stream);
  if (c->ds_host) cudaFreeHost(c->ds_host);
  if (c->kf_host) cudaFreeHost(c->kf_host);
  if (c->stage) cudaFreeHost(c->stage);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  if (c->ev_grads) cudaEventDestroy(c->ev_grads);
  for (cudaEvent_t e : c->ev_bucket)
    if (e) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (ws.ev_fork) cudaEventDestroy(ws.ev_fork);
  if (ws.ev_join) cudaEventDestroy(ws.ev_join);
  if (ws.side) cudaStreamDestroy(ws.side);
  if (ws.ev_lfork) cudaEventDestroy(ws.ev_lfork);
  if (ws.ev_ljoin) cudaEventDestroy(ws.ev_ljoin);
  if (ws.side2) cudaStreamDestroy(ws.side2);
  cudaStreamDestroy(c->stream);
  delete c;
  return GSF_OK;
}

const char* gsf_last_error(gsf_ctx c) { return c ? c->err.c_str() : "null context"; }
int64_t gsf_last_error_index(gsf_ctx c) { return c ? c->err_index : -1; }
int64_t gsf_kernel_launches(gsf_ctx c) { return c ? c->launches : 0; }

int gsf_reserve(gsf_ctx c, int64_t pair_cap, int64_t bucket_cap) {
  return guard(c, [&] {
    if (pair_cap < 0 || bucket_cap < 0 || pair_cap > (int64_t{1} << 31) || bucket_cap > (int64_t{1} << 24))
      throw EInval("reserve: capacity out of range");
    sync(c);
    Workspace& ws = c->ws;
    if (pair_cap > 0 && pair_cap != ws.pair_cap) {
      ws.pair_cap = std::max<int64_t>(pair_cap, 64);
      if (ws.skey) alloc_pairs(ws);
    }
    if (bucket_cap > 0 && bucket_cap != ws.bucket_cap) {
      ws.bucket_cap = std::max<int64_t>(bucket_cap, 32);
      if (ws.bucket) dalloc(ws.bucket, static_cast<size_t>(ws.tiles_cap) * ws.bucket_cap);
    }
  });
}

int gsf_capacity(gsf_ctx c, int64_t* pair_cap, int64_t* bucket_cap) {
  return guard(c, [&] {
    if (pair_cap) *pair_cap = c->ws.pair_cap;
    if (bucket_cap) *bucket_cap = c->ws.bucket_cap;
  });
}

int64_t gsf_track_candidates(gsf_ctx c) {
  if (!c) return -1;
  int64_t n = -1;
  const int rc = guard(c, [&] {
    read_state(c);
    n = static_cast<int64_t>(c->ds_host->ncand);
  });
  return rc == GSF_OK ? n : -1;
}
int gsf_synchronize(gsf_ctx c) {
  return guard(c, [&] { sync(c); });
}

int gsf_map_upload(gsf_ctx c, const gsf_map_host* m) {
  return guard(c, [&] {
    if (!m || m->count < 0) throw EInval("map: negative primitive count");
    const int K = m->sh_coeffs;
    if (K != 0 && K != 1 && K != 4 && K != 9 && K != 16) throw EInval("sh coefficient count must be 1, 4, 9 or 16");
    const int64_t P = m->count;
    ensure_map(c, P, K);
    const int D = c->D;
    double* h = static_cast<double*>(stage(c, sizeof(double) * std::max<int64_t>(P, 1) * D));
    for (int64_t i = 0; i < P; ++i) {
      double* o = h + i * D;
      for (int a = 0; a < 3; ++a) o[a] = m->mean[3 * i + a];
      for (int a = 0; a < 3; ++a) o[3 + a] = m->log_scale[3 * i + a];
      for (int a = 0; a < 4; ++a) o[6 + a] = m->quat[4 * i + a];
      o[10] = m->opacity_logit[i];
      for (int b = 0; b < 3 * K; ++b) o[11 + b] = m->sh[3 * K * i + b];
    }
    if (P > 0) {
      double* tmp = nullptr;
      GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&tmp), sizeof(double) * P * D));
      GSF_CUDA_CHECK(cudaMemcpyAsync(tmp, h, sizeof(double) * P * D, cudaMemcpyHostToDevice, c->stream));
      k_scatter_map_soa<<<div_up(P, 256), 256, 0, c->stream>>>(tmp, P, K, c->params);
      ++c->launches;
      sync(c);
      cudaFree(tmp);
      std::vector<double> nu(P, 0.0);
      std::vector<uint8_t> ob(P, 0);
      for (int64_t i = 0; i < P; ++i) {
        if (m->uncertainty) nu[i] = m->uncertainty[i];
        if (m->observed) ob[i] = m->observed[i];
      }
      GSF_CUDA_CHECK(cudaMemcpy(c->nu, nu.data(), sizeof(double) * P, cudaMemcpyHostToDevice));
      GSF_CUDA_CHECK(cudaMemcpy(c->observed, ob.data(), P, cudaMemcpyHostToDevice));
      GSF_CUDA_CHECK(cudaMemset(c->adam_m, 0, sizeof(float) * P * D));
      GSF_CUDA_CHECK(cudaMemset(c->adam_v, 0, sizeof(float) * P * D));
      GSF_CUDA_CHECK(cudaMemset(c->grad_accum, 0, sizeof(double) * P));
      GSF_CUDA_CHECK(cudaMemset(c->grad_count, 0, sizeof(int32_t) * P));
    }
    c->adam_step = 0.0;
    c->rng_seeded = false;   // a fresh MapState: its rng restarts from the mapper seed
    c->map_iteration = 0;
    ++c->map_gen;
    c->have_render = false;
  });
}

int gsf_map_download(gsf_ctx c, gsf_map_host* m) {
  return guard(c, [&] {
    if (!m || m->count != c->P) throw EInval("map_download: primitive count mismatch");
    const int64_t P = c->P;
    const int K = c->K, D = c->D;
    if (P == 0) return;
    double* tmp = nullptr;
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&tmp), sizeof(double) * P * D));
    k_gather_map_aos<<<div_up(P, 256), 256, 0, c->stream>>>(c->params, P, K, tmp);
    ++c->launches;
    double* h = static_cast<double*>(stage(c, sizeof(double) * P * D));
    GSF_CUDA_CHECK(cudaMemcpyAsync(h, tmp, sizeof(double) * P * D, cudaMemcpyDeviceToHost, c->stream));
    std::vector<double> nu(P);
    std::vector<uint8_t> ob(P);
    GSF_CUDA_CHECK(cudaMemcpyAsync(nu.data(), c->nu, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(ob.data(), c->observed, P, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    cudaFree(tmp);
    for (int64_t i = 0; i < P; ++i) {
      const double* o = h + i * D;
      if (m->mean) for (int a = 0; a < 3; ++a) m->mean[3 * i + a] = o[a];
      if (m->log_scale) for (int a = 0; a < 3; ++a) m->log_scale[3 * i + a] = o[3 + a];
      if (m->quat) for (int a = 0; a < 4; ++a) m->quat[4 * i + a] = o[6 + a];
      if (m->opacity_logit) m->opacity_logit[i] = o[10];
      if (m->sh && m->sh_coeffs == K) for (int b = 0; b < 3 * K; ++b) m->sh[3 * K * i + b] = o[11 + b];
      if (m->uncertainty) m->uncertainty[i] = nu[i];
      if (m->observed) m->observed[i] = ob[i];
    }
  });
}

int64_t gsf_map_count(gsf_ctx c) { return c ? c->P : -1; }
int32_t gsf_map_sh_coeffs(gsf_ctx c) { return c ? c->K : -1; }

int gsf_profile_enable(gsf_ctx c, int32_t on) {
  return guard(c, [&] {
    sync(c);
    c->prof.on = on != 0;
    c->ws.prof = on ? &c->prof : nullptr;
    for (int i = 0; i < 16; ++i) { c->prof.total_ms[i] = 0.0; c->prof.count[i] = 0; }
  });
}

int gsf_profile_read(gsf_ctx c, int32_t name, double* total_ms, int64_t* launches) {
  return guard(c, [&] {
    if (name < 0 || name >= PROF_NUM) throw EInval("profile_read: unknown kernel class");
    sync(c);
    *total_ms = c->prof.total_ms[name];
    *launches = c->prof.count[name];
  });
}

int gsf_event_record(gsf_ctx c, int32_t slot) {
  return guard(c, [&] {
    if (slot < 0 || slot >= 8) throw EInval("event slot out of range");
    if (!c->ev[slot]) GSF_CUDA_CHECK(cudaEventCreate(&c->ev[slot]));
    GSF_CUDA_CHECK(cudaEventRecord(c->ev[slot], c->stream));
  });
}

int gsf_event_elapsed(gsf_ctx c, int32_t a, int32_t b, double* ms) {
  return guard(c, [&] {
    if (a < 0 || a >= 8 || b < 0 || b >= 8 || !c->ev[a] || !c->ev[b]) throw EInval("event slot not recorded");
    GSF_CUDA_CHECK(cudaEventSynchronize(c->ev[b]));
    float f = 0.0f;
    GSF_CUDA_CHECK(cudaEventElapsedTime(&f, c->ev[a], c->ev[b]));
    *ms = f;
  });
}

int gsf_optimizer_reset(gsf_ctx c) {
  return guard(c, [&] {
    if (c->P > 0) {
      GSF_CUDA_CHECK(cudaMemsetAsync(c->adam_m, 0, sizeof(float) * c->P * c->D, c->stream));
      GSF_CUDA_CHECK(cudaMemsetAsync(c->adam_v, 0, sizeof(float) * c->P * c->D, c->stream));
      GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_accum, 0, sizeof(double) * c->P, c->stream));
      GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_count, 0, sizeof(int32_t) * c->P, c->stream));
    }
    c->adam_step = 0.0;
    c->rng_seeded = false;   // a fresh MapState: its rng restarts from the mapper seed
    c->map_iteration = 0;
    sync(c);
  });
}

int gsf_render(gsf_ctx c, const gsf_pose* pose, const gsf_intrinsics* K, const float* obs, const gsf_raster_cfg* cfg,
               gsf_render_out* out) {
  return guard(c, [&] {
    check_intrinsics(*K);
    check_raster(*cfg);
    const int W = K->width, H = K->height;
    const int64_t npix = static_cast<int64_t>(W) * H;
    ensure_ws(c, W, H);
    if (obs) upload_floats(c, c->ws.obs, obs, npix);
    render_sync(c, *pose, *K, *cfg, obs ? c->ws.obs : nullptr);
    Workspace& ws = c->ws;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst) GSF_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    };
    if (out) {
      d2h(out->color, ws.color, sizeof(float) * 3 * npix);
      d2h(out->alpha_depth, ws.alpha_depth, sizeof(float) * npix);
      d2h(out->median_depth, ws.median_depth, sizeof(float) * npix);
      d2h(out->median_valid, ws.median_valid, npix);
      d2h(out->opacity, ws.opacity, sizeof(float) * npix);
      d2h(out->uncertainty, ws.uncertainty, sizeof(float) * npix);
      d2h(out->final_transmittance, ws.final_T, sizeof(float) * npix);
      d2h(out->per_pixel_count, ws.count, sizeof(int32_t) * npix);
      d2h(out->dominant, ws.dominant, sizeof(int32_t) * npix);
      d2h(out->median_prim, ws.median_prim, sizeof(int32_t) * npix);
      d2h(out->dominant_weight, ws.dominant_w, sizeof(float) * npix);
      if (c->P > 0) d2h(out->visible, ws.visible, c->P);
      sync(c);
      out->has_uncertainty = obs ? 1 : 0;
      out->num_visible = c->ds_host->V;
      out->num_pairs = c->ds_host->M;
      if (!obs && out->uncertainty) std::memset(out->uncertainty, 0, sizeof(float) * npix);
    }
  });
}

int gsf_render_record(gsf_ctx c, uint32_t* row_start, int32_t* prim, float* alpha, float* trans, int64_t* total) {
  return guard(c, [&] {
    if (!c->have_render) throw EInval("render_record: no render on this context");
    const int W = c->rK.width, H = c->rK.height;
    const int64_t npix = static_cast<int64_t>(W) * H;
    std::vector<int32_t> cnt(npix);
    GSF_CUDA_CHECK(cudaMemcpy(cnt.data(), c->ws.count, sizeof(int32_t) * npix, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> rs(npix + 1);
    uint64_t acc = 0;
    for (int64_t i = 0; i < npix; ++i) {
      rs[i] = static_cast<uint32_t>(acc);
      acc += static_cast<uint64_t>(cnt[i]);
    }
    rs[npix] = static_cast<uint32_t>(acc);
    *total = static_cast<int64_t>(acc);
    if (row_start) std::memcpy(row_start, rs.data(), sizeof(uint32_t) * (npix + 1));
    if (!prim) return;
    uint32_t* d_rs = nullptr;
    int32_t* d_prim = nullptr;
    float *d_a = nullptr, *d_t = nullptr;
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d_rs), sizeof(uint32_t) * (npix + 1)));
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d_prim), sizeof(int32_t) * std::max<uint64_t>(acc, 1)));
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d_a), sizeof(float) * std::max<uint64_t>(acc, 1)));
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d_t), sizeof(float) * std::max<uint64_t>(acc, 1)));
    GSF_CUDA_CHECK(cudaMemcpy(d_rs, rs.data(), sizeof(uint32_t) * (npix + 1), cudaMemcpyHostToDevice));
    const RasterParams rp = make_rp(c, c->rK, c->rcfg);
    k_record<<<div_up(npix, 256), 256, 0, c->stream>>>(c->ws.ranges, c->ws.sid, c->ws.bg_id, c->ws.gg_id, c->ws.last, d_rs, W, H,
                                                        rp.tiles_x,
                                                        make_blend_consts(rp), d_prim, d_a, d_t);
    ++c->launches;
    sync(c);
    if (acc) {
      GSF_CUDA_CHECK(cudaMemcpy(prim, d_prim, sizeof(int32_t) * acc, cudaMemcpyDeviceToHost));
      if (alpha) GSF_CUDA_CHECK(cudaMemcpy(alpha, d_a, sizeof(float) * acc, cudaMemcpyDeviceToHost));
      if (trans) GSF_CUDA_CHECK(cudaMemcpy(trans, d_t, sizeof(float) * acc, cudaMemcpyDeviceToHost));
    }
    cudaFree(d_rs); cudaFree(d_prim); cudaFree(d_a); cudaFree(d_t);
  });
}

int gsf_render_tiles(gsf_ctx c, int32_t* tile_range, int64_t tiles_cap, int32_t* pair_prim, int64_t pair_cap) {
  return guard(c, [&] {
    if (!c->have_render) throw EInval("render_tiles: no render on this context");
    read_state(c);
    const uint32_t M = c->ds_host->M;
    const int tiles = ((c->rK.width + kTile - 1) / kTile) * ((c->rK.height + kTile - 1) / kTile);
    if (tile_range) {
      if (tiles_cap < tiles) throw EInval("render_tiles: tile capacity too small");
      GSF_CUDA_CHECK(cudaMemcpy(tile_range, c->ws.ranges, sizeof(int2) * tiles, cudaMemcpyDeviceToHost));
    }
    if (pair_prim && M) {
      if (pair_cap < M) throw EInval("render_tiles: pair capacity too small");
      GSF_CUDA_CHECK(cudaMemcpy(pair_prim, c->ws.sid, sizeof(int32_t) * M, cudaMemcpyDeviceToHost));
    }
  });
}

static void download_grads(gsf_ctx_s* c, gsf_grads_out* out) {
  const int64_t P = c->P;
  const int K = c->K, D = c->D;
  if (P > 0) {
    float* tmp = nullptr;
    GSF_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&tmp), sizeof(float) * P * (D + 2)));
    k_gather_grads_aos<<<div_up(P, 256), 256, 0, c->stream>>>(c->grads, P, K, c->d_mean2d, tmp);
    ++c->launches;
    std::vector<float> h(static_cast<size_t>(P) * (D + 2));
    GSF_CUDA_CHECK(cudaMemcpyAsync(h.data(), tmp, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    cudaFree(tmp);
    for (int64_t i = 0; i < P; ++i) {
      const float* o = &h[i * (D + 2)];
      if (out->d_mean) for (int a = 0; a < 3; ++a) out->d_mean[3 * i + a] = o[a];
      if (out->d_log_scale) for (int a = 0; a < 3; ++a) out->d_log_scale[3 * i + a] = o[3 + a];
      if (out->d_quat) for (int a = 0; a < 4; ++a) out->d_quat[4 * i + a] = o[6 + a];
      if (out->d_opacity_logit) out->d_opacity_logit[i] = o[10];
      if (out->d_sh) for (int b = 0; b < 3 * K; ++b) out->d_sh[3 * K * i + b] = o[11 + b];
      if (out->d_mean2d) { out->d_mean2d[2 * i] = o[D]; out->d_mean2d[2 * i + 1] = o[D + 1]; }
    }
  }
  read_state(c);
  for (int a = 0; a < 6; ++a) out->d_pose[a] = c->ds_host->d_pose[a];
}

int gsf_render_backward(gsf_ctx c, const gsf_upstream* up, const float* obs, gsf_grads_out* out) {
  return guard(c, [&] {
    if (!c->have_render) throw EInval("render_backward: no render on this context");
    if (c->render_gen != c->map_gen) throw EInval("render_backward: record does not match the primitive list");
    const int W = c->rK.width, H = c->rK.height;
    const int64_t npix = static_cast<int64_t>(W) * H;
    const bool use_c = up && up->d_color, use_ad = up && up->d_alpha_depth, use_md = up && up->d_median_depth,
               use_op = up && up->d_opacity, use_u = up && up->d_uncertainty && c->rcfg.uncertainty_full_gradient;
    if (use_u && !obs) throw EInval("render_backward: uncertainty gradient needs observed depth");
    if (c->P > 0) {
      GSF_CUDA_CHECK(cudaMemsetAsync(c->grads, 0, sizeof(float) * c->P * c->D, c->stream));
      GSF_CUDA_CHECK(cudaMemsetAsync(c->d_mean2d, 0, sizeof(float) * c->P * 2, c->stream));
    }
    GSF_CUDA_CHECK(cudaMemsetAsync(c->ds->d_pose, 0, sizeof(double) * 6, c->stream));
    if (!(use_c || use_ad || use_md || use_op || use_u)) {
      download_grads(c, out);
      return;
    }
    Workspace& ws = c->ws;
    float* u = ws.upstream;
    if (use_c) upload_floats(c, u, up->d_color, 3 * npix);
    if (use_ad) upload_floats(c, u + 3 * npix, up->d_alpha_depth, npix);
    if (use_md) upload_floats(c, u + 4 * npix, up->d_median_depth, npix);
    if (use_op) upload_floats(c, u + 5 * npix, up->d_opacity, npix);
    if (use_u) upload_floats(c, u + 6 * npix, up->d_uncertainty, npix);
    if (obs) upload_floats(c, ws.obs, obs, npix);
    BwdArgs b = bwd_args(c, c->rK, c->rcfg, obs ? ws.obs : nullptr, nullptr, make_lp(0, nullptr, c->rcfg), SEED_EXPLICIT, false);
    b.up_color = use_c ? u : nullptr;
    b.up_adepth = use_ad ? u + 3 * npix : nullptr;
    b.up_mdepth = use_md ? u + 4 * npix : nullptr;
    b.up_opacity = use_op ? u + 5 * npix : nullptr;
    b.up_uncert = use_u ? u + 6 * npix : nullptr;
    run_backward(ws, c->ds, b, c->stream, &c->launches);
    download_grads(c, out);
  });
}

static void fill_terms(gsf_ctx_s* c, gsf_loss_terms* out) {
  const DevState& h = *c->ds_host;
  *out = gsf_loss_terms{};
  out->color = h.term_color;
  out->ssim = h.term_ssim;
  out->geo = h.term_geo;
  out->align = h.term_align;
  out->iso = h.term_iso;
  out->var = h.term_var;
  out->total = h.loss_total;
  out->valid_color = static_cast<int32_t>(h.loss[LS_COLOR_CNT]);
  out->valid_geo = static_cast<int32_t>(h.loss[LS_GEO_CNT]);
  out->any_empty_mask = h.any_empty;
}

int gsf_tracking_loss(gsf_ctx c, const float* target, const float* depth, const gsf_loss_weights* w, gsf_loss_terms* out,
                      float* d_color, float* d_ad) {
  return guard(c, [&] {
    if (!c->have_render) throw EInval("tracking_loss: no render on this context");
    check_weights(*w);
    const gsf_intrinsics& k = c->rK;
    const int64_t npix = static_cast<int64_t>(k.width) * k.height;
    Workspace& ws = c->ws;
    float* tgt = ws.upstream;             // reuse: 3 planes rgb
    float* dep = ws.upstream + 3 * npix;  // 1 plane depth
    upload_floats(c, tgt, target, 3 * npix);
    upload_floats(c, dep, depth, npix);
    const LossParams lp = make_lp(1, w, c->rcfg);
    const int tiles = ((k.width + kTile - 1) / kTile) * ((k.height + kTile - 1) / kTile);
    c->ds_host->halt = 0;
    GSF_CUDA_CHECK(cudaMemsetAsync(&c->ds->halt, 0, sizeof(int32_t), c->stream));
    run_loss_tiles(ws, 1, tgt, dep, c->render_obs, k.width, k.height, k.near_plane, k.far_plane, lp.opacity_floor, c->stream, &c->launches);
    run_loss_finalize(ws, c->ds, lp, tiles, npix, -1, c->stream, &c->launches);
    float* seeds = ws.upstream + 4 * npix;   // 3 planes free (4..6) + use dssim scratch for the rest
    float* sout = ws.ssim_tmp;
    run_seeds_out(ws, c->ds, 1, tgt, dep, lp, k.width, k.height, k.near_plane, k.far_plane, sout, c->stream, &c->launches);
    (void)seeds;
    read_state(c);
    fill_terms(c, out);
    if (d_color) GSF_CUDA_CHECK(cudaMemcpy(d_color, sout, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost));
    if (d_ad) GSF_CUDA_CHECK(cudaMemcpy(d_ad, sout + 3 * npix, sizeof(float) * npix, cudaMemcpyDeviceToHost));
  });
}

static double sum_blocks(gsf_ctx_s* c, const double* dev, int n) {
  std::vector<double> h(n);
  GSF_CUDA_CHECK(cudaMemcpy(h.data(), dev, sizeof(double) * n, cudaMemcpyDeviceToHost));
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

int gsf_mapping_loss(gsf_ctx c, const float* target, const float* depth, const gsf_loss_weights* w, gsf_loss_terms* out,
                     float* d_color, float* d_ad, float* d_md, float* d_u, float* d_ls_direct) {
  return guard(c, [&] {
    if (!c->have_render) throw EInval("mapping_loss: no render on this context");
    if (c->render_gen != c->map_gen) throw EInval("mapping_loss: render does not match the primitive list");
    check_weights(*w);
    const gsf_intrinsics& k = c->rK;
    const int64_t npix = static_cast<int64_t>(k.width) * k.height;
    Workspace& ws = c->ws;
    // targets live in frame-sized scratch outside the SSIM buffers
    float* tgt = ws.upstream;
    float* dep = ws.upstream + 3 * npix;
    upload_floats(c, tgt, target, 3 * npix);
    upload_floats(c, dep, depth, npix);
    const LossParams lp = make_lp(2, w, c->rcfg);
    const int tiles = ((k.width + kTile - 1) / kTile) * ((k.height + kTile - 1) / kTile);
    GSF_CUDA_CHECK(cudaMemsetAsync(&c->ds->halt, 0, sizeof(int32_t), c->stream));
    const int32_t ho = c->render_obs ? 1 : 0;
    c->ds_host->has_obs = ho;
    GSF_CUDA_CHECK(cudaMemcpyAsync(&c->ds->has_obs, &c->ds_host->has_obs, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    run_loss_tiles(ws, 2, tgt, dep, c->render_obs, k.width, k.height, k.near_plane, k.far_plane, lp.opacity_floor, c->stream, &c->launches);
    if (w->w_ssim > 0.0) run_ssim(ws, c->ds, ws.color, tgt, k.width, k.height, 1.0f, ws.dssim, c->stream, &c->launches);
    run_iso(ws, c->ds, c->params, c->P, w->w_iso, w->iso_epsilon, nullptr, c->stream, &c->launches);
    run_loss_finalize(ws, c->ds, lp, tiles, npix, -1, c->stream, &c->launches);
    // 6 seed planes in the SSIM scratch (9 planes): its adjoint seeds u were consumed by k_ssim_bwd,
    // which precedes this on the stream; the seeds read the SSIM gradient from ws.dssim
    float* sout = ws.ssim_tmp;
    run_seeds_out(ws, c->ds, 2, tgt, dep, lp, k.width, k.height, k.near_plane, k.far_plane, sout, c->stream, &c->launches);
    if (d_ls_direct && c->P > 0) {
      GSF_CUDA_CHECK(cudaMemsetAsync(c->grads, 0, sizeof(float) * c->P * c->D, c->stream));
      if (w->w_iso > 0.0) run_iso(ws, c->ds, c->params, c->P, w->w_iso, w->iso_epsilon, c->grads, c->stream, &c->launches);
    }
    read_state(c);
    fill_terms(c, out);
    const bool have_c = w->w_color > 0.0 || w->w_ssim > 0.0;
    if (d_color) {
      if (have_c) GSF_CUDA_CHECK(cudaMemcpy(d_color, sout, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost));
      else std::memset(d_color, 0, sizeof(float) * 3 * npix);
    }
    if (d_ad) GSF_CUDA_CHECK(cudaMemcpy(d_ad, sout + 3 * npix, sizeof(float) * npix, cudaMemcpyDeviceToHost));
    if (d_md) GSF_CUDA_CHECK(cudaMemcpy(d_md, sout + 4 * npix, sizeof(float) * npix, cudaMemcpyDeviceToHost));
    if (d_u) GSF_CUDA_CHECK(cudaMemcpy(d_u, sout + 5 * npix, sizeof(float) * npix, cudaMemcpyDeviceToHost));
    if (d_ls_direct) {
      const int64_t P = c->P;
      std::vector<float> g(static_cast<size_t>(3) * P);
      if (P > 0 && w->w_iso > 0.0 && c->ds_host->V > 0)
        for (int a = 0; a < 3; ++a)
          GSF_CUDA_CHECK(cudaMemcpy(g.data() + a * P, c->grads + (3 + a) * P, sizeof(float) * P, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < P; ++i)
        for (int a = 0; a < 3; ++a) d_ls_direct[3 * i + a] = g[a * P + i];
    }
  });
}

int gsf_ssim(gsf_ctx c, const float* x, const float* y, int32_t w, int32_t h, double* value, float* d_x) {
  return guard(c, [&] {
    if (w <= 0 || h <= 0) throw EInval("ssim: empty image");
    const int64_t npix = static_cast<int64_t>(w) * h;
    ensure_ws(c, w, h);
    Workspace& ws = c->ws;
    upload_floats(c, ws.color, x, 3 * npix);
    upload_floats(c, ws.upstream, y, 3 * npix);
    run_ssim(ws, c->ds, ws.color, ws.upstream, w, h, 1.0f, d_x ? ws.dssim : nullptr, c->stream, &c->launches);
    sync(c);
    const double s = sum_blocks(c, ws.red_part, ws.ssim_blocks);
    *value = s / (3.0 * static_cast<double>(npix));
    if (d_x) GSF_CUDA_CHECK(cudaMemcpy(d_x, ws.dssim, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost));
  });
}

int gsf_frame_upload(gsf_ctx c, int32_t slot, const float* rgb, const float* depth, int32_t w, int32_t h) {
  return guard(c, [&] {
    if (slot < 0 || slot > 4096) throw EInval("frame slot out of range");
    if (w <= 0 || h <= 0) throw EInval("frame dimensions must be positive");
    if (static_cast<int>(c->frames.size()) <= slot) c->frames.resize(slot + 1);
    Frame& f = c->frames[slot];
    const int64_t npix = static_cast<int64_t>(w) * h;
    if (f.w * f.h != npix || !f.rgb) {
      dfree(f.rgb);
      dfree(f.depth);
      dalloc(f.rgb, 3 * npix);
      dalloc(f.depth, npix);
    }
    f.w = w;
    f.h = h;
    upload_floats(c, f.rgb, rgb, 3 * npix);
    upload_floats(c, f.depth, depth, npix);
  });
}

// ------------------------------------------------------------------------------------------------
// track_frame (tracker.cpp:30-84)
// ------------------------------------------------------------------------------------------------
// tracking trust region (rad, m): wide enough for a tracked frame's pose correction, small enough
// that the candidate list stays close to the visible set
constexpr double kTrustTheta = 0.03, kTrustDist = 0.05;

static void enqueue_track(gsf_ctx_s* c, const Frame& f, const gsf_intrinsics& k, const gsf_tracker_cfg& tcfg,
                          const gsf_loss_weights& w, const gsf_raster_cfg& rcfg) {
  const LossParams lp = make_lp(1, &w, rcfg);
  const int tiles = ((k.width + kTile - 1) / kTile) * ((k.height + kTile - 1) / kTile);
  const int64_t npix = static_cast<int64_t>(k.width) * k.height;
  // per iteration: forward (its last CTA finalises the loss), pose backward (its last CTA sums
  // the pose gradient) and the single-thread pose step
  // the map is constant during track_frame: validate it and cache its view-independent part once
  run_world(c->ws, c->ds, c->params, c->P, make_rp(c, k, rcfg), c->stream, &c->launches);
  // primitives that can be visible while the camera stays within kTrustTheta / kTrustDist of the
  // starting pose; the iterations preprocess only those until a step leaves the region
  run_candidates(c->ws, c->ds, c->params, c->P, make_rp(c, k, rcfg), kTrustTheta, kTrustDist, c->stream, &c->launches);
  Workspace& ws = c->ws;
  const int64_t obuf = 1 + 5 * ws.tiles_cap;   // one Workspace::order half
  for (int it = 0; it < tcfg.iterations; ++it) {
    FwdArgs fa = fwd_args(c, k, rcfg, nullptr, f.rgb, f.depth, lp, it);
    fa.cand = c->ws.cand;
    // longest-first CTA order from the previous iteration's counts (any order gives the same bits)
    fa.order = ws.order + (it & 1) * obuf;
    fa.join_order = it > 0;
    fa.want_posejac = true;
    // the two-pixel pose backward (K == 1) reads T, last and the seed signs only; the view-dependent
    // pose backward (k_backward_pose<SEED_TRACK, true>) derives its seeds from the maps
    fa.keep_maps = c->K > 1;
    fa.qmode = c->K == 1 ? 1 : 0;
    fa.clean_bins = true;   // ... and each blend leaves the bins zeroed for the next iteration
    fa.bins_clean = it > 0;
    fa.fuse_loss_final = true;
    fa.use_world = true;
    fa.want_pair_base = false;
    run_forward(c->ws, c->ds, fa, c->stream, &c->launches);
    BwdArgs b = bwd_args(c, k, rcfg, f.depth, f.rgb, lp, SEED_TRACK, true);
    b.fused_pose = true;
    b.update_iter = it;
    b.order = fa.order;
    if (!run_backward(c->ws, c->ds, b, c->stream, &c->launches)) run_track_update(c->ds, it, c->stream, &c->launches);
    // the next iteration's orders on the second side branch, beside the next preprocess and binning
    GSF_CUDA_CHECK(cudaEventRecord(ws.ev_lfork, c->stream));
    GSF_CUDA_CHECK(cudaStreamWaitEvent(ws.side2, ws.ev_lfork, 0));
    run_lpt(ws, tiles, ws.order + ((it + 1) & 1) * obuf, ws.side2, &c->launches);
    GSF_CUDA_CHECK(cudaEventRecord(ws.ev_ljoin, ws.side2));
  }
  // final render + loss without gradients (tracker.cpp:74-76)
  FwdArgs fin = fwd_args(c, k, rcfg, nullptr, f.rgb, f.depth, lp, -1);
  fin.fuse_loss_final = true;
  fin.use_world = true;
  fin.want_pair_base = false;
  fin.order = ws.order + (tcfg.iterations & 1) * obuf;
  fin.join_order = tcfg.iterations > 0;   // also rejoins the k_lpt branch before the capture ends
  run_forward(c->ws, c->ds, fin, c->stream, &c->launches);
  (void)tiles;
  (void)npix;
}

// The ~10 launches per iteration of a track_frame replayed as one CUDA graph: the loop is
// captured once per (frame buffers, camera, configuration, map, allocation generation) and
// replayed while those match; profiling (per-kernel events) and the first attempt after a
// capacity growth run eagerly.
static void run_track(gsf_ctx_s* c, const Frame& f, const gsf_intrinsics& k, const gsf_tracker_cfg& tcfg,
                      const gsf_loss_weights& w, const gsf_raster_cfg& rcfg) {
  if (!c->use_graphs || (c->ws.prof && c->ws.prof->on)) {
    enqueue_track(c, f, k, tcfg, w, rcfg);
    return;
  }
  // the captured loop reads the frame from a context-owned buffer, so a new frame (or another slot)
  // costs one device-to-device copy instead of a re-capture
  const int64_t npix = static_cast<int64_t>(f.w) * f.h;
  Frame& tin = c->track_in;
  if (tin.w * tin.h != npix || !tin.rgb) {
    dalloc(tin.rgb, 3 * npix);
    dalloc(tin.depth, npix);
  }
  tin.w = f.w;
  tin.h = f.h;
  GSF_CUDA_CHECK(cudaMemcpyAsync(tin.rgb, f.rgb, sizeof(float) * 3 * npix, cudaMemcpyDeviceToDevice, c->stream));
  GSF_CUDA_CHECK(cudaMemcpyAsync(tin.depth, f.depth, sizeof(float) * npix, cudaMemcpyDeviceToDevice, c->stream));
  const Frame& fr = tin;
  TrackGraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.rgb = fr.rgb;
  key.depth = fr.depth;
  key.params = c->params;
  key.K = k;
  key.rcfg = rcfg;
  key.w = w;
  key.iterations = tcfg.iterations;
  key.P = c->P;
  key.sh = c->K;
  key.alloc_gen = g_alloc_gen;
  for (TrackGraph& g : c->track_graphs)
    if (g.valid && std::memcmp(&g.key, &key, sizeof(key)) == 0) {
      GSF_CUDA_CHECK(cudaGraphLaunch(g.exec, c->stream));
      c->launches += g.launches;
      return;
    }
  TrackGraph& g = c->track_graphs[c->track_graph_next];
  c->track_graph_next = (c->track_graph_next + 1) % 8;
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g.exec = nullptr;
  g.valid = false;
  const int64_t l0 = c->launches;
  GSF_CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_track(c, fr, k, tcfg, w, rcfg);
  } catch (...) {
    cudaGraph_t dummy = nullptr;
    cudaStreamEndCapture(c->stream, &dummy);
    if (dummy) cudaGraphDestroy(dummy);
    throw;
  }
  cudaGraph_t graph = nullptr;
  GSF_CUDA_CHECK(cudaStreamEndCapture(c->stream, &graph));
  const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  GSF_CUDA_CHECK(ie);
  g.key = key;
  g.launches = c->launches - l0;
  g.valid = true;
  GSF_CUDA_CHECK(cudaGraphLaunch(g.exec, c->stream));
}

int gsf_track_frame(gsf_ctx c, int32_t slot, const gsf_pose* initial, const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg,
                    const gsf_loss_weights* w, const gsf_raster_cfg* rcfg, gsf_track_result* out) {
  return guard(c, [&] {
    check_intrinsics(*K);
    check_raster(*rcfg);
    check_weights(*w);
    const Frame& f = get_frame(c, slot, *K);
    ensure_ws(c, K->width, K->height);
    const Cam cam = host_cam(*initial, *K);
    for (int attempt = 0; attempt < 3; ++attempt) {
      reset_state(c, &cam);
      DevState& h = *c->ds_host;
      for (int a = 0; a < 3; ++a) { h.pose_rot[a] = initial->rotation_tangent[a]; h.pose_trans[a] = initial->translation[a]; }
      h.lr_rot = tcfg->lr_rotation;
      h.lr_trans = tcfg->lr_translation;
      h.degraded_ratio = tcfg->degraded_loss_ratio;
      GSF_CUDA_CHECK(cudaMemcpyAsync(c->ds, &h, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
      run_track(c, f, *K, *tcfg, *w, *rcfg);
      read_state(c);
      if (!h.overflow) break;
      grow_pairs(c, h.M_max);
    }
    check_overflow(c, "track_frame");
    const DevState& h = *c->ds_host;
    if (h.bad_index != std::numeric_limits<int32_t>::max()) throw_nonfinite(h.bad_index);
    *out = gsf_track_result{};
    out->initial_loss = h.initial_loss;
    if (h.halt == 1) {   // nothing to track at iteration 0: keep the prediction (tracker.cpp:46-53)
      out->pose = *initial;
      out->degraded = 1;
      out->final_loss = h.final_loss;
      out->iterations_run = 0;
      return;
    }
    if (h.halt == 2) {
      std::ostringstream m;
      m << "tracking diverged at iteration " << h.halt_iter << ": total=" << h.loss_total << " color=" << h.term_color
        << " geo=" << h.term_geo;
      throw EDiverged(m.str());
    }
    for (int a = 0; a < 3; ++a) {
      out->pose.rotation_tangent[a] = h.pose_rot[a];
      out->pose.translation[a] = h.pose_trans[a];
    }
    out->final_loss = h.loss_total;
    out->iterations_run = tcfg->iterations;
    if (tcfg->iterations == 0)
      out->degraded = (h.loss[LS_COLOR_CNT] == 0.0 && h.loss[LS_GEO_CNT] == 0.0) ? 1 : 0;
    else if (h.loss_total > tcfg->degraded_loss_ratio * h.initial_loss)
      out->degraded = 1;
  });
}

int gsf_tracking_gradient(gsf_ctx c, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K,
                          const gsf_loss_weights* w, const gsf_raster_cfg* rcfg, gsf_loss_terms* terms,
                          double d_pose[6]) {
  return guard(c, [&] {
    check_intrinsics(*K);
    check_raster(*rcfg);
    check_weights(*w);
    const Frame& f = get_frame(c, slot, *K);
    ensure_ws(c, K->width, K->height);
    const Cam cam = host_cam(*pose, *K);
    const LossParams lp = make_lp(1, w, *rcfg);
    const int tiles = ((K->width + kTile - 1) / kTile) * ((K->height + kTile - 1) / kTile);
    const int64_t npix = static_cast<int64_t>(K->width) * K->height;
    for (int attempt = 0; attempt < 3; ++attempt) {
      reset_state(c, &cam);
      FwdArgs fa = fwd_args(c, *K, *rcfg, nullptr, f.rgb, f.depth, lp, -1);
      fa.want_posejac = true;
      fa.qmode = c->K == 1 ? 2 : 0;
      run_forward(c->ws, c->ds, fa, c->stream, &c->launches);
      run_loss_finalize(c->ws, c->ds, lp, tiles, npix, -1, c->stream, &c->launches);
      BwdArgs b = bwd_args(c, *K, *rcfg, f.depth, f.rgb, lp, SEED_TRACK, true);
      b.fused_pose = true;
      run_backward(c->ws, c->ds, b, c->stream, &c->launches);
      read_state(c);
      if (!c->ds_host->overflow) break;
      grow_pairs(c, c->ds_host->M_max);
    }
    check_overflow(c, "tracking_gradient");
    if (c->ds_host->bad_index != std::numeric_limits<int32_t>::max()) throw_nonfinite(c->ds_host->bad_index);
    fill_terms(c, terms);
    for (int a = 0; a < 6; ++a) d_pose[a] = c->ds_host->d_pose[a];
    c->have_render = true;
    c->render_gen = c->map_gen;
    c->rK = *K;
    c->rcfg = *rcfg;
    c->render_obs = false;
  });
}

int gsf_track_frame_host(gsf_ctx c, const float* rgb, const float* depth, const gsf_pose* initial, const gsf_intrinsics* K,
                         const gsf_tracker_cfg* tcfg, const gsf_loss_weights* w, const gsf_raster_cfg* rcfg,
                         gsf_track_result* out) {
  const int rc = gsf_frame_upload(c, 0, rgb, depth, K->width, K->height);
  if (rc != GSF_OK) return rc;
  return gsf_track_frame(c, 0, initial, K, tcfg, w, rcfg, out);
}

// ------------------------------------------------------------------------------------------------
// map_step (mapper.cpp:232-281) and sliding_ba (tracker.cpp:119-183)
// ------------------------------------------------------------------------------------------------
static AdamGroups groups_of(const gsf_mapper_cfg& m) {
  AdamGroups g;
  g.lr[0] = m.lr_mean * m.scene_extent;
  g.lr[1] = m.lr_scale;
  g.lr[2] = m.lr_rotation;
  g.lr[3] = m.lr_opacity;
  g.lr[4] = m.lr_sh;
  return g;
}

// One mapping-objective forward/backward of keyframe k into c->grads (accumulating).
// cam_staged: the previous view's k_pose_sum already made keyframe k's camera current; next_k >= 0:
// this view's k_pose_sum stages keyframe next_k's camera for the following view.
static void enqueue_map_view(gsf_ctx_s* c, const Frame& f, int k, const gsf_intrinsics& K, const gsf_mapper_cfg& m, int it,
                             double* loss_acc, int trace_index, bool use_world = false, bool cam_staged = false,
                             int next_k = -1) {
  const LossParams lp = make_lp(2, &m.weights, m.raster);
  const int tiles = ((K.width + kTile - 1) / kTile) * ((K.height + kTile - 1) / kTile);
  const int64_t npix = static_cast<int64_t>(K.width) * K.height;
  if (!cam_staged) {
    launch_pdl(k_set_cam_from_kf, dim3(1), dim3(1), 0, c->stream, c->ds, c->kf, k, 1);
    ++c->launches;
  }
  FwdArgs fa = fwd_args(c, K, m.raster, f.depth, f.rgb, f.depth, lp, it);
  fa.use_world = use_world;
  run_forward(c->ws, c->ds, fa, c->stream, &c->launches);
#ifndef GSF_NO_MAP_LPT
  // longest-first order of the backward's (tile, quadrant) CTAs from the forward's per-quadrant steps,
  // on a side branch beside the SSIM / iso / loss tail, joined before the backward
  Workspace& wsl = c->ws;
  GSF_CUDA_CHECK(cudaEventRecord(wsl.ev_lfork, c->stream));
  GSF_CUDA_CHECK(cudaStreamWaitEvent(wsl.side2, wsl.ev_lfork, 0));
  run_lpt(wsl, tiles, wsl.order, wsl.side2, &c->launches);
  GSF_CUDA_CHECK(cudaEventRecord(wsl.ev_ljoin, wsl.side2));
#endif
  if (m.weights.w_ssim > 0.0) run_ssim(c->ws, c->ds, c->ws.color, f.rgb, K.width, K.height, 1.0f, c->ws.dssim, c->stream, &c->launches);
  run_iso(c->ws, c->ds, c->params, c->P, m.weights.w_iso, m.weights.iso_epsilon, nullptr, c->stream, &c->launches);
  run_loss_finalize(c->ws, c->ds, lp, tiles, npix, it, c->stream, &c->launches);
  BwdArgs b = bwd_args(c, K, m.raster, f.depth, f.rgb, lp, SEED_MAP, false);
#ifndef GSF_NO_MAP_LPT
  GSF_CUDA_CHECK(cudaStreamWaitEvent(c->stream, wsl.ev_ljoin, 0));
  b.order = wsl.order;
#endif
  b.iso_w = m.weights.w_iso;   // the iso gradient is added by k_chain (no second iso pass)
  b.iso_eps = m.weights.iso_epsilon;
  // k_kf_grab and the next view's k_set_cam_from_kf run in the chain's k_pose_sum
  b.post.kf = c->kf;
  b.post.grab = k;
  b.post.loss_acc = loss_acc;
  b.post.trace = c->trace_dev;
  b.post.trace_index = trace_index;
  b.post.next = next_k;
  run_backward(c->ws, c->ds, b, c->stream, &c->launches);
}

static void upload_kf(gsf_ctx_s* c, const gsf_pose* poses, int n) {
  ensure_kf(c, n);
  for (int i = 0; i < n; ++i) {
    KfPose& p = c->kf_host[i];
    std::memset(&p, 0, sizeof(KfPose));
    for (int a = 0; a < 3; ++a) { p.rot[a] = poses[i].rotation_tangent[a]; p.trans[a] = poses[i].translation[a]; }
  }
  GSF_CUDA_CHECK(cudaMemcpyAsync(c->kf, c->kf_host, sizeof(KfPose) * n, cudaMemcpyHostToDevice, c->stream));
}

static void check_mapper(const gsf_mapper_cfg& m);
static gsf_structural_change densify_and_cull(gsf_ctx_s* c, const gsf_mapper_cfg& m);

int gsf_map_step(gsf_ctx c, const int32_t* slots, const gsf_pose* poses, int32_t n, const gsf_intrinsics* K,
                 const gsf_mapper_cfg* m, int32_t iterations, double* trace) {
  return guard(c, [&] {
    if (n <= 0) throw EInval("mapping window is empty");
    check_intrinsics(*K);
    check_raster(m->raster);
    check_weights(m->weights);
    std::vector<const Frame*> fr(n);
    for (int i = 0; i < n; ++i) {
      if (slots[i] < 0 || slots[i] >= static_cast<int>(c->frames.size()) || !c->frames[slots[i]].rgb)
        throw EInval("mapping window observation missing rgb or depth");
      fr[i] = &get_frame(c, slots[i], *K);
    }
    if (iterations <= 0) return;
    check_mapper(*m);
    ensure_ws(c, K->width, K->height);
    ensure_trace(c, iterations);
    const Cam cam = host_cam(poses[0], *K);
    reset_state(c, &cam);
    upload_kf(c, poses, n);
    const AdamGroups g = groups_of(*m);
    for (int it = 0; it < iterations; ++it) {
      const int o = it % n;
      if (c->P > 0) {
        GSF_CUDA_CHECK(cudaMemsetAsync(c->grads, 0, sizeof(float) * c->P * c->D, c->stream));
        GSF_CUDA_CHECK(cudaMemsetAsync(c->d_mean2d, 0, sizeof(float) * c->P * 2, c->stream));
      }
      enqueue_map_view(c, *fr[o], o, *K, *m, static_cast<int>(c->map_iteration) + it, nullptr, it);
      run_densify_stats(c->ws.visible, c->d_mean2d, c->grad_accum, c->grad_count, c->P, K->width, K->height, c->stream, &c->launches);
      c->adam_step += 1.0;
      run_adam(c->params, c->grads, c->adam_m, c->adam_v, c->P, c->D, g, c->adam_step, c->stream, &c->launches);
      // densify_and_cull every `interval` mapping iterations (mapper.cpp:278-279)
      const int64_t done = c->map_iteration + it + 1;
      if (m->densify_interval > 0 && done % m->densify_interval == 0) {
        read_state(c);
        if (c->ds_host->halt || c->ds_host->overflow ||
            c->ds_host->bad_index != std::numeric_limits<int32_t>::max())
          break;   // reported below
        densify_and_cull(c, *m);
        ensure_ws(c, K->width, K->height);
      }
    }
    read_state(c);
    const DevState& h = *c->ds_host;
    if (h.bad_index != std::numeric_limits<int32_t>::max()) throw_nonfinite(h.bad_index);
    if (h.overflow) throw EUnsupported("map_step: pair capacity exceeded; rerun after a render at these poses");
    if (h.halt == 2) {
      std::ostringstream msg;
      msg << "mapping diverged at iteration " << h.halt_iter << ": total=" << h.loss_total << " color=" << h.term_color
          << " ssim=" << h.term_ssim << " geo=" << h.term_geo << " align=" << h.term_align << " iso=" << h.term_iso
          << " var=" << h.term_var;
      throw EDiverged(msg.str());
    }
    if (trace) GSF_CUDA_CHECK(cudaMemcpy(trace, c->trace_dev, sizeof(double) * iterations, cudaMemcpyDeviceToHost));
    c->map_iteration += iterations;
  });
}

int gsf_ba_partition(int32_t n, int32_t nranks, int32_t rank, uint8_t* owned) {
  if (n < 0 || nranks <= 0 || rank < 0 || rank >= nranks || (!owned && n > 0)) return GSF_EINVAL;
  for (int k = 0; k < n; ++k) owned[k] = (k % nranks == rank) ? 1 : 0;
  return GSF_OK;
}

int gsf_comm_unique_id(uint8_t id[128]) {
  if (!g_nccl.load()) return GSF_ECUDA;
  return g_nccl.get_unique_id(id) == 0 ? GSF_OK : GSF_ECUDA;
}

int gsf_comm_init(gsf_ctx c, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  return guard(c, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw EInval("comm_init: bad rank/size");
    c->nranks = nranks;
    c->rank = rank;
    c->host_ar = nullptr;
    if (nranks == 1) return;
    if (!g_nccl.load()) throw EUnsupported("NCCL (libnccl.so.2) could not be loaded");
    auto init = reinterpret_cast<nccl_init_fn>(dlsym(g_nccl.h, "ncclCommInitRank"));
    if (!init) throw EUnsupported("ncclCommInitRank missing");
    NcclUid uid;
    std::memcpy(uid.b, id, 128);
    const int r = init(&c->comm, nranks, uid, rank);
    if (r != 0) throw EUnsupported(std::string("ncclCommInitRank failed: ") + (g_nccl.get_error ? g_nccl.get_error(r) : "?"));
    if (!c->comm_stream) GSF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    if (!c->ev_grads) GSF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_grads, cudaEventDisableTiming));
    for (cudaEvent_t& e : c->ev_bucket)
      if (!e) GSF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  });
}

int gsf_comm_init_host(gsf_ctx c, int32_t nranks, int32_t rank, gsf_host_allreduce_fn fn, void* user) {
  return guard(c, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw EInval("comm_init: bad rank/size");
    if (nranks > 1 && !fn) throw EInval("comm_init_host: null all-reduce callback");
    if (c->comm && g_nccl.comm_destroy) g_nccl.comm_destroy(c->comm);
    c->comm = nullptr;
    c->nranks = nranks;
    c->rank = rank;
    c->host_ar = fn;
    c->host_ar_user = user;
  });
}

static double* kf_grad(gsf_ctx_s* c, int k) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(c->kf + k) + offsetof(KfPose, grad));
}

static size_t dtype_bytes(int dtype) { return dtype == GSF_DT_F64 ? 8 : 4; }

// Sum-all-reduce of a device buffer over the context's communicator, ordered on `st` (NCCL), or
// staged through pinned host memory to the caller's callback (host communicator; synchronous).
static void allreduce(gsf_ctx_s* c, void* buf, size_t count, int dtype, cudaStream_t st) {
  if (c->nranks <= 1 || count == 0) return;
  if (c->host_ar) {
    const size_t bytes = count * dtype_bytes(dtype);
    if (c->host_stage_bytes < bytes) {
      if (c->host_stage) cudaFreeHost(c->host_stage);
      c->host_stage = nullptr;
      GSF_CUDA_CHECK(cudaMallocHost(&c->host_stage, bytes));
      c->host_stage_bytes = bytes;
    }
    GSF_CUDA_CHECK(cudaMemcpyAsync(c->host_stage, buf, bytes, cudaMemcpyDeviceToHost, st));
    GSF_CUDA_CHECK(cudaStreamSynchronize(st));
    if (c->host_ar(c->host_stage, count, dtype, c->host_ar_user) != 0) throw ERuntime("host all-reduce callback failed");
    GSF_CUDA_CHECK(cudaMemcpyAsync(buf, c->host_stage, bytes, cudaMemcpyHostToDevice, st));
    GSF_CUDA_CHECK(cudaStreamSynchronize(st));
    return;
  }
  const int r = g_nccl.all_reduce(buf, buf, count, dtype, 0 /*sum*/, c->comm, st);
  if (r != 0) throw EUnsupported(std::string("ncclAllReduce failed: ") + (g_nccl.get_error ? g_nccl.get_error(r) : "?"));
}

// One exchange per sharded sliding_ba iteration: the packed fp64 scalars (loss,
// divergence flag, window pose gradients) and the fp32 Gaussian gradients, bucketed by parameter
// group (mean, log_scale, quat, opacity, SH: contiguous [field][P] slices).  Over NCCL the buckets
// run on the communicator stream and each group's Adam waits only for its own bucket, so the
// optimizer step of one group overlaps the reduction of the next; over a host communicator the
// same sequence runs synchronously.
static void exchange_and_step(gsf_ctx_s* c, int n, double* loss_acc, const AdamGroups& g, int it) {
  if (c->ba_pack_cap < 2 + 6 * n) {
    dalloc(c->ba_pack, 2 + 6 * n);
    c->ba_pack_cap = 2 + 6 * n;
  }
  k_ba_pack<<<1, 128, 0, c->stream>>>(c->ds, c->kf, n, loss_acc, c->ba_pack);
  ++c->launches;
  static const int kGroupFields[6] = {0, 3, 6, 10, 11, -1};
  const bool nccl = c->host_ar == nullptr;
  cudaStream_t cs = nccl ? c->comm_stream : c->stream;
  if (nccl) {
    GSF_CUDA_CHECK(cudaEventRecord(c->ev_grads, c->stream));
    GSF_CUDA_CHECK(cudaStreamWaitEvent(cs, c->ev_grads, 0));
  }
  allreduce(c, c->ba_pack, static_cast<size_t>(2 + 6 * n), GSF_DT_F64, cs);
  for (int b = 0; b < 5; ++b) {
    const int f0 = kGroupFields[b], f1 = b == 4 ? c->D : kGroupFields[b + 1];
    allreduce(c, c->grads + static_cast<int64_t>(f0) * c->P, static_cast<size_t>(f1 - f0) * c->P, GSF_DT_F32, cs);
    if (nccl) GSF_CUDA_CHECK(cudaEventRecord(c->ev_bucket[b], cs));
  }
  for (int b = 0; b < 5; ++b) {
    if (nccl) GSF_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_bucket[b], 0));
    if (b == 0) {
      k_ba_unpack<<<1, 128, 0, c->stream>>>(c->ds, c->kf, n, loss_acc, c->ba_pack, it);
      ++c->launches;
    }
    const int f0 = kGroupFields[b], f1 = b == 4 ? c->D : kGroupFields[b + 1];
    run_adam_fields(c->params, c->grads, c->adam_m, c->adam_v, c->P, f0, f1, g, c->adam_step, c->stream, &c->launches);
  }
}

int gsf_sliding_ba(gsf_ctx c, const int32_t* slots, gsf_pose* poses, const int32_t* frame_ids, int32_t n,
                   const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg, const gsf_mapper_cfg* m, int32_t iterations,
                   double* trace) {
  return guard(c, [&] {
    if (n <= 0) throw EInval("adjustment window is empty");
    check_intrinsics(*K);
    check_raster(m->raster);
    check_weights(m->weights);
    std::vector<const Frame*> fr(n, nullptr);
    std::vector<uint8_t> owned(n);
    gsf_ba_partition(n, c->nranks, c->rank, owned.data());
    for (int i = 0; i < n; ++i) {
      if (!owned[i]) continue;
      if (slots[i] < 0 || slots[i] >= static_cast<int>(c->frames.size()) || !c->frames[slots[i]].rgb)
        throw EInval("adjustment window holds a null keyframe");
      fr[i] = &get_frame(c, slots[i], *K);
    }
    int anchor = -1;
    if (tcfg->freeze_oldest_pose) {
      anchor = 0;
      for (int i = 1; i < n; ++i)
        if (frame_ids[i] < frame_ids[anchor]) anchor = i;
    }
    ensure_ws(c, K->width, K->height);
    ensure_trace(c, std::max(iterations, 1) + 2);
    const Cam cam = host_cam(poses[0], *K);
    reset_state(c, &cam);
    upload_kf(c, poses, n);
    const AdamGroups g = groups_of(*m);
    double* loss_acc = c->trace_dev + std::max(iterations, 1);  // scratch slot after the trace
    for (int it = 0; it < iterations; ++it) {
      if (c->P > 0) {
        GSF_CUDA_CHECK(cudaMemsetAsync(c->grads, 0, sizeof(float) * c->P * c->D, c->stream));
        GSF_CUDA_CHECK(cudaMemsetAsync(c->d_mean2d, 0, sizeof(float) * c->P * 2, c->stream));
      }
      GSF_CUDA_CHECK(cudaMemsetAsync(loss_acc, 0, sizeof(double), c->stream));
      // the map is constant across this iteration's keyframes: validate + cache it once
      run_world(c->ws, c->ds, c->params, c->P, make_rp(c, *K, m->raster), c->stream, &c->launches);
      bool staged = false;
      for (int k = 0; k < n; ++k) {
        if (!owned[k]) {
          GSF_CUDA_CHECK(cudaMemsetAsync(kf_grad(c, k), 0, sizeof(double) * 6, c->stream));
          continue;
        }
        int next = -1;   // the next owned view of this iteration (the poses change after its last view)
        for (int j = k + 1; j < n && next < 0; ++j)
          if (owned[j]) next = j;
        enqueue_map_view(c, *fr[k], k, *K, *m, it, loss_acc, -1, true, staged, next);
        staged = next >= 0;
      }
      c->adam_step += 1.0;
      if (c->nranks > 1) {
        exchange_and_step(c, n, loss_acc, g, it);
      } else {
        if (c->ws.prof) c->ws.prof->begin(PROF_ADAM, c->stream);
        run_adam(c->params, c->grads, c->adam_m, c->adam_v, c->P, c->D, g, c->adam_step, c->stream, &c->launches);
        if (c->ws.prof) c->ws.prof->end(c->stream);
      }
      k_store<<<1, 1, 0, c->stream>>>(loss_acc, c->trace_dev + it);
      ++c->launches;
      k_kf_update<<<1, 32 * div_up(n, 32), 0, c->stream>>>(c->ds, c->kf, n, anchor, tcfg->lr_rotation, tcfg->lr_translation);
      ++c->launches;
    }
    read_state(c);
    const DevState& h = *c->ds_host;
    if (h.bad_index != std::numeric_limits<int32_t>::max()) throw_nonfinite(h.bad_index);
    if (h.overflow) throw EUnsupported("sliding_ba: pair capacity exceeded; rerun after a render at these poses");
    if (h.halt == 2) {
      std::ostringstream msg;
      msg << "bundle adjustment diverged at iteration " << h.halt_iter << ": total=" << h.loss_total;
      throw EDiverged(msg.str());
    }
    GSF_CUDA_CHECK(cudaMemcpy(c->kf_host, c->kf, sizeof(KfPose) * n, cudaMemcpyDeviceToHost));
    for (int k = 0; k < n; ++k)
      for (int a = 0; a < 3; ++a) {
        poses[k].rotation_tangent[a] = c->kf_host[k].rot[a];
        poses[k].translation[a] = c->kf_host[k].trans[a];
      }
    if (trace && iterations > 0) GSF_CUDA_CHECK(cudaMemcpy(trace, c->trace_dev, sizeof(double) * iterations, cudaMemcpyDeviceToHost));
  });
}

// MapperConfig::validate (mapper.cpp:28-45) for the fields the device path reads.
static void check_mapper(const gsf_mapper_cfg& m) {
  if (m.sh_coeffs != 1 && m.sh_coeffs != 4 && m.sh_coeffs != 9 && m.sh_coeffs != 16)
    throw EInval("sh coefficient count must be 1, 4, 9 or 16");
  if (m.init_stride < 1 || m.spawn_stride < 1) throw EInval("sampling strides must be at least 1");
  if (!(m.spawn_opacity_threshold > 0.0 && m.spawn_opacity_threshold <= 1.0))
    throw EInval("spawn opacity threshold must lie in (0, 1]");
  if (!(m.init_opacity > 0.0 && m.init_opacity < 1.0)) throw EInval("initial opacity must lie in (0, 1)");
  if (!(m.scene_extent > 0.0)) throw EInval("scene extent must be positive");
  if (!(m.densify_split_factor > 1.0)) throw EInval("split factor must exceed 1");
}

// Candidate pass of initialize / spawn: count the accepted stride-sampled pixels (blocking).
static uint32_t backproject_count(gsf_ctx_s* c, BackprojectArgs& a, const Frame& f, const gsf_pose& pose,
                                  const gsf_intrinsics& K, const gsf_mapper_cfg& m, int stride, const float* opacity) {
  a.depth = f.depth;
  a.rgb = f.rgb;
  a.opacity = opacity;
  a.threshold = m.spawn_opacity_threshold;
  a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
  a.near_plane = K.near_plane;
  a.far_plane = K.far_plane;
  // pose.inverse() (pose.hpp:35-38): rotation exp(-rot), translation -(R^T t)
  double R[9], nrot[3];
  exp_map_d(pose.rotation_tangent, R);
  for (int i = 0; i < 3; ++i) nrot[i] = -pose.rotation_tangent[i];
  exp_map_d(nrot, a.Rinv);
  for (int i = 0; i < 3; ++i)
    a.tinv[i] = -(R[0 * 3 + i] * pose.translation[0] + R[1 * 3 + i] * pose.translation[1] + R[2 * 3 + i] * pose.translation[2]);
  a.logit0 = std::log(m.init_opacity / (1.0 - m.init_opacity));
  a.W = K.width;
  a.H = K.height;
  a.stride = stride;
  a.K = m.sh_coeffs;
  a.cells_x = (K.width + stride - 1) / stride;
  a.cells = static_cast<int64_t>(a.cells_x) * ((K.height + stride - 1) / stride);
  const int64_t blocks = std::max<int64_t>(1, div_up(a.cells, 256));
  if (2 * blocks + 1 > c->bp_cap) {
    dalloc(c->bp_scratch, 2 * blocks + 1);
    c->bp_cap = 2 * blocks + 1;
  }
  run_backproject_count(a, c->bp_scratch, c->bp_scratch + blocks, c->bp_scratch + 2 * blocks, c->stream, &c->launches);
  uint32_t total = 0;
  GSF_CUDA_CHECK(cudaMemcpyAsync(&total, c->bp_scratch + 2 * blocks, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return total;
}

// Re-lay the SoA map [field][P] out for P_new >= P primitives: parameters, Adam moments, nu,
// observed and the densify statistics are kept; the new tail of the moments and statistics is
// zero (AdamState::append, MapState resize).
static void grow_map_soa(gsf_ctx_s* c, int64_t P_new) {
  const int64_t P_old = c->P;
  const int D = c->D;
  float *params = nullptr, *m = nullptr, *v = nullptr;
  double *nu = nullptr, *acc = nullptr;
  uint8_t* obs = nullptr;
  int32_t* cnt = nullptr;
  dalloc(params, static_cast<size_t>(P_new) * D);
  dalloc(m, static_cast<size_t>(P_new) * D);
  dalloc(v, static_cast<size_t>(P_new) * D);
  dalloc(nu, P_new);
  dalloc(obs, P_new);
  dalloc(acc, P_new);
  dalloc(cnt, P_new);
  const size_t wb = sizeof(float) * static_cast<size_t>(P_new), ob = sizeof(float) * static_cast<size_t>(P_old);
  GSF_CUDA_CHECK(cudaMemset2DAsync(m, wb, 0, wb, D, c->stream));
  GSF_CUDA_CHECK(cudaMemset2DAsync(v, wb, 0, wb, D, c->stream));
  GSF_CUDA_CHECK(cudaMemsetAsync(acc, 0, sizeof(double) * P_new, c->stream));
  GSF_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * P_new, c->stream));
  if (P_old > 0) {
    GSF_CUDA_CHECK(cudaMemcpy2DAsync(params, wb, c->params, ob, ob, D, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpy2DAsync(m, wb, c->adam_m, ob, ob, D, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpy2DAsync(v, wb, c->adam_v, ob, ob, D, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(nu, c->nu, sizeof(double) * P_old, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(obs, c->observed, P_old, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(acc, c->grad_accum, sizeof(double) * P_old, cudaMemcpyDeviceToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(cnt, c->grad_count, sizeof(int32_t) * P_old, cudaMemcpyDeviceToDevice, c->stream));
  }
  sync(c);
  dfree(c->params); dfree(c->adam_m); dfree(c->adam_v); dfree(c->nu); dfree(c->observed); dfree(c->grad_accum);
  dfree(c->grad_count);
  c->params = params; c->adam_m = m; c->adam_v = v; c->nu = nu; c->observed = obs; c->grad_accum = acc;
  c->grad_count = cnt;
  dalloc(c->grads, static_cast<size_t>(P_new) * D);
  dalloc(c->d_mean2d, 2 * static_cast<size_t>(P_new));
  c->map_cap = P_new;
  c->P = P_new;
  ++c->map_gen;
}

int gsf_initialize_map(gsf_ctx c, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K, const gsf_mapper_cfg* mcfg,
                       int64_t* count) {
  return guard(c, [&] {
    check_mapper(*mcfg);
    check_intrinsics(*K);
    if (slot < 0 || slot >= static_cast<int>(c->frames.size()) || !c->frames[slot].rgb ||
        c->frames[slot].w != K->width || c->frames[slot].h != K->height)
      throw EInval("first frame dimensions do not match the intrinsics");
    const Frame& f = c->frames[slot];
    BackprojectArgs a;
    const uint32_t total = backproject_count(c, a, f, *pose, *K, *mcfg, mcfg->init_stride, nullptr);
    if (total == 0) throw ERuntime("cannot initialize a map: first frame has no usable depth");
    // a fresh MapState: the new primitives only, zero optimizer state and statistics
    c->P = 0;
    c->K = mcfg->sh_coeffs;
    c->D = kFieldsBase + 3 * c->K;
    grow_map_soa(c, total);
    run_backproject_write(a, c->bp_scratch + std::max<int64_t>(1, div_up(a.cells, 256)), 0, total, c->params, c->nu,
                          c->observed, c->stream, &c->launches);
    sync(c);
    c->adam_step = 0.0;
    c->rng_seeded = false;   // a fresh MapState: its rng restarts from the mapper seed
    c->map_iteration = 0;
    c->have_render = false;
    *count = total;
  });
}

int gsf_spawn_gaussians(gsf_ctx c, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K, const gsf_mapper_cfg* mcfg,
                        int32_t* spawned) {
  return guard(c, [&] {
    check_mapper(*mcfg);
    check_intrinsics(*K);
    *spawned = 0;
    if (!c->have_render || c->rK.width != K->width || c->rK.height != K->height)
      throw EInval("spawn render dimensions do not match the intrinsics");
    if (c->P > 0 && c->K != mcfg->sh_coeffs) throw EInval("spawn: sh coefficient count differs from the map's");
    if (slot < 0 || slot >= static_cast<int>(c->frames.size()) || !c->frames[slot].rgb ||
        c->frames[slot].w != K->width || c->frames[slot].h != K->height)
      throw EInval("spawn frame dimensions do not match the intrinsics");
    const Frame& f = c->frames[slot];
    BackprojectArgs a;
    const uint32_t total = backproject_count(c, a, f, *pose, *K, *mcfg, mcfg->spawn_stride, c->ws.opacity);
    if (total == 0) return;
    const int64_t P_old = c->P;
    if (P_old == 0) {
      c->K = mcfg->sh_coeffs;
      c->D = kFieldsBase + 3 * c->K;
    }
    grow_map_soa(c, P_old + total);
    run_backproject_write(a, c->bp_scratch + std::max<int64_t>(1, div_up(a.cells, 256)), P_old, P_old + total, c->params,
                          c->nu, c->observed, c->stream, &c->launches);
    sync(c);
    c->have_render = false;   // the render no longer describes this map
    *spawned = static_cast<int32_t>(total);
  });
}

// densify_and_cull (mapper.cpp:172-230) on the context's map: the per-primitive decisions run on
// the device, the host walks the codes in index order exactly like the reference loop (counts,
// output order, and the split offsets from the map state's std::mt19937_64 with one fresh
// std::normal_distribution per split parent), and the device builds the new SoA map.
static void draw3(double a, double b, double c, double* out) {
  out[0] = a;
  out[1] = b;
  out[2] = c;
}

static gsf_structural_change densify_and_cull(gsf_ctx_s* c, const gsf_mapper_cfg& m) {
  gsf_structural_change ch{0, 0, 0};
  const int64_t P = c->P;
  if (!c->rng_seeded) {
    c->rng.seed(m.seed);
    c->rng_seeded = true;
  }
  if (P == 0) return ch;
  uint8_t* d_code = nullptr;
  dalloc(d_code, P);
  run_densify_codes(c->params, P, c->grad_accum, c->grad_count, m.densify_cull_opacity, m.densify_grad_threshold,
                    m.densify_size_fraction * m.scene_extent, d_code, c->stream, &c->launches);
  std::vector<uint8_t> code(P);
  GSF_CUDA_CHECK(cudaMemcpyAsync(code.data(), d_code, P, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(d_code);
  std::vector<int32_t> src, zidx;
  std::vector<uint8_t> kind;
  std::vector<int32_t> app_src, app_z;
  std::vector<uint8_t> app_kind;
  std::vector<double> z;
  src.reserve(P);
  for (int64_t i = 0; i < P; ++i) {
    switch (code[i]) {
      case 0:
        ++ch.removed;
        break;
      case 2: {
        ++ch.split;
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (int child = 0; child < 2; ++child) {
          // the reference draws with `Vec3 z(gauss(rng), gauss(rng), gauss(rng))` (mapper.cpp:199):
          // the order of those argument evaluations is the compiler's; draw through a 3-argument
          // call as well so this build consumes the stream the way the reference's build does
          double zz[3];
          draw3(gauss(c->rng), gauss(c->rng), gauss(c->rng), zz);
          app_src.push_back(static_cast<int32_t>(i));
          app_kind.push_back(2);
          app_z.push_back(static_cast<int32_t>(z.size() / 3));
          z.insert(z.end(), zz, zz + 3);
        }
        break;
      }
      case 3:
        ++ch.cloned;
        src.push_back(static_cast<int32_t>(i));
        kind.push_back(0);
        zidx.push_back(0);
        app_src.push_back(static_cast<int32_t>(i));
        app_kind.push_back(1);
        app_z.push_back(0);
        break;
      default:
        src.push_back(static_cast<int32_t>(i));
        kind.push_back(0);
        zidx.push_back(0);
    }
  }
  if (ch.removed == 0 && ch.split == 0 && ch.cloned == 0) {
    GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_accum, 0, sizeof(double) * P, c->stream));
    GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_count, 0, sizeof(int32_t) * P, c->stream));
    return ch;
  }
  src.insert(src.end(), app_src.begin(), app_src.end());
  kind.insert(kind.end(), app_kind.begin(), app_kind.end());
  zidx.insert(zidx.end(), app_z.begin(), app_z.end());
  const int64_t P_new = static_cast<int64_t>(src.size());
  const int D = c->D;
  int32_t *d_src = nullptr, *d_zi = nullptr;
  uint8_t* d_kind = nullptr;
  double* d_z = nullptr;
  dalloc(d_src, std::max<int64_t>(P_new, 1));
  dalloc(d_zi, std::max<int64_t>(P_new, 1));
  dalloc(d_kind, std::max<int64_t>(P_new, 1));
  dalloc(d_z, std::max<size_t>(z.size(), 3));
  if (P_new > 0) {
    GSF_CUDA_CHECK(cudaMemcpyAsync(d_src, src.data(), sizeof(int32_t) * P_new, cudaMemcpyHostToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(d_zi, zidx.data(), sizeof(int32_t) * P_new, cudaMemcpyHostToDevice, c->stream));
    GSF_CUDA_CHECK(cudaMemcpyAsync(d_kind, kind.data(), P_new, cudaMemcpyHostToDevice, c->stream));
  }
  if (!z.empty())
    GSF_CUDA_CHECK(cudaMemcpyAsync(d_z, z.data(), sizeof(double) * z.size(), cudaMemcpyHostToDevice, c->stream));
  float *params = nullptr, *mm = nullptr, *vv = nullptr;
  double* nu = nullptr;
  uint8_t* obs = nullptr;
  const int64_t cap = std::max<int64_t>(P_new, 1);
  dalloc(params, static_cast<size_t>(cap) * D);
  dalloc(mm, static_cast<size_t>(cap) * D);
  dalloc(vv, static_cast<size_t>(cap) * D);
  dalloc(nu, cap);
  dalloc(obs, cap);
  run_densify_build(c->params, c->adam_m, c->adam_v, c->nu, c->observed, P, D, d_src, d_kind, d_zi, d_z,
                    std::log(m.densify_split_factor), P_new, params, mm, vv, nu, obs, c->stream, &c->launches);
  sync(c);
  dfree(d_src); dfree(d_zi); dfree(d_kind); dfree(d_z);
  dfree(c->params); dfree(c->adam_m); dfree(c->adam_v); dfree(c->nu); dfree(c->observed);
  c->params = params; c->adam_m = mm; c->adam_v = vv; c->nu = nu; c->observed = obs;
  dalloc(c->grads, static_cast<size_t>(cap) * D);
  dalloc(c->d_mean2d, 2 * static_cast<size_t>(cap));
  dalloc(c->grad_accum, cap);
  dalloc(c->grad_count, cap);
  GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_accum, 0, sizeof(double) * cap, c->stream));
  GSF_CUDA_CHECK(cudaMemsetAsync(c->grad_count, 0, sizeof(int32_t) * cap, c->stream));
  c->map_cap = cap;
  c->P = P_new;
  ++c->map_gen;
  c->have_render = false;
  return ch;
}

int gsf_densify_and_cull(gsf_ctx c, const gsf_mapper_cfg* mcfg, gsf_structural_change* out) {
  return guard(c, [&] {
    check_mapper(*mcfg);
    *out = densify_and_cull(c, *mcfg);
  });
}

int gsf_map_stats_upload(gsf_ctx c, const double* grad_accum, const int32_t* grad_count) {
  return guard(c, [&] {
    if (c->P == 0) return;
    GSF_CUDA_CHECK(cudaMemcpy(c->grad_accum, grad_accum, sizeof(double) * c->P, cudaMemcpyHostToDevice));
    GSF_CUDA_CHECK(cudaMemcpy(c->grad_count, grad_count, sizeof(int32_t) * c->P, cudaMemcpyHostToDevice));
  });
}

int gsf_map_stats_download(gsf_ctx c, double* grad_accum, int32_t* grad_count) {
  return guard(c, [&] {
    if (c->P == 0) return;
    sync(c);
    if (grad_accum) GSF_CUDA_CHECK(cudaMemcpy(grad_accum, c->grad_accum, sizeof(double) * c->P, cudaMemcpyDeviceToHost));
    if (grad_count) GSF_CUDA_CHECK(cudaMemcpy(grad_count, c->grad_count, sizeof(int32_t) * c->P, cudaMemcpyDeviceToHost));
  });
}

// render_reference (rasterizer.cpp:263-296): every pixel walks the full depth-sorted list with no
// early termination.  Every primitive a pixel can see (rho <= footprint_sigma^2) lies in that
// pixel's tile list (the tile rectangle bounds the same footprint disc), so this is the tiled
// render with the termination test disabled.
int gsf_render_reference(gsf_ctx c, const gsf_pose* pose, const gsf_intrinsics* K, const float* obs,
                         const gsf_raster_cfg* cfg, gsf_render_out* out) {
  gsf_raster_cfg nt = *cfg;
  nt.termination_threshold = 0.0;   // T < 0 never holds: no pixel terminates
  return gsf_render(c, pose, K, obs, &nt, out);
}

// GSFMAP01 checkpoint (io/checkpoint.cpp:11-100): little-endian; magic, 9 doubles of intrinsics,
// u32 SH bands, u64 count, per primitive mean 3, log_scale 3, quat 4, opacity logit, uncertainty
// (f64), observed (u8), SH bands x 3 (f64).  The device map is fp32, so a saved map is exact and a
// loaded fp64 map is rounded to fp32.
int gsf_checkpoint_save(gsf_ctx c, const char* path, const gsf_intrinsics* K) {
  return guard(c, [&] {
    if (!path || !K) throw EInval("checkpoint: null argument");
    const int64_t P = c->P;
    const int Ks = c->K;
    std::vector<double> mean(3 * P), ls(3 * P), quat(4 * P), op(P), sh(3 * Ks * std::max<int64_t>(P, 1)), nu(P);
    std::vector<uint8_t> ob(P);
    if (P > 0) {
      gsf_map_host m{P, Ks, mean.data(), ls.data(), quat.data(), op.data(), sh.data(), nu.data(), ob.data()};
      const int rc = gsf_map_download(c, &m);
      if (rc != GSF_OK) throw ERuntime(c->err);
    }
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw ERuntime(std::string("cannot open checkpoint for writing: ") + path);
    const char magic[8] = {'G', 'S', 'F', 'M', 'A', 'P', '0', '1'};
    const double header[9] = {K->fx, K->fy, K->cx, K->cy, double(K->width), double(K->height), K->depth_scale,
                              K->near_plane, K->far_plane};
    const uint32_t bands = static_cast<uint32_t>(std::max(Ks, 1));
    const uint64_t count = static_cast<uint64_t>(P);
    bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(header, sizeof(double), 9, f) == 9 &&
              std::fwrite(&bands, 4, 1, f) == 1 && std::fwrite(&count, 8, 1, f) == 1;
    for (int64_t i = 0; ok && i < P; ++i) {
      const uint8_t o = ob[i] ? 1 : 0;
      ok = std::fwrite(&mean[3 * i], sizeof(double), 3, f) == 3 && std::fwrite(&ls[3 * i], sizeof(double), 3, f) == 3 &&
           std::fwrite(&quat[4 * i], sizeof(double), 4, f) == 4 && std::fwrite(&op[i], sizeof(double), 1, f) == 1 &&
           std::fwrite(&nu[i], sizeof(double), 1, f) == 1 && std::fwrite(&o, 1, 1, f) == 1 &&
           std::fwrite(&sh[3 * Ks * i], sizeof(double), 3 * Ks, f) == static_cast<size_t>(3 * Ks);
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw ERuntime(std::string("failed writing checkpoint: ") + path);
  });
}

int gsf_checkpoint_load(gsf_ctx c, const char* path, gsf_intrinsics* K) {
  return guard(c, [&] {
    if (!path) throw EInval("checkpoint: null path");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw ERuntime(std::string("cannot open checkpoint: ") + path);
    auto rd = [&](void* dst, size_t bytes) {
      if (std::fread(dst, 1, bytes, f) != bytes) {
        std::fclose(f);
        throw ERuntime("checkpoint truncated");
      }
    };
    char magic[8];
    rd(magic, 8);
    if (std::memcmp(magic, "GSFMAP01", 8) != 0) {
      std::fclose(f);
      throw ERuntime(std::string("not a map checkpoint (bad magic): ") + path);
    }
    double header[9];
    rd(header, sizeof(header));
    uint32_t bands = 0;
    uint64_t count = 0;
    rd(&bands, 4);
    rd(&count, 8);
    if (bands == 0 || bands > 16) {
      std::fclose(f);
      throw ERuntime("checkpoint has invalid SH band count");
    }
    const int64_t P = static_cast<int64_t>(count);
    const int Ks = static_cast<int>(bands);
    std::vector<double> mean(3 * P), ls(3 * P), quat(4 * P), op(P), sh(3 * Ks * std::max<int64_t>(P, 1)), nu(P);
    std::vector<uint8_t> ob(P);
    for (int64_t i = 0; i < P; ++i) {
      rd(&mean[3 * i], 24);
      rd(&ls[3 * i], 24);
      rd(&quat[4 * i], 32);
      rd(&op[i], 8);
      rd(&nu[i], 8);
      rd(&ob[i], 1);
      rd(&sh[3 * Ks * i], sizeof(double) * 3 * Ks);
    }
    std::fclose(f);
    if (Ks != 1 && Ks != 4 && Ks != 9 && Ks != 16) throw EInval("sh coefficient count must be 1, 4, 9 or 16");
    gsf_map_host m{P, Ks, mean.data(), ls.data(), quat.data(), op.data(), sh.data(), nu.data(), ob.data()};
    const int rc = gsf_map_upload(c, &m);
    if (rc != GSF_OK) throw ERuntime(c->err);
    if (K) {
      K->fx = header[0]; K->fy = header[1]; K->cx = header[2]; K->cy = header[3];
      K->width = static_cast<int32_t>(header[4]);
      K->height = static_cast<int32_t>(header[5]);
      K->depth_scale = header[6]; K->near_plane = header[7]; K->far_plane = header[8];
    }
  });
}

int gsf_accumulate_uncertainty(gsf_ctx c, const int32_t* slots, const gsf_pose* poses, int32_t n, const gsf_intrinsics* K,
                               const gsf_raster_cfg* rcfg, int32_t* observed_count) {
  return guard(c, [&] {
    *observed_count = 0;
    if (n == 0) return;
    check_intrinsics(*K);
    check_raster(*rcfg);
    std::vector<const Frame*> fr(n);
    for (int i = 0; i < n; ++i) {
      if (slots[i] < 0 || slots[i] >= static_cast<int>(c->frames.size()) || !c->frames[slots[i]].rgb)
        throw EInval("uncertainty view missing record or depth");
      fr[i] = &c->frames[slots[i]];
      if (fr[i]->w != K->width || fr[i]->h != K->height) throw EInval("uncertainty view depth dimensions mismatch");
    }
    ensure_ws(c, K->width, K->height);
    if (c->P > c->unc_cap) {
      dalloc(c->unc_sum, c->P);
      dalloc(c->unc_cnt, c->P);
      c->unc_cap = c->P;
    }
    const int64_t P = c->P;
    if (P == 0) return;
    GSF_CUDA_CHECK(cudaMemsetAsync(c->unc_sum, 0, sizeof(double) * P, c->stream));
    GSF_CUDA_CHECK(cudaMemsetAsync(c->unc_cnt, 0, sizeof(uint32_t) * P, c->stream));
    // multi-GPU: rank g accumulates the views v = g (mod nranks) and the (sum, count) partials
    // are all-reduced before the division (Eq. 13 is order-invariant)
    for (int v = 0; v < n; ++v) {
      if (c->nranks > 1 && v % c->nranks != c->rank) continue;
      render_sync(c, poses[v], *K, *rcfg, fr[v]->depth);
      run_uncertainty_view(c->ws, c->params, P, fr[v]->depth, K->width, K->height, K->near_plane, K->far_plane, c->ds,
                           c->unc_sum, c->unc_cnt, c->stream, &c->launches);
    }
    if (c->nranks > 1) {
      allreduce(c, c->unc_sum, static_cast<size_t>(P), GSF_DT_F64, c->stream);
      allreduce(c, c->unc_cnt, static_cast<size_t>(P), GSF_DT_U32, c->stream);
    }
    GSF_CUDA_CHECK(cudaMemsetAsync(c->counters, 0, sizeof(uint32_t) * 16, c->stream));
    run_uncertainty_finalize(c->unc_sum, c->unc_cnt, c->nu, c->observed, P, c->counters, c->stream, &c->launches);
    uint32_t cnt = 0;
    GSF_CUDA_CHECK(cudaMemcpyAsync(&cnt, c->counters, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    *observed_count = static_cast<int32_t>(cnt);
  });
}

int gsf_prune_unreliable(gsf_ctx c, double tau, double reduced_opacity, int32_t* reduced) {
  return guard(c, [&] {
    if (!(tau > 0.0)) throw EInval("uncertainty threshold must be positive");
    if (!(reduced_opacity > 0.0 && reduced_opacity < 0.1)) throw EInval("reduced opacity must lie in (0, 0.1)");
    *reduced = 0;
    if (c->P == 0) return;
    if (!c->counters) dalloc(c->counters, 16);
    const float target = static_cast<float>(std::log(reduced_opacity / (1.0 - reduced_opacity)));
    GSF_CUDA_CHECK(cudaMemsetAsync(c->counters, 0, sizeof(uint32_t) * 16, c->stream));
    run_prune(c->nu, c->params + 10 * c->P, c->P, tau, target, c->counters, c->stream, &c->launches);
    uint32_t cnt = 0;
    GSF_CUDA_CHECK(cudaMemcpyAsync(&cnt, c->counters, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    *reduced = static_cast<int32_t>(cnt);
    ++c->map_gen;
  });
}

}  // extern "C"
