// raster_bwd.cu — reverse-order backward of the tile rasterizer on sm_100a.
//
// k_backward_q        render_backward phase 1 (rasterizer.cpp:374-464) for the full gradient bundle
//                     (mapping, the render_backward API): one single-warp CTA per (16x16 tile, 8x8
//                     quadrant), two pixels per lane, walking the tile list back to front from its
//                     pixels' last contributor.  Every pair is re-evaluated with the forward's exact
//                     decision arithmetic (gsf_shared.cuh), T is recovered by division from the final
//                     transmittance, and an entry's ten screen-space partials are reduced across the
//                     warp (reduce-scatter) and written ONCE into the (pair, quadrant) slot.
// k_pair_combine      folds the four quadrant slots of every (tile, primitive) pair in quadrant order.
// k_big_sum           pre-sums the pair slots of the large-footprint primitives (> kBigPairs tiles),
//                     one CTA each, for k_chain.
// k_backward_track_w  the tracking (pose-only) backward: the same walk over the forward's per-quadrant
//                     work lists, each lane contracting its pixels' partials with the entry's SE(3)
//                     Jacobian (k_posejac) so no per-pair partial is stored; the last CTA sums the
//                     rows and runs the pose step.  k_backward_pose: the view-dependent-SH variant.
// k_chain             phase 2 (rasterizer.cpp:480-570) in fp64, one thread per visible primitive (4 x 148
//                     CTAs strided over the visible list): a fixed-order gather of its pair slots (the
//                     reference's tile-order reduction, :466-478; warp-cooperative above 16 slots,
//                     k_big_sum's totals above kBigPairs), the projection/covariance chain, the SE(3) pose pieces and the
//                     world-parameter gradients; the pose 6-vector is reduced block-wise in fp64.
// k_pose_sum          fixed-order sum of the per-block pose partials (rasterizer.cpp:570).
// No float atomics on any path: results are bit-repeatable.
#include <stdexcept>

#include "kernels.h"
#include "pixel_loss.cuh"
#include "finalize.cuh"

namespace gsfk {

namespace {

// Field layout of a pair partial: 0,1 d_mean2d; 2,3,4 d_cov2d (00, 01=10, 11); 5 d_depth;
// 6,7,8 d_color; 9 d_sigma.  Pose-only mode keeps the first 6 (or 9 with view-dependent SH).
template <int N, int LO>
__device__ __forceinline__ void rs_step(float* f, bool upper, int off) {
#pragma unroll
  for (int i = 0; i < LO; ++i) {
    const float hi = (LO + i < N) ? f[LO + i] : 0.0f;
    const float send = upper ? f[i] : hi;
    const float keep = upper ? hi : f[i];
    f[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
  }
}

template <int NF>
__device__ __forceinline__ float warp_reduce_scatter(float* f, int lane) {
  constexpr int n1 = (NF + 1) / 2, n2 = (n1 + 1) / 2, n3 = (n2 + 1) / 2, n4 = (n3 + 1) / 2, n5 = (n4 + 1) / 2;
  rs_step<NF, n1>(f, lane & 16, 16);
  rs_step<n1, n2>(f, lane & 8, 8);
  rs_step<n2, n3>(f, lane & 4, 4);
  rs_step<n3, n4>(f, lane & 2, 2);
  rs_step<n4, n5>(f, lane & 1, 1);
  return f[0];
}

__device__ __forceinline__ int rs_field(int nf, int lane, bool& valid) {
  int base = 0, n = nf, end = nf;
  for (int off = 16; off >= 1; off >>= 1) {
    const int lo = (n + 1) / 2;
    if (lane & off) {
      end = min(end, base + n);
      base += lo;
    } else {
      end = min(end, base + lo);
    }
    n = lo;
  }
  valid = base < end;
  return base;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float sgnf(float v) { return v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : 0.0f); }

__device__ __forceinline__ bool dvalid(float d, double near_plane, double far_plane) {
  const double v = d;
  return isfinite(v) && v > near_plane && v < far_plane;
}

struct BwdPtrs {
  const int2* ranges;
  const uint32_t* sid;      // tile lists (primitive ids) in (depth, id) order
  const BlendG* bg;         // id-indexed
  const GuardG* gg;
  const float* color;
  const float* alpha_depth;
  const float* median_depth;
  const uint8_t* median_valid;
  const float* opacity;
  const float* final_T;
  const int32_t* last;
  const int32_t* median_prim;
  const float* obs;
  const float* target;
  const float* up_color;
  const float* up_adepth;
  const float* up_mdepth;
  const float* up_opacity;
  const float* up_uncert;
  const float* dssim;
  float* partials;
  const int4* rect;         // id-indexed tile rectangles
  const uint32_t* pair_base;  // id -> first primitive-major partial slot
  const float* pj;          // pose Jacobians (fused tracking mode), 36 floats at the primitive's slot
  const uint32_t* pj_slot;  // id -> slot in pj (position in the visible list)
  double* tile_pose;     // per-tile pose partials (fused tracking mode)
  const uint32_t* qlist;    // tracking: per (tile, quadrant) work lists (k_blend_track)
  const int32_t* lastc;     // tracking: each pixel's last contributor as a work-list position + 1
  uint8_t* qflag;           // full bundle: per (pair, quadrant) written flag (k_backward_q)
  float* qpart;             // full bundle: [pair][quadrant][10] partials (k_backward_q)
  const uint8_t* pxcode;    // tracking: per pixel, the seed signs (pixel_seed_code, k_blend_track)
  const BlendG* bg_slot;    // tracking: records by visible slot
  const GuardG* gg_slot;
};

// Per-pixel backward inputs (rasterizer.cpp:395-413): seeds, final T and the contributor limit.
struct PixBwd {
  float gc0, gc1, gc2, gad, gop, gmd, gu, D, T;
  int med, last;
};

template <int SEED>
__device__ __forceinline__ PixBwd load_pixel_bwd(const BwdPtrs& bp, int64_t pi, bool inside, const LossParams& lp,
                                                 const DevState* ds, double near_plane, double far_plane) {
  PixBwd p;
  p.gc0 = p.gc1 = p.gc2 = p.gad = p.gop = p.gmd = p.gu = p.D = 0.0f;
  p.T = 1.0f;
  p.med = -1;
  p.last = 0;
  if (!inside) return p;
  p.last = bp.last[pi];
  p.T = bp.final_T[pi];
  p.med = bp.median_prim[pi];
  if (SEED == SEED_EXPLICIT) {
    if (bp.up_color) { p.gc0 = bp.up_color[3 * pi]; p.gc1 = bp.up_color[3 * pi + 1]; p.gc2 = bp.up_color[3 * pi + 2]; }
    if (bp.up_adepth) p.gad = bp.up_adepth[pi];
    if (bp.up_opacity) p.gop = bp.up_opacity[pi];
    if (bp.up_mdepth) p.gmd = bp.up_mdepth[pi];
    if (bp.up_uncert && lp.uncertainty_full_gradient) p.gu = bp.up_uncert[pi];
    if (bp.obs) {
      p.D = bp.obs[pi];
      if (!dvalid(p.D, near_plane, far_plane)) p.gu = 0.f;
    } else {
      p.gu = 0.f;
    }
  } else {
    const PixSeeds sd = seeds_pixel<SEED == SEED_TRACK ? 1 : 2>(pi, bp.color, bp.alpha_depth[pi], bp.median_depth[pi],
                                                                bp.median_valid[pi] != 0, bp.opacity[pi], bp.target,
                                                                bp.obs, bp.dssim, ds, lp, near_plane, far_plane);
    p.gc0 = sd.gc0; p.gc1 = sd.gc1; p.gc2 = sd.gc2; p.gad = sd.gad; p.gmd = sd.gmd;
    p.gu = lp.uncertainty_full_gradient ? sd.gu : 0.0f;
    if (SEED == SEED_MAP && bp.obs) p.D = bp.obs[pi];
  }
  if (p.med < 0) p.gmd = 0.f;
  if (p.gc0 == 0.f && p.gc1 == 0.f && p.gc2 == 0.f && p.gad == 0.f && p.gop == 0.f && p.gmd == 0.f && p.gu == 0.f)
    p.last = 0;
  return p;
}

// Mapping / full-bundle backward (render_backward phase 1, rasterizer.cpp:374-464) as independent
// single-warp CTAs: CTA 4 t + q owns quadrant q (8x8 pixels, two per lane: (l & 7, l >> 3) and
// (l & 7, (l >> 3) + 4)) of tile t and walks the tile list back to front from its pixels' last
// contributor in chunks of 32 entries.  Lane e stages entry e of the chunk (record, rectangle and
// pair base by cp.async, the id two chunks ahead), tests it against the quadrant's block
// (block_hit8), and the warp walks the set bits.  Per entry the two pixels' ten partials are summed
// per lane, reduced across the warp (reduce-scatter) and written ONCE to the (pair, quadrant) slot
// (partials [pair][4][10]); no CTA barriers, no float atomics.  Fields 0..4 are kept in the
// pixel-offset basis t = g (dx, dy, dx^2, dx dy, dy^2) (k_chain re-expresses them with the conic),
// so a step forms them from the shared dx.  k_chain reads every (pair, quadrant) slot in a fixed
// order and zeroes it, so slots no quadrant walked read 0 on the next backward.
constexpr int kBqChunk = 32;
#ifndef GSF_BQ_MINB
#define GSF_BQ_MINB 20
#endif
template <int SEED>
__global__ void __launch_bounds__(32, GSF_BQ_MINB) k_backward_q(BwdPtrs bp, int W, int H, int tiles_x, BlendConsts kc,
                                                               double near_plane, double far_plane, LossParams lp,
                                                               const DevState* ds, const uint32_t* __restrict__ order,
                                                               int64_t tiles_cap) {
  // per buffer (2): 32 records (48 B) at +0, 32 rectangles (16 B) at +1536, 32 pair bases at +2048,
  // 32 ids at +2176; 2304 B per buffer
  __shared__ float4 s_buf[2 * 144];
  pdl_wait();
  pdl_trigger();
  if (ds->halt) return;
  const int lane = threadIdx.x;
  const uint32_t sb = opaque_smem_base(s_buf);
  // (tile, quadrant) item in longest-first order (k_lpt over the forward's per-quadrant steps)
  const int item = (order && 4u * order[0] == gridDim.x) ? static_cast<int>(order[1 + tiles_cap + blockIdx.x])
                                                         : static_cast<int>(blockIdx.x);
  const int tile = item >> 2, qd = item & 3;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int bx0 = tx * kTile + 8 * (qd & 1), by0 = ty * kTile + 8 * (qd >> 1);
  const int x = bx0 + (lane & 7);
  const int ya = by0 + (lane >> 3), yb = ya + 4;
  const bool in_a = x < W && ya < H, in_b = x < W && yb < H;
  const PixBwd qa = load_pixel_bwd<SEED>(bp, static_cast<int64_t>(ya) * W + x, in_a, lp, ds, near_plane, far_plane);
  const PixBwd qb = load_pixel_bwd<SEED>(bp, static_cast<int64_t>(yb) * W + x, in_b, lp, ds, near_plane, far_plane);
  const int last_a = qa.last, last_b = qb.last;
  const int maxlast = __reduce_max_sync(0xffffffffu, max(last_a, last_b));
  if (maxlast == 0) return;
  const int2 rg = bp.ranges[tile];
  const float2 gc0 = make_float2(qa.gc0, qb.gc0), gc1 = make_float2(qa.gc1, qb.gc1), gc2 = make_float2(qa.gc2, qb.gc2),
               gad = make_float2(qa.gad, qb.gad), gop = make_float2(qa.gop, qb.gop), gu = make_float2(qa.gu, qb.gu),
               Dd = make_float2(qa.D, qb.D);
  const float gmd_a = qa.gmd, gmd_b = qb.gmd;
  const int med_a = qa.med, med_b = qb.med;
  const float px = static_cast<float>(x) + 0.5f;
  const float2 py = make_float2(static_cast<float>(ya) + 0.5f, static_cast<float>(yb) + 0.5f);
  float2 T = make_float2(qa.T, qb.T), S = make_float2(0.f, 0.f);
  bool fvalid;
  const int fidx = rs_field(10, lane, fvalid);
  const int E = rg.x + maxlast;
  const int nch = (maxlast + kBqChunk - 1) / kBqChunk;
  // chunk c: list entries [lo, hi) with hi = E - 32 c; lane e holds entry hi - 1 - e (back to front)
  auto fetch = [&](int c) -> int32_t {
    if (c >= nch) return -1;
    const int j = E - kBqChunk * c - 1 - lane;
    return j >= rg.x ? static_cast<int32_t>(__ldg(bp.sid + j)) : -1;
  };
  auto issue = [&](int c, int32_t id) {
    if (c < nch && id >= 0) {
      const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 2304u;
      const float4* rec = reinterpret_cast<const float4*>(bp.bg + id);
      cp_async16_to(buf + 48u * lane, rec);
      cp_async16_to(buf + 48u * lane + 16u, rec + 1);
      cp_async16_to(buf + 48u * lane + 32u, rec + 2);
      cp_async16_to(buf + 1536u + 16u * lane, bp.rect + id);
      sts_s32(buf + 2176u + 4u * lane, id);
      sts_s32(buf + 2048u + 4u * lane, static_cast<int32_t>(__ldg(bp.pair_base + id)));
    }
    cp_async_commit();
  };
  int32_t id0 = fetch(0), id1 = fetch(1);
  issue(0, id0);
  const float qx0 = static_cast<float>(bx0), qy0 = static_cast<float>(by0);
  for (int c = 0; c < nch; ++c) {
    issue(c + 1, id1);
    const int32_t id2 = fetch(c + 2);
    cp_async_wait_1();
    __syncwarp();
    const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 2304u;
    const int hi = E - kBqChunk * c;
    bool hit = false;
    if (id0 >= 0) hit = block_hit8(lds_blend(buf + 48u * lane), qx0, qy0, kc);
    uint32_t bits = __ballot_sync(0xffffffffu, hit);
    while (bits) {
      const int e = __ffs(bits) - 1;   // lowest lane = latest entry: back to front
      bits &= bits - 1u;
      const int li = hi - 1 - e - rg.x;
      const BlendG g = lds_blend(buf + 48u * e);
      const float dx = __fadd_rn(px, -g.mx);
      const float2 dy = __fadd2_rn(py, make_float2(-g.my, -g.my));
      const float2 rho = pair_rho2(dx, dy, g);
      const bool skip_a = li >= last_a || rho.x > g.rho_hi, skip_b = li >= last_b || rho.y > g.rho_hi;
      if (__all_sync(0xffffffffu, skip_a && skip_b)) continue;
      const bool fast_a = rho.x < g.rho_fast, fast_b = rho.y < g.rho_fast;
      float2 gv = make_float2(exp_neg_half_fast(rho.x), exp_neg_half_fast(rho.y));
      bool ca = !skip_a && fast_a, cb = !skip_b && fast_b;
      gv = make_float2(ca ? gv.x : 0.0f, cb ? gv.y : 0.0f);
      float2 al = __fmul2_rn(make_float2(g.sigma, g.sigma), gv);   // 0 where the pixel does not take the entry
      float2 gz = gv;                                              // gval where the gradient flows (0 if clamped)
      const int32_t eid = lds_s32(buf + 2176u + 4u * e);
      if (!skip_a && !fast_a) {
        const GuardOut o = guard_decide(px, py.x, g, bp.gg + eid, &kc);
        ca = o.alpha >= 0.0f;
        al.x = ca ? o.alpha : 0.0f;
        gz.x = ca && !o.clamped ? o.gval : 0.0f;
      }
      if (!skip_b && !fast_b) {
        const GuardOut o = guard_decide(px, py.y, g, bp.gg + eid, &kc);
        cb = o.alpha >= 0.0f;
        al.y = cb ? o.alpha : 0.0f;
        gz.y = cb && !o.clamped ? o.gval : 0.0f;
      }
      const bool contrib = ca || cb;
      if (!__any_sync(0xffffffffu, contrib)) continue;
      const float2 inv = make_float2(rcp_approx(1.0f - al.x), rcp_approx(1.0f - al.y));
      const float2 Tpre = __fmul2_rn(T, inv);
      const float2 derr = __fadd2_rn(make_float2(g.depth, g.depth), make_float2(-Dd.x, -Dd.y));
      float2 q = __ffma2_rn(gu, __fmul2_rn(derr, derr), gop);
      q = __ffma2_rn(gc0, make_float2(g.r, g.r), q);
      q = __ffma2_rn(gc1, make_float2(g.g, g.g), q);
      q = __ffma2_rn(gc2, make_float2(g.b, g.b), q);
      q = __ffma2_rn(gad, make_float2(g.depth, g.depth), q);
      const float2 dal = __ffma2_rn(Tpre, q, __fmul2_rn(make_float2(-S.x, -S.y), inv));
      const float2 w = __fmul2_rn(al, Tpre);
      S = __ffma2_rn(w, q, S);
      T = Tpre;
      const float2 dgz = __fmul2_rn(gz, dal);                                   // d opacity-logit partial
      const float2 gdg = __fmul2_rn(dgz, make_float2(g.sigma, g.sigma));        // d rho partial (x -1/2 folded)
      float f[10];
      {
        const float G = gdg.x + gdg.y;
        const float2 gy = __fmul2_rn(gdg, dy), gy2 = __fmul2_rn(gy, dy);
        f[1] = gy.x + gy.y;
        f[0] = dx * G;
        f[2] = (dx * dx) * G;
        f[3] = dx * f[1];
        f[4] = gy2.x + gy2.y;
        const float2 dd = __ffma2_rn(make_float2(2.0f, 2.0f), __fmul2_rn(gu, derr), gad);
        const float2 f5 = __fmul2_rn(w, dd);
        f[5] = (f5.x + (ca && eid == med_a ? gmd_a : 0.0f)) + (f5.y + (cb && eid == med_b ? gmd_b : 0.0f));
        const float2 c0 = __fmul2_rn(w, gc0), c1 = __fmul2_rn(w, gc1), c2 = __fmul2_rn(w, gc2);
        f[6] = c0.x + c0.y;
        f[7] = c1.x + c1.y;
        f[8] = c2.x + c2.y;
        f[9] = dgz.x + dgz.y;
      }
      const float val = warp_reduce_scatter<10>(f, lane);
      const int4 rq = lds_i4(buf + 1536u + 16u * e);
      const uint32_t slot = static_cast<uint32_t>(lds_s32(buf + 2048u + 4u * e)) +
                            static_cast<uint32_t>((ty - rq.z) * (rq.y - rq.x + 1) + (tx - rq.x));
      if (fvalid) bp.qpart[(static_cast<size_t>(slot) * 4 + qd) * 10 + fidx] = val;
      if (lane == 0) bp.qflag[static_cast<size_t>(slot) * 4 + qd] = 1;
    }
    __syncwarp();   // buffer c & 1 is refilled by issue(c + 2)
    id0 = id1;
    id1 = id2;
  }
  cp_async_wait_all();
}

// Tracking pixel inputs from the fused forward's seed signs: seeds_pixel<1>'s values (the same
// global scale times the same sign), three loads instead of the maps, target and sensor depth.
__device__ __forceinline__ PixBwd track_pixel_bwd(const BwdPtrs& bp, int64_t pi, bool inside, const DevState* ds) {
  PixBwd p;
  p.gop = p.gmd = p.gu = p.D = 0.0f;
  p.med = -1;
  p.gc0 = p.gc1 = p.gc2 = p.gad = 0.0f;
  p.T = 1.0f;
  p.last = 0;
  if (!inside) return p;
  const uint32_t code = bp.pxcode[pi];
  const int last = bp.lastc[pi];
  p.T = bp.final_T[pi];
  const float sc = static_cast<float>(ds->seed_color), sg = static_cast<float>(ds->seed_geo);
  p.gc0 = sc * code_sgn(code & 3u);
  p.gc1 = sc * code_sgn((code >> 2) & 3u);
  p.gc2 = sc * code_sgn((code >> 4) & 3u);
  p.gad = sg * code_sgn(code >> 6);
  // all seeds zero: nothing to propagate (rasterizer.cpp:411-413)
  p.last = (p.gc0 != 0.f || p.gc1 != 0.f || p.gc2 != 0.f || p.gad != 0.f) ? last : 0;
  return p;
}

// Tracking backward (pose only).  The pose gradient is linear in every pair's screen-space
// gradient, so each lane pushes its own pixel's screen gradient through the primitive's SE(3)
// Jacobian (compute_posejac) and accumulates the 6-vector in registers: no per-(tile, primitive)
// cross-lane reduction, no pair partials in memory, no per-primitive chain kernel.  Lane sums
// are fp32 within a batch and fp64 across batches; the CTA reduces them in a fixed tree.
#ifndef GSF_POSE_BATCH
#define GSF_POSE_BATCH 256
#endif
constexpr int kPoseBatch = GSF_POSE_BATCH;   // one batch covers most tile lists: one staging barrier

template <bool VIEWDEP>
constexpr size_t pose_smem_bytes() {
  return static_cast<size_t>(kPoseBatch) * (sizeof(BlendG) + (VIEWDEP ? 14 : 9) * sizeof(float4) + sizeof(int32_t) + 1);
}

template <int SEED, bool VIEWDEP>
__global__ void __launch_bounds__(256, 4) k_backward_pose(BwdPtrs bp, int W, int H, int tiles_x, BlendConsts kc,
                                                       double near_plane, double far_plane, LossParams lp,
                                                       DevState* ds, uint32_t* ticket) {
  constexpr int kM4 = VIEWDEP ? 14 : 9;   // float4s of the pose matrix the kernel needs
  extern __shared__ float4 s_dyn[];         // pose_smem_bytes<VIEWDEP>()
  float4 (*s_pj)[kM4] = reinterpret_cast<float4 (*)[kM4]>(s_dyn);
  BlendG* s_g = reinterpret_cast<BlendG*>(s_dyn + kPoseBatch * kM4);
  int32_t* s_id = reinterpret_cast<int32_t*>(s_g + kPoseBatch);
  uint8_t* s_mask = reinterpret_cast<uint8_t*>(s_id + kPoseBatch);
  __shared__ int s_wmax[8];
  __shared__ double s_pred[8][6];
  const int tile = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ds->halt) {   // halted loop: zero gradient, no update (k_pose_sum semantics)
    __shared__ int s_last0;
    if (last_cta(ticket, &s_last0, false) && tid < 6) ds->d_pose[tid] = 0.0;
    return;
  }
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x = tx * kTile + tile_lx(tid), y = ty * kTile + tile_ly(tid);
  const bool inside = x < W && y < H;
  const int64_t pi = static_cast<int64_t>(y) * W + x;
  const int2 rg = bp.ranges[tile];
  PixBwd pb = load_pixel_bwd<SEED>(bp, pi, inside, lp, ds, near_plane, far_plane);
  const int ml = __reduce_max_sync(0xffffffffu, pb.last);
  if (lane == 0) s_wmax[warp] = ml;
  __syncthreads();
  int maxlast = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) maxlast = max(maxlast, s_wmax[w]);
  const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
  const float tile_x0 = static_cast<float>(tx * kTile), tile_y0 = static_cast<float>(ty * kTile);
  float T = pb.T, S = 0.0f;
  if (lane < 6) s_pred[warp][lane] = 0.0;   // per-warp fp64 sums across batches (fixed order)
  const int end = rg.x + maxlast;
  for (int bend = end; bend > rg.x; bend -= kPoseBatch) {
    const int bstart = max(rg.x, bend - kPoseBatch);
    const int cnt = bend - bstart;
    if (tid < cnt) {
      const int id = static_cast<int>(bp.sid[bstart + tid]);
      const BlendG gj = bp.bg[id];
      s_g[tid] = gj;
      s_id[tid] = id;
      s_mask[tid] = static_cast<uint8_t>(warp_block_mask(gj, tile_x0, tile_y0, kc));
    }
    __syncthreads();
    for (int i = tid; i < cnt * kM4; i += 256) {
      const int k = i / kM4, j = i - kM4 * k;
      if (s_mask[k])   // entries no warp block can see are never read
        s_pj[k][j] = reinterpret_cast<const float4*>(bp.pj)[(kPjFloats / 4) * static_cast<size_t>(bp.pj_slot[s_id[k]]) + j];
    }
    __syncthreads();
    // (rot0, rot1), (rot2, trans0), (trans1, trans2) of this batch, accumulated with FFMA2
    float2 pa = make_float2(0.f, 0.f), pb2 = make_float2(0.f, 0.f), pc2 = make_float2(0.f, 0.f);
    // back to front over only the entries whose footprint can reach this warp's block
    for (int c0 = ((cnt - 1) >> 5) << 5; c0 >= 0; c0 -= 32) {
     const int kk = c0 + lane;
     uint32_t bits = __ballot_sync(0xffffffffu, kk < cnt && ((s_mask[kk] >> warp) & 1u));
     while (bits) {
      const int j = 31 - __clz(bits);
      bits &= ~(1u << j);
      const int k = c0 + j;
      const int li = bstart + k - rg.x;
      if (li >= pb.last) continue;
      const BlendG g = s_g[k];
      const PairEval e = eval_pair_t<true>(px, py, g, bp.gg + s_id[k], kc);
      if (!e.code) continue;
      const float alpha = e.alpha;
      const float inv = rcp_approx(1.0f - alpha);
      const float Tpre = T * inv;
      // the tracking loss seeds colour and alpha depth only (losses.cpp:284-339): no opacity,
      // median-depth or uncertainty seeds on that path
      constexpr bool kTrack = SEED == SEED_TRACK;
      const float derr = kTrack ? 0.0f : g.depth - pb.D;
      const float2 q2 = __ffma2_rn(make_float2(pb.gc2, pb.gad), make_float2(g.b, g.depth),
                                   __fmul2_rn(make_float2(pb.gc0, pb.gc1), make_float2(g.r, g.g)));
      float q = q2.x + q2.y;
      if (!kTrack) q += pb.gop + pb.gu * derr * derr;
      const float dal = Tpre * q - S * inv;
      const float w = alpha * Tpre;
      S += w * q;
      T = Tpre;
      const float s5 = kTrack ? w * pb.gad
                              : w * (pb.gad + 2.0f * pb.gu * derr) + (s_id[k] == pb.med ? pb.gmd : 0.0f);
      float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
      float s4 = 0.f;
      if (!e.clamped) {
        const float gdg = e.gval * (dal * g.sigma);
        const float c01 = 0.5f * g.c01x2;
        const float2 u = __ffma2_rn(make_float2(c01, g.c11), make_float2(e.dy, e.dy),
                                    __fmul2_rn(make_float2(g.c00, c01), make_float2(e.dx, e.dx)));
        const float ux = u.x, uy = u.y;
        s01 = __fmul2_rn(make_float2(gdg, gdg), u);   // d_mean2d
        s23 = __fmul2_rn(make_float2(s01.x, s01.x), make_float2(ux, uy)); // 2 x d_cov 00, 01
        s4 = s01.y * uy;                                                 // 2 x d_cov 11
      }
      // pose += M s, M column-major (compute_posejac): columns 0..5, then the colour columns
      const float4* M = s_pj[k];
#define GSF_COL(F4A, F4B, F4C, SV)                                                    \
      {                                                                               \
        const float2 sv = make_float2(SV, SV);                                        \
        pa = __ffma2_rn(sv, F4A, pa);                                                 \
        pb2 = __ffma2_rn(sv, F4B, pb2);                                               \
        pc2 = __ffma2_rn(sv, F4C, pc2);                                               \
      }
      const float4 m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3], m4 = M[4], m5 = M[5], m6 = M[6], m7 = M[7], m8 = M[8];
      GSF_COL(make_float2(m0.x, m0.y), make_float2(m0.z, m0.w), make_float2(m1.x, m1.y), s01.x)
      GSF_COL(make_float2(m1.z, m1.w), make_float2(m2.x, m2.y), make_float2(m2.z, m2.w), s01.y)
      GSF_COL(make_float2(m3.x, m3.y), make_float2(m3.z, m3.w), make_float2(m4.x, m4.y), s23.x)
      GSF_COL(make_float2(m4.z, m4.w), make_float2(m5.x, m5.y), make_float2(m5.z, m5.w), s23.y)
      GSF_COL(make_float2(m6.x, m6.y), make_float2(m6.z, m6.w), make_float2(m7.x, m7.y), s4)
      GSF_COL(make_float2(m7.z, m7.w), make_float2(m8.x, m8.y), make_float2(m8.z, m8.w), s5)
      if (VIEWDEP) {
        const float4 m9 = M[9], m10 = M[10], m11 = M[11], m12 = M[12], m13 = M[13];
        GSF_COL(make_float2(m9.x, m9.y), make_float2(m9.z, m9.w), make_float2(m10.x, m10.y), w * pb.gc0)
        GSF_COL(make_float2(m10.z, m10.w), make_float2(m11.x, m11.y), make_float2(m11.z, m11.w), w * pb.gc1)
        GSF_COL(make_float2(m12.x, m12.y), make_float2(m12.z, m12.w), make_float2(m13.x, m13.y), w * pb.gc2)
      }
#undef GSF_COL
     }
    }
    {   // lane sums (fp32 within the batch) -> warp sum in fp64 -> the warp's running total
      const float lv[6] = {pa.x, pa.y, pb2.x, pb2.y, pc2.x, pc2.y};
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        double v = lv[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) s_pred[warp][a] += v;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid < 6) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_pred[w][tid];
    bp.tile_pose[static_cast<size_t>(tile) * 6 + tid] = t;
  }
  // the last tile CTA sums the tile partials in a fixed order (k_pose_sum without a launch)
  __shared__ int s_last;
  __shared__ double s_pose[6];
  if (last_cta(ticket, &s_last, tid < 6)) {
    block_reduce_rows<6>(bp.tile_pose, gridDim.x, s_pose, s_pred);
    if (tid < 6) ds->d_pose[tid] = s_pose[tid];
  }
}

// Tracking backward (k_backward_pose<SEED_TRACK, false>) with two pixels per lane, the layout of
// k_blend_track: the pair arithmetic of both pixels runs on packed FP32x2 (shared dx); their
// screen-space gradients are added before the contraction with the entry's pose matrix, so the
// 18 FFMA2 of M s and the staging reads are paid once per two pixels.  Decisions (contributes /
// clamped) are the forward's: same rho, same tests.
//
// Independent single-warp CTAs: CTA 4 t + q owns quadrant q (8x8
// pixels, two per lane) of tile t and walks the tile list back to front in chunks of 32 entries,
// one per lane: the lane stages its entry, tests it against the warp's block and, if it can
// reach it, stages the entry's pose matrix.  No CTA barriers: a warp that has passed its
// pixels' last contributors retires and frees its slot.  Per-warp pose rows are reduced by
// warp_grid_reduce (fixed order).
#ifndef GSF_TBW_MINB
#define GSF_TBW_MINB 22
#endif
__global__ void __launch_bounds__(32, GSF_TBW_MINB) k_backward_track_w(BwdPtrs bp, int W, int H, int tiles_x,
                                                                      BlendConsts kc, double near_plane,
                                                                      double far_plane, LossParams lp, DevState* ds,
                                                                      uint32_t* gtickets, int rows, int upd_iter,
                                                                      double bc1, double bc2, const uint32_t* __restrict__ order,
                                                                      int64_t tiles_cap) {
  // one staging buffer: 32 records (3 float4), 32 pose matrices (9 float4), 32 slots
  // two staging buffers of 16 entries: records (3 float4) at +0, pose matrices (9 float4) at +768 B;
  // their slots at 6144 + 64 b
  __shared__ float4 s_buf[2 * 16 * 12 + 8];
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x;
  const uint32_t sb = opaque_smem_base(s_buf);
  // (tile, quadrant) item in longest-first order (k_lpt; identity when the order is for another grid)
  const int item = (order && 4u * order[0] == gridDim.x) ? static_cast<int>(order[1 + tiles_cap + blockIdx.x])
                                                         : static_cast<int>(blockIdx.x);
  const int tile = item >> 2, qd = item & 3;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x = tx * kTile + 8 * (qd & 1) + (lane & 7);
  const int ya = ty * kTile + 8 * (qd >> 1) + (lane >> 3), yb = ya + 4;
  const bool in_a = x < W && ya < H, in_b = x < W && yb < H;
  double pd[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (!ds->halt) {
    const int2 rg = bp.ranges[tile];
    const PixBwd qa = track_pixel_bwd(bp, static_cast<int64_t>(ya) * W + x, in_a, ds);
    const PixBwd qb = track_pixel_bwd(bp, static_cast<int64_t>(yb) * W + x, in_b, ds);
    const int last_a = qa.last, last_b = qb.last;
    const int maxlast = __reduce_max_sync(0xffffffffu, max(last_a, last_b));
    const float2 gc0 = make_float2(qa.gc0, qb.gc0), gc1 = make_float2(qa.gc1, qb.gc1), gc2 = make_float2(qa.gc2, qb.gc2),
                 gad = make_float2(qa.gad, qb.gad);
    const float px = static_cast<float>(x) + 0.5f;
    const float2 py = make_float2(static_cast<float>(ya) + 0.5f, static_cast<float>(yb) + 0.5f);
    float2 T = make_float2(qa.T, qb.T), S = make_float2(0.f, 0.f);
    // The quadrant's work list (the entries of the tile list whose footprint can reach this 8x8
    // block, recorded by the forward's walk) is walked back to front from the pixels' last
    // contributor in chunks of kC = 16 entries, double-buffered: while chunk c is processed, the
    // records and pose matrices of chunk c + 1 stream into the other buffer with cp.async, and the
    // slots of chunk c + 2 load into registers (lanes 0..15).
    constexpr int kC = 16;
    const int E = maxlast;
    const int nch = (maxlast + kC - 1) / kC;
    const uint32_t* ql = bp.qlist + 4 * static_cast<int64_t>(rg.x) + static_cast<int64_t>(qd) * (rg.y - rg.x);
    auto fetch = [&](int c, uint32_t& m, uint32_t& sl) {
      m = 0u;
      sl = 0u;
      if (c < nch) {
        const int lo = max(0, E - kC * (c + 1)), hi = E - kC * c;
        if (lane < hi - lo) {
          m = 1u;
          sl = __ldg(ql + lo + lane);
        }
      }
    };
    auto issue = [&](int c, uint32_t m, uint32_t sl) {
      if (c < nch) {
        const int e = lane & 15;
        const uint32_t me = __shfl_sync(0xffffffffu, m, e), se = __shfl_sync(0xffffffffu, sl, e);
        if (me) {
          const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 3072u;
          const float4* rec = reinterpret_cast<const float4*>(bp.bg_slot + se);
          const float4* pjm = reinterpret_cast<const float4*>(bp.pj) + (kPjFloats / 4) * static_cast<size_t>(se);
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            const int j = (lane >> 4) + 2 * t;   // float4 j of the entry: 0..2 record, 3..11 pose matrix
            if (j < 3) cp_async16_to(buf + 48u * e + 16u * j, rec + j);
            else cp_async16_to(buf + 768u + 144u * e + 16u * (j - 3), pjm + (j - 3));
          }
          if (lane < 16) sts_s32(sb + 6144u + static_cast<uint32_t>(c & 1) * 64u + 4u * e, static_cast<int32_t>(se));
        }
      }
      cp_async_commit();
    };
    uint32_t m0, s0, m1, s1;
    fetch(0, m0, s0);
    fetch(1, m1, s1);
    issue(0, m0, s0);
    for (int c = 0; c < nch; ++c) {
      issue(c + 1, m1, s1);
      uint32_t m2, s2;
      fetch(c + 2, m2, s2);
      cp_async_wait_1();   // chunk c has landed (chunk c + 1 may still be in flight)
      __syncwarp();
      const int lo = max(0, E - kC * (c + 1));
      const uint32_t buf = sb + static_cast<uint32_t>(c & 1) * 3072u, idb = sb + 6144u + static_cast<uint32_t>(c & 1) * 64u;
      uint32_t bits = (E - kC * c - lo) >= 32 ? 0xffffffffu : ((1u << (E - kC * c - lo)) - 1u);
      float2 pa = make_float2(0.f, 0.f), pb2 = make_float2(0.f, 0.f), pc2 = make_float2(0.f, 0.f);
      while (bits) {
        const int k = 31 - __clz(bits);
        bits &= ~(1u << k);
        const int li = lo + k;
        const BlendG g = lds_blend(buf + 48u * k);
        const float dx = __fadd_rn(px, -g.mx);
        const float2 dy = __fadd2_rn(py, make_float2(-g.my, -g.my));
        const float2 rho = pair_rho2(dx, dy, g);
        const bool skip_a = li >= last_a || rho.x > g.rho_hi, skip_b = li >= last_b || rho.y > g.rho_hi;
        if (skip_a && skip_b) continue;   // per-lane (a warp-uniform walk measured 1.5 us slower here)
        const bool fast_a = rho.x < g.rho_fast, fast_b = rho.y < g.rho_fast;
        float2 gv = make_float2(exp_neg_half_fast(rho.x), exp_neg_half_fast(rho.y));
        float2 al = __fmul2_rn(make_float2(g.sigma, g.sigma), gv);
        bool ca = !skip_a && fast_a, cb = !skip_b && fast_b;
        // al = the pixel's alpha (0 where it does not take the entry: T, S unchanged), ga = the alpha the
        // gradient flows through (0 also where the alpha is clamped, rasterizer.cpp:451): no selects after
        al = make_float2(ca ? al.x : 0.0f, cb ? al.y : 0.0f);
        float2 ga = al;
        if (!skip_a && !fast_a) {
          const GuardOut o = guard_decide(px, py.x, g, bp.gg_slot + lds_s32(idb + 4u * k), &kc);
          ca = o.alpha >= 0.0f;
          al.x = ca ? o.alpha : 0.0f;
          ga.x = ca && !o.clamped ? o.alpha : 0.0f;
        }
        if (!skip_b && !fast_b) {
          const GuardOut o = guard_decide(px, py.y, g, bp.gg_slot + lds_s32(idb + 4u * k), &kc);
          cb = o.alpha >= 0.0f;
          al.y = cb ? o.alpha : 0.0f;
          ga.y = cb && !o.clamped ? o.alpha : 0.0f;
        }
        if (!ca && !cb) continue;
        const float2 am = al;
        const float2 inv = make_float2(rcp_approx(1.0f - am.x), rcp_approx(1.0f - am.y));
        const float2 Tpre = __fmul2_rn(T, inv);
        float2 q = __fmul2_rn(gc0, make_float2(g.r, g.r));
        q = __ffma2_rn(gc1, make_float2(g.g, g.g), q);
        q = __ffma2_rn(gc2, make_float2(g.b, g.b), q);
        q = __ffma2_rn(gad, make_float2(g.depth, g.depth), q);
        const float2 dal = __ffma2_rn(Tpre, q, __fmul2_rn(make_float2(-S.x, -S.y), inv));
        const float2 w = __fmul2_rn(am, Tpre);
        S = __ffma2_rn(w, q, S);
        T = Tpre;   // a pixel that does not take the entry has am = 0: rcp(1) = 1 exactly, T unchanged
        const float2 gdg = __fmul2_rn(ga, dal);
        // the pose matrix takes t = g (dx, dy, dx^2, dx dy, dy^2) (compute_posejac's offset basis);
        // both pixels share dx, so the pair sums need no per-pixel ux, uy
        const float G = gdg.x + gdg.y;
        const float2 gy = __fmul2_rn(gdg, dy), gy2 = __fmul2_rn(gy, dy);
        const float2 s5 = __fmul2_rn(w, gad);
        const float f1 = gy.x + gy.y;
        const float f0 = dx * G, f2 = (dx * dx) * G, f3 = dx * f1, f4 = gy2.x + gy2.y, f5 = s5.x + s5.y;
        const uint32_t M = buf + 768u + 144u * k;
#define GSF_COL(F4A, F4B, F4C, SV)                   \
        {                                            \
          const float2 sv = make_float2(SV, SV);     \
          pa = __ffma2_rn(sv, F4A, pa);              \
          pb2 = __ffma2_rn(sv, F4B, pb2);            \
          pc2 = __ffma2_rn(sv, F4C, pc2);            \
        }
        const float4 m0 = lds_f4(M), m1 = lds_f4(M + 16), m2 = lds_f4(M + 32), m3 = lds_f4(M + 48), m4 = lds_f4(M + 64),
                     m5 = lds_f4(M + 80), m6 = lds_f4(M + 96), m7 = lds_f4(M + 112), m8 = lds_f4(M + 128);
        GSF_COL(make_float2(m0.x, m0.y), make_float2(m0.z, m0.w), make_float2(m1.x, m1.y), f0)
        GSF_COL(make_float2(m1.z, m1.w), make_float2(m2.x, m2.y), make_float2(m2.z, m2.w), f1)
        GSF_COL(make_float2(m3.x, m3.y), make_float2(m3.z, m3.w), make_float2(m4.x, m4.y), f2)
        GSF_COL(make_float2(m4.z, m4.w), make_float2(m5.x, m5.y), make_float2(m5.z, m5.w), f3)
        GSF_COL(make_float2(m6.x, m6.y), make_float2(m6.z, m6.w), make_float2(m7.x, m7.y), f4)
        GSF_COL(make_float2(m7.z, m7.w), make_float2(m8.x, m8.y), make_float2(m8.z, m8.w), f5)
#undef GSF_COL
      }
      pd[0] += pa.x; pd[1] += pa.y; pd[2] += pb2.x; pd[3] += pb2.y; pd[4] += pc2.x; pd[5] += pc2.y;
      __syncwarp();   // buffer c & 1 is refilled by issue(c + 2)
      m0 = m1; s0 = s1; m1 = m2; s1 = s2;
    }
    cp_async_wait_all();
  }
#pragma unroll
  for (int a = 0; a < 6; ++a) pd[a] = warp_sum_f64(pd[a]);
  if (lane == 0)
#pragma unroll
    for (int a = 0; a < 6; ++a) bp.tile_pose[static_cast<size_t>(item) * 6 + a] = pd[a];
  double tot[6];
  if (warp_grid_reduce<6>(bp.tile_pose, bp.tile_pose + static_cast<size_t>(rows) * 6, rows, gtickets,
                          gtickets + (rows + 31) / 32, tot, lane == 0, item) && lane == 0) {
#pragma unroll
    for (int a = 0; a < 6; ++a) ds->d_pose[a] = ds->halt ? 0.0 : tot[a];
    // the iteration's pose step (k_track_update) in the same CTA: one kernel boundary less
    if (upd_iter >= 0) track_update(ds, upd_iter, bc1, bc2);
  }
}

// k_backward_q's four quadrant slots of every (tile, primitive) pair folded in quadrant order into the
// pair's [10] partial (the layout k_chain gathers): one thread per pair slot, the slots of consecutive
// threads contiguous, flags of the slots no quadrant wrote mask stale values and are cleared.
__global__ void __launch_bounds__(256) k_pair_combine(const float* __restrict__ qpart, uint32_t* __restrict__ qflag,
                                                      float* __restrict__ partials, const uint32_t* counters) {
  // a warp folds 32 consecutive pairs: their 32 x 160 B of slots are read coalesced (lane-contiguous
  // 16 B pieces) into shared memory, each lane folds its own pair from there, and the 32 x 40 B of
  // results leave through the same buffer as contiguous 16 B stores (per-lane 160 B / 40 B strides
  // left the LSU queue throttled: ncu lg_throttle)
  __shared__ float4 s_q[8][32 * 10];
  pdl_wait();
  pdl_trigger();
  const uint32_t M = counters[kCntPairAlloc];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* sq = s_q[warp];
  for (uint32_t base = (blockIdx.x * 8u + warp) * 32u; base < M; base += gridDim.x * 8u * 32u) {
    const int np = static_cast<int>(min(32u, M - base));
    const float4* src = reinterpret_cast<const float4*>(qpart) + static_cast<size_t>(base) * 10;
#pragma unroll
    for (int h = 0; h < 10; ++h) {
      const int i = h * 32 + lane;
      if (i < np * 10) sq[i] = __ldcs(src + i);   // read once: streaming
    }
    uint32_t fl = 0u;
    if (lane < np) {
      fl = qflag[base + lane];
      if (fl) qflag[base + lane] = 0u;
    }
    __syncwarp();
    float t[10];
#pragma unroll
    for (int f = 0; f < 10; ++f) t[f] = 0.0f;
    if (lane < np) {
      float4 v[10];
#pragma unroll
      for (int h = 0; h < 10; ++h) v[h] = sq[lane * 10 + h];
      // all four slots are read; the unwritten ones are masked by their flag
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        if (!((fl >> (8 * qd)) & 1u)) continue;
        const float* q = reinterpret_cast<const float*>(v) + qd * 10;
#pragma unroll
        for (int f = 0; f < 10; ++f) t[f] += q[f];
      }
    }
    __syncwarp();
    float* so = reinterpret_cast<float*>(sq);
    if (lane < np)
#pragma unroll
      for (int h = 0; h < 5; ++h) reinterpret_cast<float2*>(so + lane * 10)[h] = make_float2(t[2 * h], t[2 * h + 1]);
    __syncwarp();
    float4* dst = reinterpret_cast<float4*>(partials + static_cast<size_t>(base) * 10);
    for (int i = lane; i < np * 10 / 4; i += 32) dst[i] = sq[i];
    if (lane == 0 && (np * 10) % 4)   // a tail pair count leaves two floats
      reinterpret_cast<float2*>(partials + static_cast<size_t>(base) * 10)[np * 5 - 1] =
          reinterpret_cast<const float2*>(so)[np * 5 - 1];
    __syncwarp();
  }
}

// The chain ADDS each primitive's bundle into the gradient buffer (GradientBundle::add,
// output.cpp:36-48): callers zero it once, and a sliding_ba window sums its keyframes' bundles in
// window order (tracker.cpp:164) before the single optimizer step.  One thread owns a primitive's
// entries, so the read-modify-write is race-free and the order is fixed.
__device__ __forceinline__ void acc_grad(float* __restrict__ g, int64_t i, double v) {
  g[i] = static_cast<float>(static_cast<double>(g[i]) + v);
}

// SH basis gradients (sh.cpp:44-72), fp64.
__device__ void sh_basis_grad(int degree, double x, double y, double z, double* g /*16*3*/) {
  const double C1 = 0.4886025119029199;
  for (int i = 0; i < 48; ++i) g[i] = 0.0;
  if (degree < 1) return;
  g[3 * 1 + 1] = -C1;
  g[3 * 2 + 2] = C1;
  g[3 * 3 + 0] = -C1;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  const double c20 = 1.0925484305920792, c21 = -1.0925484305920792, c22 = 0.31539156525252005, c23 = -1.0925484305920792,
               c24 = 0.5462742152960396;
  g[12] = c20 * y; g[13] = c20 * x; g[14] = 0.0;
  g[15] = 0.0; g[16] = c21 * z; g[17] = c21 * y;
  g[18] = c22 * (-2.0 * x); g[19] = c22 * (-2.0 * y); g[20] = c22 * (4.0 * z);
  g[21] = c23 * z; g[22] = 0.0; g[23] = c23 * x;
  g[24] = c24 * (2.0 * x); g[25] = c24 * (-2.0 * y); g[26] = 0.0;
  if (degree < 3) return;
  const double c30 = -0.5900435899266435, c31 = 2.890611442640554, c32 = -0.4570457994644658, c33 = 0.3731763325901154,
               c34 = -0.4570457994644658, c35 = 1.445305721320277, c36 = -0.5900435899266435;
  g[27] = c30 * (6.0 * x * y); g[28] = c30 * (3.0 * xx - 3.0 * yy); g[29] = 0.0;
  g[30] = c31 * (y * z); g[31] = c31 * (x * z); g[32] = c31 * (x * y);
  g[33] = c32 * (-2.0 * x * y); g[34] = c32 * (4.0 * zz - xx - 3.0 * yy); g[35] = c32 * (8.0 * y * z);
  g[36] = c33 * (-6.0 * x * z); g[37] = c33 * (-6.0 * y * z); g[38] = c33 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
  g[39] = c34 * (4.0 * zz - 3.0 * xx - yy); g[40] = c34 * (-2.0 * x * y); g[41] = c34 * (8.0 * x * z);
  g[42] = c35 * (2.0 * x * z); g[43] = c35 * (-2.0 * y * z); g[44] = c35 * (xx - yy);
  g[45] = c36 * (3.0 * xx - 3.0 * yy); g[46] = c36 * (-6.0 * x * y); g[47] = 0.0;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// eval_sh_color_backward (sh.cpp:88-108) along the view direction for sh_coeffs > 1, fp64:
// writes d sh into grads (if non-null) and returns d mean through the view direction.
static __device__ __noinline__ void sh_backward(const float* __restrict__ params, int64_t P, int64_t id, int K,
                                                const Cam& cam, double m0, double m1, double m2, const double* dcol,
                                                float* __restrict__ grads, double* through) {
  const double d0 = m0 - cam.center[0], d1 = m1 - cam.center[1], d2 = m2 - cam.center[2];
  const double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  double dir[3] = {0.0, 0.0, 1.0};
  if (len > 1e-12) { dir[0] = d0 / len; dir[1] = d1 / len; dir[2] = d2 / len; }
  const int deg = sh_degree(K);
  double b[16];
  sh_basis(deg, dir[0], dir[1], dir[2], b);
  double masked[3];
  for (int c = 0; c < 3; ++c) {
    double raw = 0.5;
    for (int k = 0; k < K; ++k) raw += b[k] * params[(11 + 3 * k + c) * P + id];
    masked[c] = raw < 0.0 ? 0.0 : dcol[c];
  }
  if (grads)
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < 3; ++c) acc_grad(grads, (11 + 3 * k + c) * P + id, b[k] * masked[c]);
  through[0] = through[1] = through[2] = 0.0;
  if (deg >= 1 && len > 1e-12) {
    double gb[48];
    sh_basis_grad(deg, dir[0], dir[1], dir[2], gb);
    double dd[3] = {0.0, 0.0, 0.0};
    for (int k = 1; k < K; ++k) {
      const double md = masked[0] * params[(11 + 3 * k + 0) * P + id] + masked[1] * params[(11 + 3 * k + 1) * P + id] +
                        masked[2] * params[(11 + 3 * k + 2) * P + id];
      for (int a = 0; a < 3; ++a) dd[a] += gb[3 * k + a] * md;
    }
    const double dot = dir[0] * dd[0] + dir[1] * dd[1] + dir[2] * dd[2];
    for (int a = 0; a < 3; ++a) through[a] = (dd[a] - dir[a] * dot) / len;
  }
}

#ifndef GSF_CHAIN_COOP
#define GSF_CHAIN_COOP 16
#endif
constexpr int kChainCoop = GSF_CHAIN_COOP;

// The large-footprint primitives (k_preprocess's big list: more than kBigPairs tiles, up to a few
// thousand pair slots each) summed before k_chain, one CTA per primitive: coalesced lane-strided
// reads of the primitive's contiguous [pair][10] slots, per-thread fp64 sums, a fixed-order CTA
// tree, and the ten fp64 totals written over the primitive's first two slots (80 B), which
// k_chain reads instead of gathering.  In k_chain one warp walked such a list alone while the rest
// of the grid had finished (the kernel's tail: SMs active ~40 % of its duration under ncu).
#ifndef GSF_BIGSUM_THREADS
#define GSF_BIGSUM_THREADS 256
#endif
constexpr int kBigSumThreads = GSF_BIGSUM_THREADS;
__global__ void __launch_bounds__(kBigSumThreads) k_big_sum(const uint32_t* __restrict__ big_ids, const uint32_t* counters,
                                                            const int4* __restrict__ rect_id,
                                                            const uint32_t* __restrict__ pair_base, float* partials) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_w[kBigSumThreads / 32][10];
  const uint32_t nbig = counters[kCntBig];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
    const uint32_t id = big_ids[b];
    const int4 q = rect_id[id];
    const int c = (q.y - q.x + 1) * (q.w - q.z + 1);
    float* pp = partials + static_cast<size_t>(pair_base[id]) * 10;
    double acc[10];
#pragma unroll
    for (int f = 0; f < 10; ++f) acc[f] = 0.0;
    for (int k0 = threadIdx.x; k0 < c; k0 += 2 * kBigSumThreads) {
      float2 v[2][5];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u * kBigSumThreads;
#pragma unroll
        for (int f = 0; f < 5; ++f)
          v[u][f] = k < c ? __ldg(reinterpret_cast<const float2*>(pp + static_cast<size_t>(k) * 10) + f) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int f = 0; f < 5; ++f) {
          acc[2 * f] += static_cast<double>(v[u][f].x);
          acc[2 * f + 1] += static_cast<double>(v[u][f].y);
        }
    }
#pragma unroll
    for (int f = 0; f < 10; ++f) {
      const double t = warp_sum_d(acc[f]);
      if (lane == 0) s_w[warp][f] = t;
    }
    __syncthreads();   // every read of the slots is done before they are overwritten
    if (threadIdx.x < 10) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kBigSumThreads / 32; ++w) t += s_w[w][threadIdx.x];
      reinterpret_cast<double*>(pp)[threadIdx.x] = t;
    }
    __syncthreads();
  }
}

template <int NF, bool FULL>
#ifndef GSF_CHAIN_MINB
#define GSF_CHAIN_MINB 2
#endif
__global__ void __launch_bounds__(256, GSF_CHAIN_MINB) k_chain(const uint32_t* __restrict__ vis_list, const uint32_t* counters,
                                               const int4* __restrict__ rect_id, const uint32_t* __restrict__ pair_base,
                                               const float* __restrict__ partials, const DevState* ds,
                                               const float* __restrict__ params, int64_t P, int K,
                                               float* __restrict__ grads, float* __restrict__ d_mean2d,
                                               double* __restrict__ pose_part, const BlendG* __restrict__ bg,
                                               double iso_w, double iso_eps) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  __shared__ double s_red[8][6];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double pose[6] = {0, 0, 0, 0, 0, 0};
  const uint32_t V = counters[kCntVisible];
  // CTAs past the visible list have no primitive and no pose row (k_pose_sum reads the rows of
  // the first min(grid, ceil(V / 256)) CTAs only)
  if (blockIdx.x * blockDim.x >= V) return;
  float pf_par[14];
#define GSF_PAR(F) pf_par[F]
  float gpre[16];
#define GSF_ACC(ARR, F, IDX, V)                                                      \
  {                                                                                  \
    const float nv_ = static_cast<float>(static_cast<double>(gpre[F]) + (V));        \
    gpre[F] = nv_;                                                                   \
    ARR[IDX] = nv_;                                                                  \
  }
  const bool halted = ds->halt != 0;
  // CTA-strided over the visible list (a grid of the resident CTAs, not one CTA per 256 of P: the
  // thousands of empty CTAs past V cost dispatch time); each CTA keeps one pose row
  for (uint32_t rb = blockIdx.x * blockDim.x; rb < V; rb += gridDim.x * blockDim.x) {
  const uint32_t r = rb + tid;
  bool active = r < V;   // halted: the slots are still read, no gradient is written
  int64_t id = 0;
  int c = 0;
  const float* pp = partials;
  if (active) {
    id = vis_list[r];
    // the primitive's parameters, loaded before the pair gather so their latency overlaps it
#pragma unroll
    for (int f = 0; f < 14; ++f) pf_par[f] = (f < 11 || K == 1) ? params[f * P + id] : 0.0f;
    // ... and its accumulated gradients: the read-modify-writes below then need no load each (a load
    // after a store into the same array cannot be hoisted by the compiler: 14 serial round trips)
    if (FULL) {
#pragma unroll
      for (int f = 0; f < 14; ++f) gpre[f] = (f < 11 || K == 1) ? grads[f * P + id] : 0.0f;
      if (d_mean2d) { gpre[14] = d_mean2d[id]; gpre[15] = d_mean2d[P + id]; }
    }
    const int4 q = rect_id[id];
    c = (q.y - q.x + 1) * (q.w - q.z + 1);
    pp = partials + static_cast<size_t>(pair_base[id]) * NF;
  }
  // fixed-order gather of the primitive's pair partials: its slots hold the tiles of its
  // rectangle in row-major order (the reference's tile-order reduction, rasterizer.cpp:466-478).
  // Short lists (<= kChainCoop = 16 pairs) are summed by their own lane; a longer list by the
  // whole warp (lane-strided, then a fixed shuffle tree) so one huge footprint cannot leave a
  // single thread walking thousands of L2 round trips.
  double sg[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) sg[f] = 0.0;
  // c > kBigPairs: summed by k_big_sum into the first two slots (fp64)
  const bool presum = c > kBigPairs;
  if (presum) {
#pragma unroll
    for (int f = 0; f < NF; ++f) sg[f] = __ldg(reinterpret_cast<const double*>(pp) + f);
  }
  const bool coop = c > kChainCoop && !presum;
  if (!coop && !presum) {
    // 8-byte vectors (a pair slot is 40 B): 5 loads per pair instead of 10 (chain -8 us per view;
    // two or four pairs' loads in flight measured slower: more registers at the 128 cap)
    static_assert(NF % 2 == 0, "pair slots are read as float2");
    for (int k = 0; k < c; ++k) {
      const float2* v = reinterpret_cast<const float2*>(pp + k * NF);
#pragma unroll
      for (int f = 0; f < NF / 2; ++f) {
        const float2 x = __ldg(v + f);
        sg[2 * f] += static_cast<double>(x.x);
        sg[2 * f + 1] += static_cast<double>(x.y);
      }
    }
  }
  uint32_t big = __ballot_sync(0xffffffffu, coop);
  while (big) {
    const int j = __ffs(big) - 1;
    big &= big - 1u;
    const int cj = __shfl_sync(0xffffffffu, c, j);
    const float* pj = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(pp), j));
    double acc[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f] = 0.0;
#ifndef GSF_COOP_U
#define GSF_COOP_U 4
#endif
    // GSF_COOP_U lane-strided pairs' loads in flight per round, summed in k order: one primitive
    // covering thousands of tiles otherwise leaves its warp walking L2 round trips one at a time
    // (the kernel's tail: ncu saw the SMs active 36 % of its duration)
    constexpr int kCU = GSF_COOP_U;
    for (int k0 = lane; k0 < cj; k0 += 32 * kCU) {
      float2 v[kCU][NF / 2];
#pragma unroll
      for (int u = 0; u < kCU; ++u) {
        const int k = k0 + 32 * u;
#pragma unroll
        for (int f = 0; f < NF / 2; ++f)
          v[u][f] = k < cj ? __ldg(reinterpret_cast<const float2*>(pj + k * NF) + f) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kCU; ++u)
        if (k0 + 32 * u < cj)
#pragma unroll
          for (int f = 0; f < NF / 2; ++f) {
            acc[2 * f] += static_cast<double>(v[u][f].x);
            acc[2 * f + 1] += static_cast<double>(v[u][f].y);
          }
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      double v = acc[f];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == j) sg[f] = v;
    }
  }
  if (halted) active = false;
  if (active && NF == 10) {
    // fields 0..4 arrive in the pixel-offset basis t = g (dx, dy, dx^2, dx dy, dy^2): back to
    // (d_mean2d x, y, d_cov2d 00, 01, 11) with the record's conic (ux, uy = conic rows . (dx, dy))
    const BlendG gr = bg[id];
    const double c00 = gr.c00, c01 = 0.5 * static_cast<double>(gr.c01x2), c11 = gr.c11;
    const double t0 = sg[0], t1 = sg[1], t2 = sg[2], t3 = sg[3], t4 = sg[4];
    sg[0] = c00 * t0 + c01 * t1;
    sg[1] = c01 * t0 + c11 * t1;
    sg[2] = 0.5 * (c00 * c00 * t2 + 2.0 * c00 * c01 * t3 + c01 * c01 * t4);
    sg[3] = 0.5 * (c00 * c01 * t2 + (c00 * c11 + c01 * c01) * t3 + c01 * c11 * t4);
    sg[4] = 0.5 * (c01 * c01 * t2 + 2.0 * c01 * c11 * t3 + c11 * c11 * t4);
  }
  if (active) {
    bool zero = true;
#pragma unroll
    for (int f = 0; f < NF; ++f) zero = zero && sg[f] == 0.0;
    if (!zero) {
      const Cam& cam = ds->cam;
      const double* Wr = cam.W;
      const double m0 = GSF_PAR(0), m1 = GSF_PAR(1), m2 = GSF_PAR(2);
      const double pc[3] = {Wr[0] * m0 + Wr[1] * m1 + Wr[2] * m2 + cam.t[0], Wr[3] * m0 + Wr[4] * m1 + Wr[5] * m2 + cam.t[1],
                            Wr[6] * m0 + Wr[7] * m1 + Wr[8] * m2 + cam.t[2]};
      const double iz = 1.0 / pc[2], iz2 = iz * iz, z = pc[2];
      const double J[2][3] = {{cam.fx * iz, 0.0, -cam.fx * pc[0] * iz2}, {0.0, cam.fy * iz, -cam.fy * pc[1] * iz2}};
      const double qw0 = GSF_PAR(6), qx0 = GSF_PAR(7), qy0 = GSF_PAR(8), qz0 = GSF_PAR(9);
      const double qlen = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
      const double qn[4] = {qw0 / qlen, qx0 / qlen, qy0 / qlen, qz0 / qlen};
      const double w = qn[0], x = qn[1], y = qn[2], zq = qn[3];
      const double R[3][3] = {{1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y)},
                              {2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x)},
                              {2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)}};
      const double s[3] = {exp(static_cast<double>(GSF_PAR(3))), exp(static_cast<double>(GSF_PAR(4))),
                           exp(static_cast<double>(GSF_PAR(5)))};
      double Cw[3][3], Cc[3][3], T1[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          Cw[a][b] = R[a][0] * (s[0] * s[0]) * R[b][0] + R[a][1] * (s[1] * s[1]) * R[b][1] + R[a][2] * (s[2] * s[2]) * R[b][2];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) T1[a][b] = Wr[3 * a + 0] * Cw[0][b] + Wr[3 * a + 1] * Cw[1][b] + Wr[3 * a + 2] * Cw[2][b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Cc[a][b] = T1[a][0] * Wr[3 * b + 0] + T1[a][1] * Wr[3 * b + 1] + T1[a][2] * Wr[3 * b + 2];
      const double dC[2][2] = {{sg[2], sg[3]}, {sg[3], sg[4]}};
      // d_cov_cam = J^T dC J ; d_jac = 2 dC J Cc   (rasterizer.cpp:503-504)
      double dCc[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          const double t0 = J[0][a] * dC[0][0] + J[1][a] * dC[1][0];
          const double t1 = J[0][a] * dC[0][1] + J[1][a] * dC[1][1];
          dCc[a][b] = t0 * J[0][b] + t1 * J[1][b];
        }
      double dJ[2][3];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) {
          double acc = 0.0;
          for (int c = 0; c < 3; ++c) acc += (2.0 * dC[a][0] * J[0][c] + 2.0 * dC[a][1] * J[1][c]) * Cc[c][b];
          dJ[a][b] = acc;
        }
      const double iz3 = iz2 / z;
      double dp[3] = {0.0, 0.0, 0.0};
      dp[0] += dJ[0][2] * (-cam.fx * iz2);
      dp[1] += dJ[1][2] * (-cam.fy * iz2);
      dp[2] += dJ[0][0] * (-cam.fx * iz2) + dJ[1][1] * (-cam.fy * iz2) + dJ[0][2] * (2.0 * cam.fx * pc[0] * iz3) +
               dJ[1][2] * (2.0 * cam.fy * pc[1] * iz3);
      for (int a = 0; a < 3; ++a) dp[a] += J[0][a] * sg[0] + J[1][a] * sg[1];
      dp[2] += sg[5];
      // pose (rasterizer.cpp:519-526): this primitive's part, added to the thread's row below
      double pz[6];
      pz[0] = pc[1] * dp[2] - pc[2] * dp[1];
      pz[1] = pc[2] * dp[0] - pc[0] * dp[2];
      pz[2] = pc[0] * dp[1] - pc[1] * dp[0];
      pz[3] = dp[0];
      pz[4] = dp[1];
      pz[5] = dp[2];
      for (int j = 0; j < 3; ++j) {
        // E = skew(unit_j); sum dCc .* (E Cc - Cc E)
        double E[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (j == 0) { E[1][2] = -1.0; E[2][1] = 1.0; }
        if (j == 1) { E[0][2] = 1.0; E[2][0] = -1.0; }
        if (j == 2) { E[0][1] = -1.0; E[1][0] = 1.0; }
        double acc = 0.0;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            double ec = 0.0, ce = 0.0;
            for (int c = 0; c < 3; ++c) { ec += E[a][c] * Cc[c][b]; ce += Cc[a][c] * E[c][b]; }
            acc += dCc[a][b] * (ec - ce);
          }
        pz[j] += acc;
      }
      double through[3] = {0.0, 0.0, 0.0};
      double dcol[3] = {0.0, 0.0, 0.0};
      if (NF >= 9) { dcol[0] = sg[6]; dcol[1] = sg[7]; dcol[2] = sg[8]; }
      if (K == 1 && FULL) {
        // degree 0: colour_c = max(0.5 + C0 sh_c, 0), no view-direction gradient (sh.cpp:88-108)
        for (int c = 0; c < 3; ++c) {
          const double raw = 0.5 + 0.28209479177387814 * GSF_PAR(11 + c);
          GSF_ACC(grads, 11 + c, (11 + c) * P + id, raw < 0.0 ? 0.0 : 0.28209479177387814 * dcol[c]);
        }
      } else if (K > 1) {
        sh_backward(params, P, id, K, cam, m0, m1, m2, dcol, FULL ? grads : nullptr, through);
        for (int a = 0; a < 3; ++a) pz[3 + a] += Wr[3 * a + 0] * through[0] + Wr[3 * a + 1] * through[1] + Wr[3 * a + 2] * through[2];
      }
#pragma unroll
      for (int a = 0; a < 6; ++a) pose[a] += pz[a];
      if (FULL) {
        if (d_mean2d) { GSF_ACC(d_mean2d, 14, id, sg[0]); GSF_ACC(d_mean2d, 15, P + id, sg[1]); }
        // world parameters (rasterizer.cpp:528-546)
        for (int a = 0; a < 3; ++a) {
          const double dm = Wr[0 * 3 + a] * dp[0] + Wr[1 * 3 + a] * dp[1] + Wr[2 * 3 + a] * dp[2] + through[a];
          GSF_ACC(grads, a, a * P + id, dm);
        }
        double dCw[3][3], T2[3][3];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) T2[a][b] = Wr[0 * 3 + a] * dCc[0][b] + Wr[1 * 3 + a] * dCc[1][b] + Wr[2 * 3 + a] * dCc[2][b];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) dCw[a][b] = T2[a][0] * Wr[0 * 3 + b] + T2[a][1] * Wr[1 * 3 + b] + T2[a][2] * Wr[2 * 3 + b];
        double dM[3][3];  // 2 dCw (R diag(s))
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            dM[a][b] = 2.0 * (dCw[a][0] * R[0][b] * s[b] + dCw[a][1] * R[1][b] * s[b] + dCw[a][2] * R[2][b] * s[b]);
        for (int a = 0; a < 3; ++a) {
          const double ds_ = R[0][a] * dM[0][a] + R[1][a] * dM[1][a] + R[2][a] * dM[2][a];
          GSF_ACC(grads, 3 + a, (3 + a) * P + id, ds_ * s[a]);
        }
        double dR[3][3];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) dR[a][b] = dM[a][b] * s[b];
        // rotation_quat_jacobians (rasterizer.cpp:320-335)
        const double jq[4][9] = {{0, -zq, y, zq, 0, -x, -y, x, 0},
                                 {0, y, zq, y, -2 * x, -w, zq, w, -2 * x},
                                 {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y},
                                 {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0}};
        double dqn[4];
        for (int kq = 0; kq < 4; ++kq) {
          double acc = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) acc += dR[a][b] * (2.0 * jq[kq][3 * a + b]);
          dqn[kq] = acc;
        }
        const double qd = qn[0] * dqn[0] + qn[1] * dqn[1] + qn[2] * dqn[2] + qn[3] * dqn[3];
        for (int a = 0; a < 4; ++a) GSF_ACC(grads, 6 + a, (6 + a) * P + id, (dqn[a] - qn[a] * qd) / qlen);
        const double sig = 1.0 / (1.0 + exp(-static_cast<double>(GSF_PAR(10))));
        GSF_ACC(grads, 10, 10 * P + id, (NF >= 10 ? sg[9] : 0.0) * sig * (1.0 - sig));
      }
    }
  }
  if (active && FULL && iso_w > 0.0) {
    // the iso term's direct log-scale gradient of every visible primitive (losses.cpp:272-280, k_iso's
    // arithmetic), added after the primitive's bundle like the stand-alone pass did
    const double sx[3] = {exp(static_cast<double>(GSF_PAR(3))), exp(static_cast<double>(GSF_PAR(4))),
                          exp(static_cast<double>(GSF_PAR(5)))};
    int a = 0, b = 0;
    for (int c = 1; c < 3; ++c) {
      if (sx[c] > sx[a]) a = c;
      if (sx[c] < sx[b]) b = c;
    }
    const double ratio = sx[a] / sx[b];
    if (ratio > iso_eps) {
      const double g = iso_w * ratio / static_cast<double>(V);
#pragma unroll
      for (int c = 0; c < 3; ++c) {   // static register indices
        if (c == a) GSF_ACC(grads, 3 + c, (3 + c) * P + id, g);
        if (c == b) GSF_ACC(grads, 3 + c, (3 + c) * P + id, -g);
      }
    }
  }
  }
  // deterministic block reduction of the pose pieces
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    const double t = warp_sum_d(pose[a]);
    if (lane == 0) s_red[warp][a] = t;
  }
  __syncthreads();
  if (tid < 6) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_red[w][tid];
    pose_part[static_cast<size_t>(blockIdx.x) * 6 + tid] = t;
  }
}
#undef GSF_PAR
#undef GSF_ACC

__global__ void __launch_bounds__(1024) k_pose_sum(const double* __restrict__ pose_part, int blocks, DevState* ds,
                                                   const uint32_t* counters, PoseSumPost post) {
  pdl_wait();   // PDL: the predecessor's results are complete from here
  pdl_trigger();
  blocks = min(blocks, static_cast<int>((counters[kCntVisible] + 255u) / 256u));   // k_chain's CTAs with a row
  __shared__ double s_red[32][6];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int b = tid; b < blocks; b += blockDim.x)
    for (int a = 0; a < 6; ++a) acc[a] += __ldcg(pose_part + static_cast<size_t>(b) * 6 + a);
  for (int a = 0; a < 6; ++a) {
    const double t = warp_sum_d(acc[a]);
    if (lane == 0) s_red[warp][a] = t;
  }
  __syncthreads();
  if (tid < 6) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += s_red[w][tid];
    t = ds->halt ? 0.0 : t;
    ds->d_pose[tid] = t;
    if (post.grab >= 0) post.kf[post.grab].grad[tid] = t;   // k_kf_grab's copy
  }
  if (tid == 0) {
    if (post.loss_acc) *post.loss_acc += ds->loss_total;
    if (post.trace && post.trace_index >= 0) post.trace[post.trace_index] = ds->loss_total;
    if (post.next >= 0) {   // k_set_cam_from_kf for the next view (every reader of this view's camera ran)
      const Cam old = ds->cam;
      const KfPose& p = post.kf[post.next];
      ds->cam = make_cam(p.rot, p.trans, old.fx, old.fy, old.cx, old.cy, old.width, old.height, old.near_plane,
                         old.far_plane);
      ds->has_obs = 1;
    }
  }
}

template <int SEED>
__global__ void k_seeds_out(int64_t npix, const float* __restrict__ color, const float* __restrict__ ad,
                            const float* __restrict__ md, const uint8_t* __restrict__ mv, const float* __restrict__ op,
                            const float* __restrict__ target, const float* __restrict__ depth, const float* __restrict__ dssim,
                            const DevState* ds, LossParams lp, double near_plane, double far_plane, float* __restrict__ out) {
  const int64_t pi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pi >= npix) return;
  const PixSeeds s = seeds_pixel<SEED>(pi, color, ad[pi], md[pi], mv[pi] != 0, op[pi], target, depth, dssim, ds, lp,
                                       near_plane, far_plane);
  out[3 * pi] = s.gc0;
  out[3 * pi + 1] = s.gc1;
  out[3 * pi + 2] = s.gc2;
  out[3 * npix + pi] = s.gad;
  out[4 * npix + pi] = s.gmd;
  out[5 * npix + pi] = s.gu;
}

}  // namespace

void run_seeds_out(Workspace& ws, DevState* ds, int mode, const float* target, const float* depth, const LossParams& lp,
                   int W, int H, double near_plane, double far_plane, float* out, cudaStream_t st, int64_t* L) {
  const int64_t npix = static_cast<int64_t>(W) * H;
  const float* dssim = (mode == 2 && lp.w_ssim > 0.0) ? ws.dssim : nullptr;
  if (mode == 1)
    k_seeds_out<1><<<div_up(npix, 256), 256, 0, st>>>(npix, ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid,
                                                       ws.opacity, target, depth, dssim, ds, lp, near_plane, far_plane, out);
  else
    k_seeds_out<2><<<div_up(npix, 256), 256, 0, st>>>(npix, ws.color, ws.alpha_depth, ws.median_depth, ws.median_valid,
                                                       ws.opacity, target, depth, dssim, ds, lp, near_plane, far_plane, out);
  ++*L;
}

bool run_backward(Workspace& ws, DevState* ds, const BwdArgs& a, cudaStream_t st, int64_t* L) {
  const int ntiles = a.rp.tiles_x * a.rp.tiles_y;
  BwdPtrs bp;
  bp.ranges = ws.ranges;
  bp.sid = ws.sid;
  bp.bg = ws.bg_id;
  bp.gg = ws.gg_id;
  bp.color = ws.color;
  bp.alpha_depth = ws.alpha_depth;
  bp.median_depth = ws.median_depth;
  bp.median_valid = ws.median_valid;
  bp.opacity = ws.opacity;
  bp.final_T = ws.final_T;
  bp.last = ws.last;
  bp.median_prim = ws.median_prim;
  bp.obs = a.obs;
  bp.target = a.target_rgb;
  bp.up_color = a.up_color;
  bp.up_adepth = a.up_adepth;
  bp.up_mdepth = a.up_mdepth;
  bp.up_opacity = a.up_opacity;
  bp.up_uncert = a.up_uncert;
  bp.dssim = (a.seed_mode == SEED_MAP && a.lp.w_ssim > 0.0) ? ws.dssim : nullptr;
  bp.partials = ws.partials;
  bp.qflag = reinterpret_cast<uint8_t*>(ws.qflag);
  bp.qpart = ws.qpart;
  bp.pj = nullptr;
  bp.pj_slot = nullptr;
  bp.rect = ws.rect_id;
  bp.pair_base = ws.pair_base;
  bp.tile_pose = nullptr;
  bp.qlist = ws.qlist;
  bp.lastc = ws.lastc;
  bp.pxcode = ws.pxcode;
  bp.bg_slot = ws.bg_slot;
  bp.gg_slot = ws.gg_slot;
  const bool view_dep = a.K > 1;
  const int nf = a.pose_only ? (view_dep ? 9 : 6) : 10;
  if (a.pose_only && a.fused_pose) {
    // tracking: per-tile pose partials through the per-primitive Jacobians; the last CTA reduces
    // them, so neither a chain nor a pose-sum launch follows
    bp.pj = ws.pj_id;
    bp.pj_slot = ws.pj_slot;
    bp.tile_pose = ws.pose_part;
    uint32_t* ticket = ws.bin_counters + kCntBwdTicket;
    bool fused_update = false;
    if (ws.prof) ws.prof->begin(PROF_BACKWARD, st);
#define GSF_BWDP(SM, VD)                                                                                        \
  do {                                                                                                          \
    static bool attr_set = false;                                                                               \
    if (!attr_set) {                                                                                            \
      GSF_CUDA_CHECK(cudaFuncSetAttribute(k_backward_pose<SM, VD>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          static_cast<int>(pose_smem_bytes<VD>())));                          \
      attr_set = true;                                                                                          \
    }                                                                                                           \
    k_backward_pose<SM, VD><<<ntiles, 256, pose_smem_bytes<VD>(), st>>>(bp, a.W, a.H, a.rp.tiles_x, a.kc,      \
                                                                       a.near_plane, a.far_plane, a.lp, ds, ticket); \
  } while (0)
    if (a.seed_mode == SEED_TRACK && nf == 6) {
      const double t = static_cast<double>(a.update_iter + 1);   // AdamState bias corrections (adam.cpp:40-53)
      launch_pdl(k_backward_track_w, dim3(4 * ntiles), dim3(32), 0, st, bp, a.W, a.H, a.rp.tiles_x, a.kc, a.near_plane, a.far_plane, a.lp, ds,
                                                     ws.wtickets + ws.wtickets_half, 4 * ntiles, a.update_iter,
                                                     1.0 - std::pow(0.9, t), 1.0 - std::pow(0.999, t), a.order,
                                                     static_cast<int64_t>(ws.tiles_cap));
      fused_update = a.update_iter >= 0;
    } else if (a.seed_mode == SEED_TRACK) {
      GSF_BWDP(SEED_TRACK, true);
    } else {
      if (nf == 6) GSF_BWDP(SEED_EXPLICIT, false); else GSF_BWDP(SEED_EXPLICIT, true);
    }
#undef GSF_BWDP
    ++*L;
    if (ws.prof) ws.prof->end(st);
    return fused_update;
  }
  if (ws.prof) ws.prof->begin(PROF_BACKWARD, st);
  // the full bundle (a pose-only backward always takes the fused path above): per-quadrant
  // single-warp CTAs (k_backward_q), then the quadrant slots folded per pair
  if (nf != 10) throw std::logic_error("render_backward: a pose-only backward needs the fused pose path");
  {
#define GSF_BQ(SM) launch_pdl(k_backward_q<SM>, dim3(4 * ntiles), dim3(32), 0, st, bp, a.W, a.H, a.rp.tiles_x, a.kc, \
                              a.near_plane, a.far_plane, a.lp, static_cast<const DevState*>(ds), a.order,           \
                              static_cast<int64_t>(ws.tiles_cap))
    if (a.seed_mode == SEED_TRACK) GSF_BQ(SEED_TRACK);
    else if (a.seed_mode == SEED_MAP) GSF_BQ(SEED_MAP);
    else GSF_BQ(SEED_EXPLICIT);
#undef GSF_BQ
    ++*L;
    launch_pdl(k_pair_combine, dim3(4 * 148), dim3(256), 0, st, static_cast<const float*>(ws.qpart), ws.qflag, ws.partials,
               static_cast<const uint32_t*>(ws.bin_counters));
  }
  ++*L;
  if (ws.prof) ws.prof->end(st);
  if (ws.prof) ws.prof->begin(PROF_CHAIN, st);
  launch_pdl(k_big_sum, dim3(2 * 148), dim3(kBigSumThreads), 0, st, static_cast<const uint32_t*>(ws.big_ids),
             static_cast<const uint32_t*>(ws.bin_counters), static_cast<const int4*>(ws.rect_id),
             static_cast<const uint32_t*>(ws.pair_base), ws.partials);
  ++*L;
#ifndef GSF_CHAIN_CTAS
#define GSF_CHAIN_CTAS (4 * 148)
#endif
  const int blocks = std::max(1, std::min(div_up(a.P, 256), GSF_CHAIN_CTAS));
  launch_pdl(k_chain<10, true>, dim3(blocks), dim3(256), 0, st, ws.vis_list, ws.bin_counters, ws.rect_id, ws.pair_base,
             ws.partials, ds, a.params, a.P, a.K, a.grads, a.d_mean2d, ws.pose_part, ws.bg_id, a.iso_w, a.iso_eps);
  ++*L;
  launch_pdl(k_pose_sum, dim3(1), dim3(1024), 0, st, ws.pose_part, blocks, ds, static_cast<const uint32_t*>(ws.bin_counters),
             a.post);
  ++*L;
  if (ws.prof) ws.prof->end(st);
  return false;
}

}  // namespace gsfk
