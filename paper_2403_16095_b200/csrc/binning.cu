// binning.cu — per-tile lists of the visible primitives in exact (depth, id) order.
//
// The reference sorts the visible ids globally by (fp64 depth, id) (sorted_visible,
// rasterizer.cpp:69-79) and appends each one to every tile its footprint rectangle overlaps
// (rasterizer.cpp:193-212), so every tile list is in global depth order.  Only the per-tile
// order is observable, so the device bins first and sorts each tile's (short) list:
//
//   k_preprocess    (raster_fwd.cu) scatters every (tile, primitive) pair into its tile's bucket
//                   with one atomic on the tile's fill counter (one counter per L2 sector); a warp
//                   flattens the pairs of its 32 primitives over its lanes, and lists the few
//                   primitives with more than kBigPairs tiles instead, so a primitive covering a
//                   thousand tiles does not serialise one warp (order inside a bucket is arbitrary)
//   k_tile_sort     one CTA per tile: appends the listed large primitives covering the tile to its
//                   bucket, takes its list start from a single-pass decoupled look-back scan
//                   of the tile counts (pair total M, longest list; a bucket overflow makes the
//                   host grow the buckets and re-run), 32-key runs sorted in registers (warp bitonic), then
//                   pairwise run merges by rank (binary search in the partner run) in shared
//                   memory; lists longer than kSortChunk are chunk-sorted and merged (merge path)
//                   through global memory by the same CTA.  A final pass re-orders the rare runs
//                   whose fp32 depths tie by the exact fp64 depth (then id).  In the tracking loop
//                   and the mapping forward the lists are read back only through `ranges`, so each
//                   tile takes its start from one atomic (any_order: no look-back; the last CTA to
//                   place its list records M and re-zeroes the counters; 128-thread CTAs for the
//                   tracking loop's short lists): -4 us per tracking iteration, -1 us per view.  Measured and dropped: the sort fused
//                   into the tracking blend (+20 us: the CTA-serial sort phases stretch every
//                   blend CTA), one warp per tile with register bitonic sorts (+25 us: 3 k
//                   warps leave the SMs 21 % occupied and each warp's 36-stage shuffle chain is
//                   latency-bound), unrolled loads of the large-primitive list (+3 us).
//
// Sort key: (fp32 bits of the depth) << 32 | id, one 64-bit integer.  Positive floats order like
// their bit patterns and fp32 rounding is monotone, so this is the reference order except inside
// runs of equal fp32 depth, which the fix-up resolves with the fp64 depth.  Keys are unique (id),
// so the result does not depend on the scatter order: deterministic.
#include "kernels.h"
#include "tilesort.cuh"

namespace gsfk {

namespace {

// Exclusive start of tile t's compacted list: a single-pass scan over the tile counts with
// decoupled look-back (warp 0).  Tile t publishes its count (flag 1) as soon as it starts and its
// inclusive prefix (flag 2) once known, in one 64-bit word next to its fill counter (same L2
// sector, zeroed by the per-render memset); it sums its predecessors' words back to the nearest
// published prefix.  Tiles are claimed in order from an atomic ticket (not blockIdx), so every
// tile a CTA waits on already belongs to a running CTA, whatever order the CTAs are dispatched in.
__device__ constexpr unsigned long long kScanAgg = 1ull << 32, kScanPrefix = 2ull << 32;
__device__ __forceinline__ unsigned long long* scan_word(uint32_t* fill, int64_t t) {
  return reinterpret_cast<unsigned long long*>(fill + t * kBinStride + 2);
}
__device__ __forceinline__ void tile_count_publish(uint32_t* fill, int t, uint32_t n) {
  atomicExch(scan_word(fill, t), (t == 0 ? kScanPrefix : kScanAgg) | n);
}
__device__ uint32_t tile_list_start(uint32_t* fill, int t, uint32_t n) {   // warp 0, after tile_count_publish
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  for (int j = t - 1; j >= 0; j -= 32) {
    const int idx = j - lane;
    unsigned long long v;
    do {
      v = idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(scan_word(fill, idx)) : kScanPrefix;
    } while (__any_sync(0xffffffffu, (v >> 32) == 0ull));
    const uint32_t pm = __ballot_sync(0xffffffffu, (v >> 32) == 2ull);
    const int stop = pm ? __ffs(pm) - 1 : 31;   // nearest published prefix
    uint32_t x = lane <= stop ? static_cast<uint32_t>(v) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    excl += x;
    if (pm) break;
  }
  if (lane == 0 && t > 0) atomicExch(scan_word(fill, t), kScanPrefix | (excl + n));
  return excl;
}

__global__ void __launch_bounds__(256) k_tile_sort(uint32_t* fill, uint32_t pair_cap, unsigned long long* bucket,
                                                   uint32_t bucket_cap, unsigned long long* skey, uint32_t* __restrict__ sid,
                                                   const double* __restrict__ depth_id, int2* __restrict__ ranges,
                                                   const uint32_t* __restrict__ pj_slot, uint32_t* __restrict__ sslot,
                                                   DevState* ds, const uint32_t* counters,
                                                   const uint32_t* __restrict__ big_ids, const int4* __restrict__ rect_id,
                                                   int tiles_x, uint32_t* ticket, uint32_t* alloc) {
  __shared__ unsigned long long s_k[2][kSortChunk];
  __shared__ uint32_t s_start, s_nbig, s_tile;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_tile = alloc ? blockIdx.x : atomicAdd(ticket, 1u);
  __syncthreads();
  const int t = static_cast<int>(s_tile);
  const int tx = t % tiles_x, ty = t / tiles_x;
  unsigned long long* bk = bucket + static_cast<int64_t>(t) * bucket_cap;
  // the listed large-footprint primitives (k_preprocess: more than kBigPairs tiles) that cover this
  // tile join its bucket behind the scattered pairs (keys are unique, the sort fixes the order)
  const uint32_t fs = fill[static_cast<int64_t>(t) * kBinStride];
  const uint32_t nbig = counters[kCntBig];
  if (threadIdx.x == 0) s_nbig = 0u;
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbig; b += blockDim.x) {
    const uint32_t id = big_ids[b];
    const int4 q = rect_id[id];
    if (tx >= q.x && tx <= q.y && ty >= q.z && ty <= q.w) {
      const uint32_t slot = fs + atomicAdd(&s_nbig, 1u);
      if (slot < bucket_cap) bk[slot] = pair_key(depth_id[id], id);
    }
  }
  __syncthreads();
  const uint32_t f = fs + s_nbig;
  const uint32_t nb = min(f, bucket_cap);
  if (alloc) {   // any list placement will do: one atomic, no look-back
    if (threadIdx.x == 0) {
      const uint32_t e = nb ? atomicAdd(alloc, nb) : 0u;
      s_start = e;
      if (f > 0) atomicMax(&ds->max_tile, f);
      if (f > bucket_cap) ds->overflow = 1u;
      if (e + nb > pair_cap) ds->overflow = 1u;
      if (t == 0) ds->V = counters[kCntVisible];
      // the last CTA to place its list records the pair total M and re-zeroes both counters
      __threadfence();
      if (atomicAdd(ticket, 1u) == gridDim.x - 1) {   // (the ticket is free: tiles go by blockIdx here)
        __threadfence();
        const uint32_t m = atomicAdd(alloc, 0u);
        ds->M = m;
        atomicMax(&ds->M_max, m);
        if (m > pair_cap) ds->overflow = 1u;
        *alloc = 0u;
        *ticket = 0u;
      }
    }
  } else if (threadIdx.x == 0) {
    tile_count_publish(fill, t, nb);
  }
  // a short list is sorted in shared memory before its start is known: the look-back's waits
  // overlap the sort
  const bool in_smem = nb <= static_cast<uint32_t>(kSortChunk);
  unsigned long long* k = (in_smem && nb > 0) ? s_k[sort_chunk(bk, static_cast<int>(nb), s_k)] : nullptr;
  if (!alloc && threadIdx.x < 32) {
    const uint32_t e = tile_list_start(fill, t, nb);
    if (threadIdx.x == 0) {
      s_start = e;
      if (f > 0) atomicMax(&ds->max_tile, f);
      if (f > bucket_cap) ds->overflow = 1u;
      if (t == 0) ds->V = counters[kCntVisible];
      if (t == static_cast<int>(gridDim.x) - 1) {   // the pair total M (k_tile_scan's, without its launch)
        ds->M = e + nb;
        atomicMax(&ds->M_max, e + nb);
        if (e + nb > pair_cap) ds->overflow = 1u;
      }
    }
  }
  __syncthreads();
  const uint32_t s0 = min(s_start, pair_cap);
  const int n = static_cast<int>(min(nb, pair_cap - s0));
  if (threadIdx.x == 0) ranges[t] = n ? make_int2(static_cast<int>(s0), static_cast<int>(s0) + n) : make_int2(0, 0);
  if (n == 0) return;
  unsigned long long* sk = skey + s0;
  if (in_smem) {
    fix_ties(k, n, depth_id);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t id = static_cast<uint32_t>(k[i]);
      sid[s0 + i] = id;
      if (sslot) sslot[s0 + i] = pj_slot[id];
    }
    return;
  }
  sort_long(bk, sk, n, s_k, depth_id);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t id = static_cast<uint32_t>(sk[i]);
    sid[s0 + i] = id;
    if (sslot) sslot[s0 + i] = pj_slot[id];
  }
}


}  // namespace

void run_binning(Workspace& ws, DevState* ds, int64_t P, int tiles_x, int ntiles, cudaStream_t st, int64_t* L,
                 bool want_slots, bool any_order) {
  const uint32_t pair_cap = static_cast<uint32_t>(ws.pair_cap);
  const uint32_t bcap = static_cast<uint32_t>(ws.bucket_cap);
  // the tracking loop's short lists sort as fast with 128 threads, and more CTAs fit an SM
#ifndef GSF_MAP_SORT_THREADS
#define GSF_MAP_SORT_THREADS 256
#endif
  const int threads = any_order ? (want_slots ? 128 : GSF_MAP_SORT_THREADS) : 256;
  launch_pdl(k_tile_sort, dim3(ntiles), dim3(threads), 0, st, ws.tile_fill, pair_cap, ws.bucket, bcap, ws.skey, ws.sid, ws.depth_id, ws.ranges,
                                      ws.pj_slot, want_slots ? ws.sslot : nullptr, ds, ws.bin_counters, ws.big_ids,
                                      ws.rect_id, tiles_x, ws.bin_counters + kCntSortTicket,
                                      any_order ? ws.bin_counters + kCntTileAlloc : nullptr);
  ++*L;
}

}  // namespace gsfk
