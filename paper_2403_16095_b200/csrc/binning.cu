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
//                   whose fp32 depths tie by the exact fp64 depth (then id).
//
// Sort key: (fp32 bits of the depth) << 32 | id, one 64-bit integer.  Positive floats order like
// their bit patterns and fp32 rounding is monotone, so this is the reference order except inside
// runs of equal fp32 depth, which the fix-up resolves with the fp64 depth.  Keys are unique (id),
// so the result does not depend on the scatter order: deterministic.
#include "kernels.h"

namespace gsfk {

namespace {

constexpr int kSortChunk = 1024;   // longest list sorted entirely in shared memory (2 x 8 KB)

// Ascending bitonic sort of 32 keys, one per lane, in registers.
__device__ __forceinline__ unsigned long long warp_sort32(unsigned long long k) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      const unsigned long long p = __shfl_xor_sync(0xffffffffu, k, j);
      const bool keep_min = ((lane & j) == 0) == ((lane & size) == 0 || size == 32);
      k = keep_min ? min(k, p) : max(k, p);
    }
  }
  return k;
}

// Number of keys of the sorted run r[0, len) below k (upper: at or below).
__device__ __forceinline__ int run_rank(const unsigned long long* r, int len, unsigned long long k, bool upper) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    const unsigned long long v = r[m];
    if (upper ? v <= k : v < k)
      lo = m + 1;
    else
      hi = m;
  }
  return lo;
}

// Sort n <= kSortChunk keys of src (global) in shared memory: register-sorted 32-runs, then
// pairwise merges by rank.  Returns the s_k buffer holding the sorted keys (first n; the padding
// ~0 sorts to the end, and equal padding keys are separated by the lower/upper rank rule of the
// two runs, so every element gets a distinct slot).
__device__ int sort_chunk(const unsigned long long* src, int n, unsigned long long (*s_k)[kSortChunk]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int nruns = (n + 31) >> 5;
  const int N = nruns << 5;
  for (int r = warp; r < nruns; r += nwarps) {
    const int i = (r << 5) + lane;
    s_k[0][i] = warp_sort32(i < n ? src[i] : ~0ull);
  }
  __syncthreads();
  int buf = 0;
  for (int w = 32; w < N; w <<= 1) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const int r = i / w;
      const int pbeg = (r ^ 1) * w;
      const unsigned long long k = s_k[buf][i];
      int pos = i;
      if (pbeg < N) pos = (r & ~1) * w + (i - r * w) + run_rank(&s_k[buf][pbeg], min(w, N - pbeg), k, (r & 1) != 0);
      s_k[buf ^ 1][pos] = k;
    }
    __syncthreads();
    buf ^= 1;
  }
  return buf;
}

// Runs of equal fp32 depth in (fp64 depth, id) order (rasterizer.cpp:74-77).  Inside such a run
// the keys are already in id order, so the list is in reference order iff no adjacent pair of equal
// fp32 depth has a smaller fp64 depth behind it: one parallel round of depth reads settles the
// common case (duplicate layers share their fp64 depth); otherwise the first thread of each run
// insertion-sorts it (runs are a handful of keys).  Ends with a __syncthreads().
__device__ void fix_ties(unsigned long long* k, int n, const double* __restrict__ depth_id) {
  __shared__ int s_inv;
  if (threadIdx.x == 0) s_inv = 0;
  __syncthreads();
  bool inv = false;
  for (int i = threadIdx.x; i + 1 < n; i += blockDim.x) {
    const unsigned long long a = k[i], b = k[i + 1];
    if ((a >> 32) == (b >> 32) && __ldg(depth_id + static_cast<uint32_t>(b)) < __ldg(depth_id + static_cast<uint32_t>(a)))
      inv = true;
  }
  if (inv) s_inv = 1;
  __syncthreads();
  if (!s_inv) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t hi = static_cast<uint32_t>(k[i] >> 32);
    const bool starts = (i == 0 || static_cast<uint32_t>(k[i - 1] >> 32) != hi) && i + 1 < n &&
                        static_cast<uint32_t>(k[i + 1] >> 32) == hi;
    if (!starts) continue;
    int e = i + 2;
    while (e < n && static_cast<uint32_t>(k[e] >> 32) == hi) ++e;
    for (int a = i + 1; a < e; ++a) {
      const unsigned long long ka = k[a];
      const uint32_t ida = static_cast<uint32_t>(ka);
      const double da = depth_id[ida];
      int b = a - 1;
      while (b >= i) {
        const uint32_t idb = static_cast<uint32_t>(k[b]);
        const double db = depth_id[idb];
        if (db < da || (db == da && idb < ida)) break;
        k[b + 1] = k[b];
        --b;
      }
      k[b + 1] = ka;
    }
  }
  __syncthreads();
}

// One merge pass over a segment of n keys: runs of width w in a -> runs of 2w in b.
__device__ void merge_pass(const unsigned long long* a, unsigned long long* b, int n, int w) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  int o = threadIdx.x * per;
  const int o1 = min(n, o + per);
  while (o < o1) {
    const int plo = (o / (2 * w)) * (2 * w);
    const int mid = min(plo + w, n), phi = min(plo + 2 * w, n);
    const int la = mid - plo, lb = phi - mid;
    const unsigned long long* A = a + plo;
    const unsigned long long* B = a + mid;
    const int d = o - plo;
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {   // merge path: number of A keys among the first d outputs
      const int m = (lo + hi) >> 1;
      if (B[d - 1 - m] < A[m])
        hi = m;
      else
        lo = m + 1;
    }
    int ia = lo, ib = d - lo;
    const int pend = min(o1, phi);
    for (; o < pend; ++o) b[o] = (ia < la && (ib >= lb || A[ia] < B[ib])) ? A[ia++] : B[ib++];
  }
  __syncthreads();
}

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
                                                   int tiles_x, uint32_t* ticket) {
  __shared__ unsigned long long s_k[2][kSortChunk];
  __shared__ uint32_t s_start, s_nbig, s_tile;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
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
  if (threadIdx.x == 0) tile_count_publish(fill, t, nb);
  // a short list is sorted in shared memory before its start is known: the look-back's waits
  // overlap the sort
  const bool in_smem = nb <= static_cast<uint32_t>(kSortChunk);
  unsigned long long* k = (in_smem && nb > 0) ? s_k[sort_chunk(bk, static_cast<int>(nb), s_k)] : nullptr;
  if (threadIdx.x < 32) {
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
  // long list: sorted chunks into skey, then merge passes ping-ponging with the (consumed) bucket
  for (int c = 0; c < n; c += kSortChunk) {
    const int m = min(kSortChunk, n - c);
    const unsigned long long* k = s_k[sort_chunk(bk + c, m, s_k)];
    for (int i = threadIdx.x; i < m; i += blockDim.x) sk[c + i] = k[i];
    __syncthreads();
  }
  bool in_s = true;
  for (int w = kSortChunk; w < n; w *= 2) {
    merge_pass(in_s ? sk : bk, in_s ? bk : sk, n, w);
    in_s = !in_s;
  }
  if (!in_s) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) sk[i] = bk[i];
    __syncthreads();
  }
  fix_ties(sk, n, depth_id);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t id = static_cast<uint32_t>(sk[i]);
    sid[s0 + i] = id;
    if (sslot) sslot[s0 + i] = pj_slot[id];
  }
}

}  // namespace

void run_binning(Workspace& ws, DevState* ds, int64_t P, int tiles_x, int ntiles, cudaStream_t st, int64_t* L,
                 bool want_slots) {
  const uint32_t pair_cap = static_cast<uint32_t>(ws.pair_cap);
  const uint32_t bcap = static_cast<uint32_t>(ws.bucket_cap);
#ifndef GSF_SORT_THREADS
#define GSF_SORT_THREADS 256
#endif
  launch_pdl(k_tile_sort, dim3(ntiles), dim3(GSF_SORT_THREADS), 0, st, ws.tile_fill, pair_cap, ws.bucket, bcap, ws.skey, ws.sid, ws.depth_id, ws.ranges,
                                      ws.pj_slot, want_slots ? ws.sslot : nullptr, ds, ws.bin_counters, ws.big_ids,
                                      ws.rect_id, tiles_x, ws.bin_counters + kCntSortTicket);
  ++*L;
}

}  // namespace gsfk
