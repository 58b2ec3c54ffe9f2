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
//                   primitives with more than kBigPairs tiles (order inside a bucket is arbitrary)
//   k_scatter_big   one 1024-thread CTA per listed large-footprint primitive, so a primitive
//                   covering a thousand tiles does not serialise one warp
//   k_tile_scan     one CTA: exclusive scan of the tile counts -> list starts, pair total M,
//                   longest list (a bucket overflow makes the host grow the buckets and re-run)
//   k_tile_sort     one CTA per tile: 32-key runs sorted in registers (warp bitonic), then
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

__global__ void __launch_bounds__(1024) k_tile_scan(const uint32_t* __restrict__ fill, int ntiles, uint32_t bucket_cap,
                                                    uint32_t* __restrict__ start, const uint32_t* counters,
                                                    uint32_t pair_cap, DevState* ds) {
  constexpr int kPer = 4;   // consecutive tiles per thread: one pass covers 4096 tiles (configs[1]: 3,225)
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_max[32];
  __shared__ uint32_t s_carry, s_mx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = s_mx = 0;
  __syncthreads();
  for (int base = 0; base < ntiles; base += 1024 * kPer) {
    uint32_t v[kPer], f[kPer], run = 0, fm = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int t = base + tid * kPer + q;
      f[q] = t < ntiles ? fill[static_cast<int64_t>(t) * kBinStride] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      v[q] = min(f[q], bucket_cap);
      run += v[q];
      fm = max(fm, f[q]);
    }
    uint32_t x = run;   // inclusive warp scan of the per-thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const uint32_t wm = __reduce_max_sync(0xffffffffu, fm);
    if (lane == 31) s_warp[warp] = x;
    if (lane == 0) s_max[warp] = wm;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;
      const uint32_t m = __reduce_max_sync(0xffffffffu, s_max[lane]);
      if (lane == 0) s_mx = max(s_mx, m);
    }
    __syncthreads();
    uint32_t e = s_carry + (warp ? s_warp[warp - 1] : 0u) + x - run;   // exclusive start of this thread's tiles
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int t = base + tid * kPer + q;
      if (t < ntiles) start[t] = e;
      e += v[q];
    }
    __syncthreads();
    if (tid == 1023) s_carry = e;
    __syncthreads();
  }
  if (tid == 0) {
    ds->M = s_carry;
    ds->V = counters[kCntVisible];
    ds->max_tile = s_mx;
    if (s_carry > pair_cap || s_mx > bucket_cap) ds->overflow = 1u;
  }
}

__global__ void __launch_bounds__(1024) k_scatter_big(const uint32_t* __restrict__ big_ids, const uint32_t* counters,
                                                      const int4* __restrict__ rect_id, const double* __restrict__ depth_id,
                                                      int tiles_x, uint32_t* __restrict__ fill, uint32_t bucket_cap,
                                                      unsigned long long* __restrict__ bucket) {
  const uint32_t nbig = counters[kCntBig];
  for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
    const uint32_t id = big_ids[b];
    const int4 q = rect_id[id];
    const unsigned long long key = pair_key(depth_id[id], id);
    const int w = q.y - q.x + 1;
    const int c = w * (q.w - q.z + 1);
    for (int r = threadIdx.x; r < c; r += blockDim.x) {
      const int row = r / w;
      bucket_put(fill, bucket, bucket_cap, (q.z + row) * tiles_x + q.x + (r - row * w), key);
    }
  }
}

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

__global__ void __launch_bounds__(256) k_tile_sort(const uint32_t* __restrict__ fill, const uint32_t* __restrict__ start,
                                                   uint32_t pair_cap, unsigned long long* bucket, uint32_t bucket_cap,
                                                   unsigned long long* skey, uint32_t* __restrict__ sid,
                                                   const double* __restrict__ depth_id, int2* __restrict__ ranges,
                                                   const uint32_t* __restrict__ pj_slot, uint32_t* __restrict__ sslot) {
  __shared__ unsigned long long s_k[2][kSortChunk];
  const int t = blockIdx.x;
  const uint32_t s0 = min(start[t], pair_cap);
  const int n = static_cast<int>(min(min(fill[static_cast<int64_t>(t) * kBinStride], bucket_cap), pair_cap - s0));
  if (threadIdx.x == 0) ranges[t] = n ? make_int2(static_cast<int>(s0), static_cast<int>(s0) + n) : make_int2(0, 0);
  if (n == 0) return;
  unsigned long long* bk = bucket + static_cast<int64_t>(t) * bucket_cap;
  unsigned long long* sk = skey + s0;
  if (n <= kSortChunk) {
    unsigned long long* k = s_k[sort_chunk(bk, n, s_k)];
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
  if (P > 0) {   // the regular pairs were scattered by k_preprocess
    k_scatter_big<<<32, 1024, 0, st>>>(ws.big_ids, ws.bin_counters, ws.rect_id, ws.depth_id, tiles_x, ws.tile_fill, bcap,
                                        ws.bucket);
    ++*L;
  }
  k_tile_scan<<<1, 1024, 0, st>>>(ws.tile_fill, ntiles, bcap, ws.tile_start, ws.bin_counters, pair_cap, ds);
  ++*L;
  k_tile_sort<<<ntiles, 256, 0, st>>>(ws.tile_fill, ws.tile_start, pair_cap, ws.bucket, bcap, ws.skey, ws.sid, ws.depth_id,
                                      ws.ranges, ws.pj_slot, want_slots ? ws.sslot : nullptr);
  ++*L;
}

}  // namespace gsfk
