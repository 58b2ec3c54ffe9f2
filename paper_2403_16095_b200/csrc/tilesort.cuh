// tilesort.cuh — per-tile list sort building blocks (binning.cu's k_tile_sort and the tracking
// loop's fused sort + blend, raster_fwd.cu): register-sorted 32-key runs merged by rank in shared
// memory, merge-path passes through global memory for long lists, and the fp64 tie fix-up.
#pragma once
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

// A list longer than kSortChunk: chunks sorted in shared memory into sk, then merge passes
// ping-ponging between sk and the (consumed) bucket bk; the sorted, tie-fixed list ends in sk.
__device__ void sort_long(unsigned long long* bk, unsigned long long* sk, int n, unsigned long long (*s_k)[kSortChunk],
                          const double* __restrict__ depth_id) {
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
}

}  // namespace
}  // namespace gsfk
