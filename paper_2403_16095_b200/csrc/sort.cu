// sort.cu — hand-written decoupled-lookback scan and onesweep LSD radix sort (sm_100a).
//
// Replaces the reference's single-threaded std::sort of visible ids by (depth, id)
// (rasterizer.cpp:69-79) and its serial push_back construction of per-tile lists
// (rasterizer.cpp:193-212).  Both passes are stable, so:
//   depth sort:  keys = fp32 depth bits (offset by near), values = ids in id order, then a
//                fixup pass orders fp32-equal runs by the exact fp64 (depth, id) comparison;
//   tile sort:   pairs are generated in depth-rank order, so a stable sort by tile id yields
//                every tile list in global depth order — exactly the reference's lists.
#include "kernels.h"

namespace gsfk {

namespace {

constexpr uint32_t kFlagA = 1u << 30;   // aggregate published
constexpr uint32_t kFlagP = 2u << 30;   // inclusive prefix published
constexpr uint32_t kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }
__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Exclusive scan of one value per thread over a 256-thread block; returns the block total.
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t& excl, uint32_t* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t incl = warp_incl_scan(v, lane);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < 8 ? s_warp[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w, lane);
    if (lane < 8) s_warp[lane] = wi - w;
    if (lane == 7) s_warp[8] = wi;
  }
  __syncthreads();
  excl = s_warp[warp] + incl - v;
  const uint32_t total = s_warp[8];
  __syncthreads();
  return total;
}

}  // namespace

// ---------------------------------------------------------------------------------------
// Exclusive scan (u32) with decoupled look-back.  n is read from the device when n_dev is set.
// ---------------------------------------------------------------------------------------
constexpr int kScanBlock = 256, kScanIpt = 8, kScanTile = kScanBlock * kScanIpt;

__global__ void __launch_bounds__(kScanBlock) k_scan_excl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                          const uint32_t* n_dev, uint32_t n_host, uint32_t* total_out,
                                                          unsigned long long* state, uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_warp[9];
  const int tid = threadIdx.x;
  const uint32_t n = n_dev ? min(*n_dev, n_host) : n_host;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kScanTile;
  if (base >= n) {
    if (n == 0 && tile == 0 && tid == 0) *total_out = 0;
    return;
  }
  uint32_t v[kScanIpt];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kScanIpt; ++j) {
    const uint32_t idx = base + tid * kScanIpt + j;
    v[j] = idx < n ? in[idx] : 0u;
    sum += v[j];
  }
  uint32_t texcl;
  const uint32_t btotal = block_excl_scan_256(sum, texcl, s_warp);
  if (tid == 0) {
    uint32_t excl = 0;
    if (tile == 0) {
      atomicExch(&state[0], (2ull << 32) | btotal);
    } else {
      atomicExch(&state[tile], (1ull << 32) | btotal);
      int p = static_cast<int>(tile) - 1;
      bool done = false;
      while (!done) {
        unsigned long long s[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = (p - j >= 0) ? ld_vol64(&state[p - j]) : (2ull << 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (!done) {
            unsigned long long v = s[j];
            while ((v >> 32) == 0) v = ld_vol64(&state[p - j]);
            excl += static_cast<uint32_t>(v);
            if ((v >> 32) == 2) done = true;
          }
        }
        p -= 8;
      }
      atomicExch(&state[tile], (2ull << 32) | (excl + btotal));
    }
    s_prefix = excl;
  }
  __syncthreads();
  uint32_t running = s_prefix + texcl;
#pragma unroll
  for (int j = 0; j < kScanIpt; ++j) {
    const uint32_t idx = base + tid * kScanIpt + j;
    if (idx < n) out[idx] = running;
    running += v[j];
  }
  if (base + kScanTile >= n && tid == 0) *total_out = s_prefix + btotal;
}

// ---------------------------------------------------------------------------------------
// Onesweep radix sort: one histogram kernel for all digits, then one scatter kernel per digit
// with per-digit decoupled look-back.  8-bit digits, 256 threads x 16 keys per CTA tile.
// ---------------------------------------------------------------------------------------
constexpr int kRsBlock = 256, kRsWarps = 8, kRsIpt = 16, kRsTile = kRsBlock * kRsIpt, kRadix = 256;

__global__ void __launch_bounds__(kRsBlock) k_radix_hist(const uint32_t* __restrict__ keys, const uint32_t* n_dev,
                                                         uint32_t n_host, int passes, int begin_bit, uint32_t* hist) {
  __shared__ uint32_t s_h[4][kRadix];
  const uint32_t n = n_dev ? min(*n_dev, n_host) : n_host;
  for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0u;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p][(k >> (begin_bit + 8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const uint32_t c = (&s_h[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

__global__ void __launch_bounds__(kRsBlock) k_onesweep(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                       uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                       const uint32_t* n_dev, uint32_t n_host, int shift,
                                                       const uint32_t* __restrict__ hist, uint32_t* lookback,
                                                       uint32_t* tile_ctr) {
  __shared__ uint32_t s_whist[kRsWarps][kRadix + 1];
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_warp[9];
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = n_dev ? min(*n_dev, n_host) : n_host;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kRsTile;
  if (base >= n) return;
  for (int i = tid; i < kRsWarps * (kRadix + 1); i += kRsBlock) (&s_whist[0][0])[i] = 0u;
  __syncthreads();
  const uint32_t wbase = base + warp * 32 * kRsIpt;
  uint32_t k[kRsIpt], v[kRsIpt], rank[kRsIpt];
#pragma unroll
  for (int j = 0; j < kRsIpt; ++j) {
    const uint32_t idx = wbase + j * 32 + lane;
    if (idx < n) {
      k[j] = keys_in[idx];
      v[j] = vals_in ? vals_in[idx] : idx;
    } else {
      k[j] = 0u;
      v[j] = 0u;
    }
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kRsIpt; ++j) {
    const uint32_t idx = wbase + j * 32 + lane;
    const uint32_t d = idx < n ? ((k[j] >> shift) & 255u) : 256u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t r = __popc(peers & lt_mask);
    const uint32_t prev = s_whist[warp][d];
    __syncwarp();
    if (r == 0) s_whist[warp][d] = prev + __popc(peers);
    __syncwarp();
    rank[j] = prev + r;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, look-back over tiles, global base
  {
    const int d = tid;
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t t = s_whist[w][d];
      s_whist[w][d] = cnt;
      cnt += t;
    }
    uint32_t* lb = lookback + static_cast<size_t>(tile) * kRadix;
    uint32_t excl = 0;
    if (tile == 0) {
      st_vol(&lb[d], kFlagP | cnt);
    } else {
      st_vol(&lb[d], kFlagA | cnt);
      // batched look-back: 8 predecessor words in flight per round instead of a serial chain
      int p = static_cast<int>(tile) - 1;
      bool done = false;
      while (!done) {
        uint32_t s[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = (p - j >= 0) ? ld_vol(&lookback[static_cast<size_t>(p - j) * kRadix + d]) : kFlagP;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (!done) {
            uint32_t v = s[j];
            while ((v & ~kValMask) == 0) v = ld_vol(&lookback[static_cast<size_t>(p - j) * kRadix + d]);
            excl += v & kValMask;
            if (v & kFlagP) done = true;
          }
        }
        p -= 8;
      }
      st_vol(&lb[d], kFlagP | (excl + cnt));
    }
    uint32_t dexcl;
    block_excl_scan_256(hist[d], dexcl, s_warp);
    s_base[d] = dexcl + excl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRsIpt; ++j) {
    const uint32_t idx = wbase + j * 32 + lane;
    if (idx < n) {
      const uint32_t d = (k[j] >> shift) & 255u;
      const uint32_t pos = s_base[d] + s_whist[warp][d] + rank[j];
      keys_out[pos] = k[j];
      vals_out[pos] = v[j];
    }
  }
}

// Orders runs of equal fp32 depth keys by the exact (fp64 depth, id) rule of
// rasterizer.cpp:74-77.  Runs are tiny except for exactly coplanar primitives, whose fp64
// depths are then equal too and the id order left by the stable sort is already final.
__global__ void k_sort_fixup(const uint32_t* __restrict__ keys, uint32_t* vals, const double* __restrict__ depth_id,
                             const uint32_t* n_dev, uint32_t n_cap) {
  const uint32_t n = min(*n_dev, n_cap);
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;
  if (i + 1 >= n || keys[i + 1] != key) return;
  uint32_t e = i + 1;
  bool sorted = true;
  double prev_d = depth_id[vals[i]];
  uint32_t prev_id = vals[i];
  while (e < n && keys[e] == key) {
    const uint32_t id = vals[e];
    const double dd = depth_id[id];
    if (dd < prev_d || (dd == prev_d && id < prev_id)) sorted = false;
    prev_d = dd;
    prev_id = id;
    ++e;
  }
  if (sorted) return;
  for (uint32_t a = i + 1; a < e; ++a) {
    const uint32_t id = vals[a];
    const double dd = depth_id[id];
    uint32_t b = a;
    while (b > i) {
      const uint32_t pid = vals[b - 1];
      const double pd = depth_id[pid];
      if (pd < dd || (pd == dd && pid < id)) break;
      vals[b] = pid;
      --b;
    }
    vals[b] = id;
  }
}

// ---------------------------------------------------------------------------------------
// Host wrappers
// ---------------------------------------------------------------------------------------
void launch_scan_excl(const uint32_t* in, uint32_t* out, const uint32_t* n_dev, uint32_t n_max, uint32_t* total_out,
                      ScanTemp& tmp, cudaStream_t st, int64_t* launches) {
  const int tiles = div_up(n_max > 0 ? n_max : 1, kScanTile);
  GSF_CUDA_CHECK(cudaMemsetAsync(tmp.state, 0, sizeof(unsigned long long) * tiles + sizeof(uint32_t) * 4, st));
  uint32_t* ctr = reinterpret_cast<uint32_t*>(tmp.state + tiles);
  k_scan_excl<<<tiles, kScanBlock, 0, st>>>(in, out, n_dev, n_max, total_out, tmp.state, ctr);
  ++*launches;
}

size_t scan_temp_bytes(uint32_t n_max) {
  return sizeof(unsigned long long) * (div_up(n_max > 0 ? n_max : 1, kScanTile) + 1) + 64;
}

size_t radix_temp_bytes(uint32_t n_max, int max_passes) {
  const size_t tiles = div_up(n_max > 0 ? n_max : 1, kRsTile);
  return sizeof(uint32_t) * (4 * kRadix + max_passes * (tiles * kRadix + 32)) + 64;
}

int radix_sort_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                   uint32_t n_max, int begin_bit, int end_bit, bool vals_are_index, uint32_t* temp, cudaStream_t st,
                   int64_t* launches) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  if (passes <= 0) return 0;
  const size_t tiles = div_up(n_max > 0 ? n_max : 1, kRsTile);
  uint32_t* hist = temp;
  uint32_t* lb = temp + 4 * kRadix;
  const size_t per_pass = tiles * kRadix + 32;
  GSF_CUDA_CHECK(cudaMemsetAsync(temp, 0, sizeof(uint32_t) * (4 * kRadix + passes * per_pass), st));
  const int hist_blocks = std::max(1, std::min(div_up(n_max > 0 ? n_max : 1, kRsBlock * 16), 148 * 4));
  k_radix_hist<<<hist_blocks, kRsBlock, 0, st>>>(keys, n_dev, n_max, passes, begin_bit, hist);
  ++*launches;
  uint32_t* kin = keys;
  uint32_t* vin = vals;
  uint32_t* kout = keys_alt;
  uint32_t* vout = vals_alt;
  for (int p = 0; p < passes; ++p) {
    uint32_t* pass_lb = lb + p * per_pass;
    uint32_t* ctr = pass_lb + tiles * kRadix;
    k_onesweep<<<static_cast<int>(tiles), kRsBlock, 0, st>>>(kin, (p == 0 && vals_are_index) ? nullptr : vin, kout, vout,
                                                              n_dev, n_max, begin_bit + 8 * p, hist + p * kRadix, pass_lb, ctr);
    ++*launches;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  return passes;  // result is in (keys, vals) if passes is even, else in the *_alt buffers
}

void launch_sort_fixup(const uint32_t* keys, uint32_t* vals, const double* depth_id, const uint32_t* n_dev, uint32_t n_max,
                       cudaStream_t st, int64_t* launches) {
  if (n_max == 0) return;
  k_sort_fixup<<<div_up(n_max, 256), 256, 0, st>>>(keys, vals, depth_id, n_dev, n_max);
  ++*launches;
}

}  // namespace gsfk
