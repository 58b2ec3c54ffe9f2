// Micro-probe: throughput of global integer atomics on B200 for the binning pattern
// (N increments spread over T counters, with and without a returned value).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_red(const uint32_t* idx, int n, uint32_t* cnt, int stride) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[idx[i] * stride], 1u);
}
__global__ void k_ret(const uint32_t* idx, int n, uint32_t* cnt, uint32_t* out, int stride) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = atomicAdd(&cnt[idx[i] * stride], 1u);
}
__global__ void k_smem_hist(const uint32_t* idx, int n, uint32_t* cnt, int T) {
  extern __shared__ uint32_t h[];
  for (int t = threadIdx.x; t < T; t += blockDim.x) h[t] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(&h[idx[i]], 1u);
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) if (h[t]) atomicAdd(&cnt[t], h[t]);
}

int main() {
  const int n = 563609;
  for (int T : {3225, 32768}) {
    uint32_t* h = new uint32_t[n];
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % T); }
    uint32_t *idx, *cnt, *out;
    cudaMalloc(&idx, n * 4); cudaMalloc(&cnt, (size_t)T * 32 * 4); cudaMalloc(&out, n * 4);
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int stride : {1, 8, 32}) {
      for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemset(cnt, 0, (size_t)T * 32 * 4);
          cudaEventRecord(a);
          if (mode == 0) k_red<<<(n + 255) / 256, 256>>>(idx, n, cnt, stride);
          else k_ret<<<(n + 255) / 256, 256>>>(idx, n, cnt, out, stride);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("T=%d stride=%d %s: %.1f us\n", T, stride, mode ? "atomic-ret" : "red", best * 1e3);
      }
    }
    if (T <= 12000) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(cnt, 0, (size_t)T * 4);
        cudaEventRecord(a);
        k_smem_hist<<<148 * 2, 1024, T * 4>>>(idx, n, cnt, T);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("T=%d smem-hist: %.1f us\n", T, best * 1e3);
    }
    cudaFree(idx); cudaFree(cnt); cudaFree(out); delete[] h;
  }
  return 0;
}
