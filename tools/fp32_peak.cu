// fp32_peak.cu — measured FP32 FMA-pipe throughput of this B200 (the roofline denominator of the
// blend / backward kernels, which are FP32-issue bound and use packed FFMA2).
//
//   scalar FFMA : 8 independent a = a * b + c chains per thread
//   packed FFMA2: 8 independent float2 chains (__ffma2_rn, one instruction = 2 FMAs)
//
// Grid = 148 SMs x 8 CTAs x 256 threads, 8192 iterations, timed with CUDA events (best of 5 after a
// warm-up).  Prints one JSON object; bench.py reads profiles/*fp32_peak*.json for roofline.peak.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 8192;

__global__ void __launch_bounds__(256) k_ffma(float* out, float b, float c) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float* out, float b, float c) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-7f + i, threadIdx.x * 2e-7f - i);
  const float2 bb = make_float2(b, b), cc = make_float2(c, c);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], bb, cc);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
static double run(K kern, int blocks, float* out, double flops_per_thread) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(out, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<blocks, 256>>>(out, 0.999f, 1e-4f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return flops_per_thread * blocks * 256.0 / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int blocks = prop.multiProcessorCount * 8;
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  const double f1 = run(k_ffma, blocks, out, 2.0 * 8 * kIters);
  const double f2 = run(k_ffma2, blocks, out, 4.0 * 8 * kIters);
  const double nominal = prop.multiProcessorCount * 128.0 * 2.0 * clk_khz * 1e3 / 1e12;
  std::printf("{\"ffma_tflops\": %.3f, \"ffma2_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
              "\"nominal_tflops_128_lanes\": %.3f, \"how\": \"best of 5 CUDA-event-timed launches, %d CTAs x 256 threads, "
              "8 independent chains x %d iterations per thread\"}\n",
              f1, f2, prop.multiProcessorCount, clk_khz / 1e3, nominal, blocks, kIters);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
