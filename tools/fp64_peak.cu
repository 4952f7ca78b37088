// fp64 FMA peak of this GPU (the roofline denominator for the fp64-issue-bound element kernels;
// MEASURED_PEAKS.json has HBM and bf16 only).  Every thread runs 8 independent DFMA chains of
// length ITERS; grid = 148 SMs x 8 CTAs x 256 threads.  Prints one JSON line:
//   {"fp64_tflops": best-of-10, "dfma_per_launch": ..., "ms": ...}
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CHAINS = 8;

__global__ void k_dfma(double* out, double a, double b) {
  double r[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) r[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r[c] = fma(r[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += r[c];
  if (s == 12345.678) out[0] = s;   // never true; keeps the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  double* d;
  cudaMalloc(&d, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(d, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = double(blocks) * threads * ITERS * CHAINS;
  const double tflops = 2.0 * dfma / (best * 1e-3) / 1e12;
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  std::printf("{\"fp64_tflops\": %.4f, \"dfma_per_launch\": %.0f, \"ms\": %.5f, \"sms\": %d}\n", tflops, dfma, best, sms);
  return 0;
}
