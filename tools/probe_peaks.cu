// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// fp64 FMA throughput (DFMA, CUDA cores) and host<->device copy rates.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
         a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dfma_loop<<<sms * 8, 512>>>(out, 16);
  cudaEventRecord(a);
  dfma_loop<<<sms * 8, 512>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fmas = (double)sms * 8 * 512 * iters * 16 * 8;
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"clock_mhz\": %d, \"ms\": %.3f}\n",
         2 * fmas / (ms * 1e-3) / 1e12, sms, clk / 1000, ms);
  // copies
  const size_t bytes = 1ull << 30;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, bytes, 0);
  cudaHostAlloc(&h2, bytes, 0);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double h2d = bytes / (ms * 1e-3) / 1e9;
    cudaEventRecord(a, s1);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double d2h = bytes / (ms * 1e-3) / 1e9;
    cudaDeviceSynchronize();
    cudaEvent_t c0, c1;
    cudaEventCreate(&c0);
    cudaEventCreate(&c1);
    cudaEventRecord(a, s1);
    cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(c0, s2);
    cudaStreamWaitEvent(s1, c0, 0);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"h2d_gbs\": %.1f, \"d2h_gbs\": %.1f, \"both_concurrent_gbs_each\": %.1f}\n", h2d,
           d2h, bytes / (ms * 1e-3) / 1e9);
  }
  int engines = 0;
  cudaDeviceGetAttribute(&engines, cudaDevAttrAsyncEngineCount, dev);
  printf("{\"async_engines\": %d}\n", engines);
  return 0;
}
