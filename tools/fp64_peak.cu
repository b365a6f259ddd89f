// FP64 peak microbenchmark for B200 (sm_100a): FFMA (DFMA) and DMMA.8x8x4.
// Used once to obtain the FP64 roofline denominator, which MEASURED_PEAKS.json
// does not carry. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double s) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], s, 1e-12);
  }
  double r = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) r += acc[c];
  if (r == 1234.5) out[0] = r;
}

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double d[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) r += d[c][0] + d[c][1];
  if (r == 1234.5) out[0] = r;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * bpsm;
      dfma_loop<8><<<blocks, threads>>>(out, 100, 0.9999);
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, threads>>>(out, iters, 0.9999);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)blocks * threads;
      printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.3f}\n", bpsm, threads,
             flops / (ms * 1e-3) / 1e12);
      dmma_loop<4><<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<4><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double mma_flops = 512.0 * 4 * iters * (double)blocks * (threads / 32);
      printf("{\"kind\":\"dmma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.3f}\n", bpsm, threads,
             mma_flops / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\":\"%s\",\"sms\":%d}\n", cudaGetErrorString(err), sms);
  return err == cudaSuccess ? 0 : 1;
}
