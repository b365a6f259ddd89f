// Dependent-chain latency probe (one warp): DFMA, DADD, LDS.64/128, FFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, int n) {
  __shared__ double2 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double2(1.0 / (i + 1), 0.5);
  __syncthreads();
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);  // DFMA chain
  long long t1 = clock64();
  float fa = (float)out[3], fb = (float)out[4];
  for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, 0.5f);  // FFMA chain
  long long t2 = clock64();
  int idx = threadIdx.x & 7;
  double acc = 0;
  for (int i = 0; i < n; ++i) {  // LDS.128 chain (address depends on the previous load)
    double2 v = s[idx];
    idx = ((int)v.y + i) & 1023;
    acc += v.x;
  }
  long long t3 = clock64();
  double2 z = make_double2(0, 0);
  double2 w = make_double2(out[5], out[6]), x = make_double2(out[7], out[8]);
  for (int i = 0; i < n; ++i) {  // complex fma chain (4 DFMA, depth 2)
    z.x = fma(w.x, x.x, z.x);
    z.x = fma(-w.y, x.y, z.x);
    z.y = fma(w.x, x.y, z.y);
    z.y = fma(w.y, x.x, z.y);
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
  out[16 + threadIdx.x] = a + fa + acc + z.x + z.y;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 64);
  double h[16] = {1.0, 0.999, 1e-3, 1.0, 0.999, 0.3, 0.2, 0.1, 0.4};
  cudaMemcpy(out, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 4096;
  for (int threads : {32, 128, 512}) {
    probe<<<1, threads>>>(out, cyc, n);
    long long c[4];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("threads %3d: DFMA %.1f  FFMA %.1f  LDS.128-chain %.1f  cfma(4 DFMA) %.1f cycles/step\n", threads,
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n);
  }
  probe<<<148 * 4, 512>>>(out, cyc, n);
  long long c[4];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("full chip 4x512/SM: DFMA %.1f  FFMA %.1f  LDS %.1f  cfma %.1f\n", c[0] / (double)n, c[1] / (double)n,
         c[2] / (double)n, c[3] / (double)n);
  return 0;
}
