// Cost of one grid-wide reduction step of the fused MGS (krylov.cu) on 148
// co-resident 512-thread blocks: (a) cooperative_groups grid.sync() alone,
// (b) the MGS fold (block sum -> partial -> grid.sync -> every block folds
// the 148 partials), (c) the same fold over a flag barrier (partial stored,
// one release add per block, acquire spin, fold), (d) (c) with the partials
// read by 5 warps (one 32-partial slice each) instead of one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gsp tools/grid_sync_probe.cu && /tmp/gsp
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int T = 512;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) t = warp_sum(threadIdx.x < T / 32 ? sh[threadIdx.x] : 0.0);
  __syncthreads();
  return t;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(T, 1) probe(int mode, int iters, double* part, unsigned* counter, double* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  __shared__ double bc;
  const int G = gridDim.x, tid = threadIdx.x;
  double x = 1.0 + blockIdx.x * 1e-3 + tid * 1e-6;
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      grid.sync();
      continue;
    }
    const double b = block_sum(x, sh);
    double* slot = part + (it & 1) * G;
    if (mode == 1) {
      if (tid == 0) slot[blockIdx.x] = b;
      grid.sync();
    } else {
      if (tid == 0) {
        slot[blockIdx.x] = b;
        red_release_add(counter, 1u);  // orders the partial before the arrival
        const unsigned target = static_cast<unsigned>(G) * (it + 1);
        while (ld_acquire(counter) < target) {
        }
      }
      __syncthreads();
    }
    if (mode <= 2) {
      if (tid < 32) {
        double acc = 0.0;
        for (int i = tid; i < G; i += 32) acc += slot[i];
        acc = warp_sum(acc);
        if (tid == 0) bc = acc;
      }
    } else {  // 5 warps read a 32-partial slice each, then warp 0 combines in order
      const int w = tid >> 5, l = tid & 31;
      if (w < (G + 31) / 32) {
        const int i = w * 32 + l;
        double v = i < G ? __ldcg(slot + i) : 0.0;
        v = warp_sum(v);
        if (l == 0) sh[w] = v;
      }
      __syncthreads();
      if (tid == 0) {
        double acc = 0.0;
        for (int k = 0; k < (G + 31) / 32; ++k) acc += sh[k];
        bc = acc;
      }
    }
    __syncthreads();
    x = x * 0.5 + bc * 1e-9;
  }
  if (tid == 0) out[blockIdx.x] = x;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out;
  unsigned* counter;
  cudaMalloc(&part, 2 * sms * sizeof(double));
  cudaMalloc(&out, sms * sizeof(double));
  cudaMalloc(&counter, sizeof(unsigned));
  const char* names[] = {"grid.sync alone", "MGS fold (grid.sync)", "fold over flag barrier",
                         "flag barrier, 5-warp fold"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      int iters = 2000;
      cudaMemset(counter, 0, sizeof(unsigned));
      void* args[] = {&mode, &iters, &part, &counter, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, dim3(sms), dim3(T), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 1)
        printf("%-28s %s %.3f us per step (%d blocks)\n", names[mode], e ? cudaGetErrorString(e) : "",
               1e3 * ms / iters, sms);
    }
  }
  return 0;
}
