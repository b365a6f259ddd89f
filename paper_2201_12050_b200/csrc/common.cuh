// Shared device helpers for the sm_100a periodic-FMBEM kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fpbem_cu {

using c64 = double2;  // (re, im), layout-identical to std::complex<double>

__host__ __device__ __forceinline__ c64 cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ c64 cadd(c64 a, c64 b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ c64 csub(c64 a, c64 b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ c64 cmul(c64 a, c64 b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a * b
__host__ __device__ __forceinline__ c64 cfma(c64 a, c64 b, c64 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a) * b
__host__ __device__ __forceinline__ c64 cfma_conj(c64 a, c64 b, c64 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__host__ __device__ __forceinline__ c64 cscale(c64 a, double s) { return cmk(a.x * s, a.y * s); }

constexpr int kNumSMs = 148;

// cp.async 16-byte global->shared copy with zero fill when !valid
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D += A * B on one 8x8x4 fp64 tensor-core tile (DMMA.8x8x4 in SASS)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace fpbem_cu
