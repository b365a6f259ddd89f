// Shared device helpers for the sm_100a periodic-FMBEM kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

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

constexpr int kNumSMs = 148;  // grid-sizing hint only; co-residency checks use device_sms()

// SM count of the current device (cached per device)
inline int device_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kNumSMs;
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = kNumSMs;
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

// ---- programmatic dependent launch (PDL). A kernel launched through launch_ex(..., pdl = true)
// may start while the kernel before it on the stream is still draining: its CTAs become resident as
// SMs free up and run their prologue (twiddle tables, barrier init, copies of operator data that no
// earlier kernel writes), and pdl_wait() — griddepcontrol.wait: returns when every kernel before it
// on the stream has completed and its writes are visible — must precede the first access to data an
// earlier kernel produces or still reads. Launched normally, pdl_wait() / pdl_trigger() are no-ops.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// lets the next kernel's CTAs be scheduled once every CTA of this grid has issued it (or exited)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
#endif

// FPBEM_PDL (read once): 0 (default) off; 2 the lattice DFT passes; 1 the mode product as well.
// Measured on cfg3: the passes alone 0.359 -> 0.355 ms per product, but the GMRES solve 0.1441 ->
// 0.1465 s and the host-pointer product 1.170 -> 1.165e9 DOF/s; with the mode product too 0.375 ms
// (its early-resident CTAs take the SM slots the far field's Λ stream would have used). Never while
// the stream is being captured into a graph.
inline int pdl_level() {
  static const int level = [] {
    const char* v = std::getenv("FPBEM_PDL");
    return v ? std::atoi(v) : 0;
  }();
  return level;
}
inline bool pdl_enabled(cudaStream_t stream, bool mode_product = false) {
  const int level = pdl_level();
  if (level <= 0 || (mode_product && level == 2)) return false;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) != cudaSuccess) return false;
  return st == cudaStreamCaptureStatusNone;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, bool pdl,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int kMaxDynSmem = 227 * 1024;  // sm_100a opt-in limit per CTA

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (call site, device):
// the attribute is per device context, so a process-wide flag would skip it on
// a second GPU
inline cudaError_t ensure_max_smem(std::atomic<unsigned long long>& done, const void* func, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ULL << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  // the dynamic limit is what the opt-in maximum leaves after the kernel's static shared memory
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, func);
  if (e != cudaSuccess) return e;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const int room = optin - static_cast<int>(fa.sharedSizeBytes);
  if (bytes > room) bytes = room;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

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

// ---- mbarrier / bulk-copy helpers (shared::cta addresses as u32)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D bulk copy global -> shared, completion counted in bytes on `bar` (UBLKCP in SASS)
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cp_async16_u32(unsigned dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// D += A * B on one 8x8x4 fp64 tensor-core tile (DMMA.8x8x4 in SASS)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace fpbem_cu
