// Streaming-bandwidth probe for the M2L Λ stream: every CTA pulls chunks of
// `chunk` bytes through a `ring`-deep shared-memory ring with cp.async.bulk +
// mbarrier (the m2l_zpipe_kernel pattern), touching one value per chunk so
// the copies cannot be elided. Also an LDG.128 grid-stride reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bsb tools/bulk_stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void bulk_ring(const char* __restrict__ src, size_t n_chunks, int chunk, int ring, int stride_mode,
                          double* sink) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long full[32];
  const int tid = threadIdx.x;
  // chunk order: stride_mode 0 = CTA-contiguous slices, 1 = round-robin over CTAs
  const size_t per = (n_chunks + gridDim.x - 1) / gridDim.x;
  auto chunk_id = [&](size_t i) -> size_t {
    return stride_mode ? blockIdx.x + i * gridDim.x : blockIdx.x * per + i;
  };
  size_t mine = 0;
  for (size_t i = 0;; ++i) {
    size_t c = chunk_id(i);
    if (c >= n_chunks || (stride_mode == 0 && i >= per)) break;
    ++mine;
  }
  if (tid == 0) {
    for (int s = 0; s < ring; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t issued = 0;
  auto issue = [&](size_t upto) {
    for (; issued < upto && issued < mine; ++issued) {
      const int s = issued % ring;
      const unsigned bar = su32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(buf + static_cast<size_t>(s) * chunk)),
                   "l"(src + chunk_id(issued) * chunk), "r"(chunk), "r"(bar)
                   : "memory");
    }
  };
  if (tid == 0) issue(ring);
  double acc = 0;
  const int half = ring / 2 > 0 ? ring / 2 : 1;
  for (size_t i = 0; i < mine; i += half) {
    const size_t n = (mine - i < (size_t)half) ? mine - i : half;
    for (size_t j = i; j < i + n; ++j) {
      const unsigned bar = su32(&full[j % ring]);
      const unsigned par = (j / ring) & 1;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(bar),
          "r"(par)
          : "memory");
      acc += reinterpret_cast<const double*>(buf + (j % ring) * chunk)[tid % (chunk / 8)];
    }
    __syncthreads();
    if (tid == 0) issue(i + n + ring);
  }
  if (acc == 12345.678) sink[0] = acc;
}

__device__ bool wait_bounded(unsigned bar, unsigned par, int who, unsigned i) {
  for (long long it = 0; it < (1LL << 26); ++it) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    if (ok) return true;
  }
  printf("timeout block %d who %d i %u par %u\n", blockIdx.x, who, i, par);
  return false;
}

// warp-specialised: warp 0 lane 0 produces (waits `empty`, issues), the
// other warps consume modes round-robin and release each slot on `empty`
__global__ void bulk_ws(const char* __restrict__ src, unsigned n_chunks, int chunk, int ring, double* sink,
                        int work = 0, int lz = 0) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long full[32], empty[32];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, n_cons = blockDim.x / 32 - 1;
  const unsigned mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < ring; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // lz > 0: the m2l_zpipe_kernel order — this CTA's columns b, b + grid, ..., each column's lz modes at a
  // stride of plane = n_chunks / lz chunks; else CTA-interleaved consecutive chunks
  auto chunk_index = [&](unsigned i) -> size_t {
    if (lz == 0) return (size_t)blockIdx.x + (size_t)i * gridDim.x;
    const int l = lz > 0 ? lz : -lz;
    const size_t col = blockIdx.x + (size_t)(i / l) * gridDim.x;
    if (lz < 0) return col * l + i % l;  // column-contiguous layout [column][qz]
    const size_t plane = n_chunks / l;
    return (size_t)(i % l) * plane + col;
  };
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (unsigned i = 0; i < mine; ++i) {
        if (i >= (unsigned)ring) {
          if (!wait_bounded(su32(&empty[s]), ph ^ 1u, -1, i)) return;
        }
        const unsigned bar = su32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(buf + (size_t)s * chunk)), "l"(src + chunk_index(i) * chunk), "r"(chunk), "r"(bar) : "memory");
        if (++s == ring) { s = 0; ph ^= 1u; }
      }
    }
  } else {
  double acc = 0;
  const int cw = warp - 1;
  int s = cw % ring;
  unsigned ph = (cw / ring) & 1;
  for (unsigned i = cw; i < mine; i += n_cons) {
    if (!wait_bounded(su32(&full[s]), ph, cw, i)) break;
    if (work > 0) {  // mode-product-like consumer: a dependent FMA chain over the chunk (25 lanes x 25 terms)
      const double2* blk = reinterpret_cast<const double2*>(buf + (size_t)s * chunk);
      double a0 = 0, a1 = 0;
      for (int c = 0; c < work; ++c) {
        const double2 v = blk[(lane % 25) + 25 * (c % 25)];
        a0 = fma(v.x, a1 + 1.0, a0);
        a1 = fma(v.y, a0, a1);
      }
      acc += a0 + a1;
    } else {
      for (int k = lane; k < chunk / 16; k += 32) acc += reinterpret_cast<const double2*>(buf + (size_t)s * chunk)[k].x;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    s += n_cons;
    while (s >= ring) { s -= ring; ph ^= 1u; }
  }
  if (acc == 12345.678) sink[0] = acc;
  }
  __syncthreads();  // keep the issuing thread alive until every copy landed
}

__global__ void ldg_stream(const double2* __restrict__ src, size_t n, double* sink) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc += src[i].x;
  if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t bytes = 328ull << 20;
  char* src;
  double* sink;
  cudaMalloc(&src, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
  };
  float ms = time([&] { ldg_stream<<<148 * 8, 256>>>((const double2*)src, bytes / 16, sink); });
  printf("ldg_stream  %.1f us  %.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int chunks[] = {10000, 10000, 10000, 10000, 10000, 4096, 16384, 2048};
  int rings[] = {16, 8, 4, 16, 20, 32, 8, 32};
  int ctas[] = {1, 2, 2, 1, 1, 1, 1, 2};
  int modes[] = {1, 1, 1, 0, 1, 1, 1, 1};
  for (int t = 0; t < 8; ++t) {
    const int chunk = chunks[t] / 16 * 16, ring = rings[t], c = ctas[t];
    const size_t smem = (size_t)chunk * ring;
    if (smem * c > 225 * 1024) continue;
    const size_t n_chunks = bytes / chunk;
    ms = time([&] { bulk_ring<<<148 * c, 256 / c * 2, smem>>>(src, n_chunks, chunk, ring, modes[t], sink); });
    printf("bulk chunk=%5d ring=%2d ctas/SM=%d mode=%d  %.1f us  %.0f GB/s\n", chunk, ring, c, modes[t], ms * 1e3,
           n_chunks * chunk / ms / 1e6);
  }
  cudaFuncSetAttribute(bulk_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    bulk_ws<<<148, 544, 159744>>>(src, bytes / 9984, 9984, 16, sink);
    printf("ws single launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    printf("ws single sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  int wchunks[] = {10000, 10000, 10000, 10000, 20000, 10000};
  int wrings[] = {16, 12, 16, 20, 8, 16};
  int wthreads[] = {32 * 17, 32 * 13, 32 * 9, 32 * 11, 32 * 9, 32 * 17};  // n_cons divides ring
  for (int t = 0; t < 6; ++t) {
    const int chunk = wchunks[t] / 16 * 16, ring = wrings[t];
    const size_t smem = (size_t)chunk * ring;
    if (smem > 220 * 1024) continue;
    const unsigned n_chunks = bytes / chunk;
    ms = time([&] { bulk_ws<<<148, wthreads[t], smem>>>(src, n_chunks, chunk, ring, sink); });
    printf("ws   chunk=%5d ring=%2d threads=%d  %.1f us  %.0f GB/s\n", chunk, ring, wthreads[t], ms * 1e3,
           (double)n_chunks * chunk / ms / 1e6);
  }
  for (int work : {25, 50, 100}) {  // 7 consumer warps x 2 slots (ring 14), like m2l_zpipe_kernel's mode warps
    const int chunk = 10000 / 16 * 16, ring = 14;
    const unsigned n_chunks = bytes / chunk;
    ms = time([&] { bulk_ws<<<148, 32 * 8, (size_t)chunk * ring>>>(src, n_chunks, chunk, ring, sink, work); });
    printf("ws+work %3d  chunk=%5d ring=%2d consumers=7  %.1f us  %.0f GB/s\n", work, chunk, ring, ms * 1e3,
           (double)n_chunks * chunk / ms / 1e6);
  }
  for (int lz : {32, 7, -32, -7}) {
    const int chunk = 10000 / 16 * 16, ring = 14;
    const unsigned plane = (lz == 32 || lz == -32 ? 1024 : 3969), n_chunks = plane * (lz > 0 ? lz : -lz);
    if ((size_t)n_chunks * chunk > bytes) continue;
    for (int work : {0, 25}) {
      ms = time([&] { bulk_ws<<<148, 32 * 8, (size_t)chunk * ring>>>(src, n_chunks, chunk, ring, sink, work, lz); });
      printf("ws zpipe-order lz=%3d (%s) work=%2d  %.1f us  %.0f GB/s\n", lz, lz > 0 ? "[qz][col]" : "[col][qz]", work, ms * 1e3,
             (double)n_chunks * chunk / ms / 1e6);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
