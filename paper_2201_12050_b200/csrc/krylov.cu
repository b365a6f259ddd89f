// GMRES vector operations on the device (src/solver.cpp:56-72, 109-112).
//
// All reductions are deterministic: a fixed grid of kRedBlocks blocks strides
// over the vector, each block reduces in a fixed shared-memory tree, and the
// last block to finish (counter) sums the per-block partials in index order.
// The MGS step is fused so that the update w -= h_i v_i and the next
// projection <v_{i+1}, w> (or the norm ||w|| after the last one) are one pass.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpbem_cu {

namespace {

constexpr int RT = 256;

template <typename T>
__device__ __forceinline__ T zero_v();
template <>
__device__ __forceinline__ double zero_v<double>() {
  return 0.0;
}
template <>
__device__ __forceinline__ c64 zero_v<c64>() {
  return cmk(0.0, 0.0);
}
__device__ __forceinline__ double add_v(double a, double b) { return a + b; }
__device__ __forceinline__ c64 add_v(c64 a, c64 b) { return cadd(a, b); }

template <typename T>
__device__ __forceinline__ T block_reduce(T v, T* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = RT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = add_v(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  return sh[0];
}

// publish the block partial; the last block folds all partials in order
template <typename T>
__device__ void finish_reduce(T block_sum, T* partials, unsigned* counter, T* result, T* sh) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_sum;
    __threadfence();
    unsigned done = atomicAdd(counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  T v = zero_v<T>();
  for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += RT) v = add_v(v, partials[i]);
  T total = block_reduce(v, sh);
  if (threadIdx.x == 0) {
    *result = total;
    *counter = 0u;
  }
}

// Grid-stride loops are unrolled by 4 (independent loads in flight); the
// per-thread partial sums are still accumulated in a fixed order.
#define GRID_STRIDE_4(i, n, BODY)                                                        \
  {                                                                                      \
    const long long stride_ = static_cast<long long>(gridDim.x) * RT;                    \
    long long i0_ = blockIdx.x * static_cast<long long>(RT) + threadIdx.x;               \
    for (; i0_ + 3 * stride_ < (n); i0_ += 4 * stride_) {                                \
      _Pragma("unroll") for (int u_ = 0; u_ < 4; ++u_) {                                 \
        const long long i = i0_ + u_ * stride_;                                          \
        BODY                                                                             \
      }                                                                                  \
    }                                                                                    \
    for (long long i = i0_; i < (n); i += stride_) {                                     \
      BODY                                                                               \
    }                                                                                    \
  }

// result = ||w||^2 ; flag |= non-finite entry present
__global__ void __launch_bounds__(RT) sqnorm_kernel(const c64* __restrict__ w, long long n, double* partials,
                                                    unsigned* counter, double* result, int* nonfinite) {
  __shared__ double sh[RT];
  double s = 0.0;
  bool bad = false;
  GRID_STRIDE_4(i, n, {
    c64 v = w[i];
    bad |= !isfinite(v.x) || !isfinite(v.y);
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  })
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  double b = block_reduce(s, sh);
  finish_reduce(b, partials, counter, result, sh);
}

// result = <a, b> = sum conj(a) b
__global__ void __launch_bounds__(RT) dotc_kernel(const c64* __restrict__ a, const c64* __restrict__ b,
                                                  long long n, c64* partials, unsigned* counter, c64* result) {
  __shared__ c64 sh[RT];
  c64 s = cmk(0.0, 0.0);
  GRID_STRIDE_4(i, n, { s = cfma_conj(a[i], b[i], s); })
  c64 t = block_reduce(s, sh);
  finish_reduce(t, partials, counter, result, sh);
}

// w -= (*h) v ; then result = <vn, w> (vn != null) — the fused MGS step
__global__ void __launch_bounds__(RT) axpy_dotc_kernel(c64* __restrict__ w, const c64* __restrict__ v,
                                                       const c64* __restrict__ h, const c64* __restrict__ vn,
                                                       long long n, c64* partials, unsigned* counter,
                                                       c64* result) {
  __shared__ c64 sh[RT];
  const c64 hh = *h;
  c64 s = cmk(0.0, 0.0);
  GRID_STRIDE_4(i, n, {
    c64 wi = csub(w[i], cmul(hh, v[i]));
    w[i] = wi;
    s = cfma_conj(vn[i], wi, s);
  })
  c64 t = block_reduce(s, sh);
  finish_reduce(t, partials, counter, result, sh);
}

// w -= (*h) v ; then result = ||w||^2
__global__ void __launch_bounds__(RT) axpy_sqnorm_kernel(c64* __restrict__ w, const c64* __restrict__ v,
                                                         const c64* __restrict__ h, long long n,
                                                         double* partials, unsigned* counter, double* result) {
  __shared__ double sh[RT];
  const c64 hh = *h;
  double s = 0.0;
  GRID_STRIDE_4(i, n, {
    c64 wi = csub(w[i], cmul(hh, v[i]));
    w[i] = wi;
    s = fma(wi.x, wi.x, s);
    s = fma(wi.y, wi.y, s);
  })
  double t = block_reduce(s, sh);
  finish_reduce(t, partials, counter, result, sh);
}

// out = in / d   (basis.col(j+1) = w / hlast ; v0 = r / rnorm)
__global__ void div_kernel(const c64* __restrict__ in, c64* __restrict__ out, long long n, double d) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    c64 v = in[i];
    out[i] = cmk(v.x / d, v.y / d);
  }
}

// x += sum_i V[:, i] y_i   (x += basis.leftCols(j) * y)
__global__ void update_x_kernel(c64* __restrict__ x, const c64* __restrict__ basis, long long ld,
                                const c64* __restrict__ y, int j, long long n) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    c64 acc = cmk(0.0, 0.0);
    for (int i = 0; i < j; ++i) acc = cfma(basis[static_cast<long long>(i) * ld + k], __ldg(y + i), acc);
    x[k] = cadd(x[k], acc);
  }
}

// r = b - ax ; result = ||r||^2
__global__ void __launch_bounds__(RT) residual_kernel(const c64* __restrict__ b, const c64* __restrict__ ax,
                                                      c64* __restrict__ r, long long n, double* partials,
                                                      unsigned* counter, double* result) {
  __shared__ double sh[RT];
  double s = 0.0;
  GRID_STRIDE_4(i, n, {
    c64 v = csub(b[i], ax[i]);
    r[i] = v;
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  })
  double t = block_reduce(s, sh);
  finish_reduce(t, partials, counter, result, sh);
}

// ---------------------------------------------------------------------------
// Classical Gram-Schmidt passes of the distributed GMRES (gmres_dist.cu): one
// pass is a batched projection h = V^H w (+ ||w||^2 and a non-finite count)
// followed, after the all-reduce of h over the ranks, by w -= V h (+ the new
// ||w||^2). Each thread keeps kCgsR entries of w in registers and streams the
// basis columns past them; per-column sums go warp -> shared memory -> block
// partial -> the last block folds the partials in block order (deterministic).
constexpr int kCgsR = 4;
constexpr int kCgsWarps = RT / 32;

__device__ __forceinline__ c64 warp_sum_c(c64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// out[i] = <V_i, w> (i < cols); out[cols] = (||w||^2, number of non-finite entries of w)
__global__ void __launch_bounds__(RT) cgs_dots_kernel(const c64* __restrict__ V, long long ld, int cols,
                                                      const c64* __restrict__ w, long long n,
                                                      c64* __restrict__ partials, unsigned* counter,
                                                      c64* __restrict__ out) {
  extern __shared__ c64 acc[];  // [cols + 1][kCgsWarps]
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (cols + 1) * kCgsWarps; i += RT) acc[i] = cmk(0.0, 0.0);
  __syncthreads();
  c64 nrm = cmk(0.0, 0.0);
  const long long tile = static_cast<long long>(RT) * kCgsR;
  for (long long t0 = blockIdx.x * tile; t0 < n; t0 += static_cast<long long>(gridDim.x) * tile) {
    c64 wr[kCgsR];
#pragma unroll
    for (int u = 0; u < kCgsR; ++u) {
      const long long k = t0 + u * RT + threadIdx.x;
      wr[u] = k < n ? w[k] : cmk(0.0, 0.0);
      nrm.x = fma(wr[u].x, wr[u].x, nrm.x);
      nrm.x = fma(wr[u].y, wr[u].y, nrm.x);
      if (!isfinite(wr[u].x) || !isfinite(wr[u].y)) nrm.y += 1.0;
    }
    for (int i = 0; i < cols; ++i) {
      const c64* v = V + static_cast<long long>(i) * ld;
      c64 sum = cmk(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < kCgsR; ++u) {
        const long long k = t0 + u * RT + threadIdx.x;
        if (k < n) sum = cfma_conj(v[k], wr[u], sum);
      }
      sum = warp_sum_c(sum);
      if (lane == 0) acc[i * kCgsWarps + warp] = cadd(acc[i * kCgsWarps + warp], sum);
    }
  }
  nrm = warp_sum_c(nrm);
  if (lane == 0) acc[cols * kCgsWarps + warp] = cadd(acc[cols * kCgsWarps + warp], nrm);
  __syncthreads();
  for (int i = threadIdx.x; i <= cols; i += RT) {
    c64 sum = cmk(0.0, 0.0);
    for (int q = 0; q < kCgsWarps; ++q) sum = cadd(sum, acc[i * kCgsWarps + q]);
    partials[static_cast<long long>(i) * gridDim.x + blockIdx.x] = sum;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i <= cols; i += RT) {
    c64 sum = cmk(0.0, 0.0);
    for (unsigned q = 0; q < gridDim.x; ++q) sum = cadd(sum, __ldcg(partials + static_cast<long long>(i) * gridDim.x + q));
    out[i] = sum;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// w -= sum_i h_i V_i (in column order, as the reference's MGS subtracts);
// result = ||w||^2
__global__ void __launch_bounds__(RT) cgs_update_kernel(c64* __restrict__ w, const c64* __restrict__ V, long long ld,
                                                        int cols, const c64* __restrict__ h, long long n,
                                                        double* partials, unsigned* counter, double* result) {
  __shared__ double sh[RT];
  double nrm = 0.0;
  const long long tile = static_cast<long long>(RT) * kCgsR;
  for (long long t0 = blockIdx.x * tile; t0 < n; t0 += static_cast<long long>(gridDim.x) * tile) {
    c64 wr[kCgsR];
#pragma unroll
    for (int u = 0; u < kCgsR; ++u) {
      const long long k = t0 + u * RT + threadIdx.x;
      wr[u] = k < n ? w[k] : cmk(0.0, 0.0);
    }
    for (int i = 0; i < cols; ++i) {
      const c64 hi = __ldg(h + i);
      const c64* v = V + static_cast<long long>(i) * ld;
#pragma unroll
      for (int u = 0; u < kCgsR; ++u) {
        const long long k = t0 + u * RT + threadIdx.x;
        if (k < n) wr[u] = csub(wr[u], cmul(hi, v[k]));
      }
    }
#pragma unroll
    for (int u = 0; u < kCgsR; ++u) {
      const long long k = t0 + u * RT + threadIdx.x;
      if (k < n) {
        w[k] = wr[u];
        nrm = fma(wr[u].x, wr[u].x, nrm);
        nrm = fma(wr[u].y, wr[u].y, nrm);
      }
    }
  }
  const double t = block_reduce(nrm, sh);
  finish_reduce(t, partials, counter, result, sh);
}

// ---------------------------------------------------------------------------
// Fused modified Gram-Schmidt of one Arnoldi step in a single cooperative
// launch: ||w||^2 (+ non-finite flag), then for i = 0..j
//   h_i = <v_i, w>;  w -= h_i v_i          (src/solver.cpp:58-62, same order)
// and finally ||w||^2. One block of kMgsThreads per SM keeps its contiguous
// chunk of w in shared memory for the whole sequence; each thread owns the
// chunk elements e = tid + k kMgsThreads and holds its slice of v_i in
// registers: the pass that applies h_i v_i reads v_{i+1} for the next dot and
// keeps it, so every basis vector is streamed from HBM exactly once per step
// (the previous kernel re-read v_i). Block partials use a fixed shuffle
// tree, and every block folds all block partials in index order, so h_i is
// bitwise identical everywhere and run to run.
constexpr int kMgsThreads = 512;
constexpr int kMgsK = 18;  // elements per thread (N <= 148 x 9216)
constexpr long long kMgsMaxChunk = static_cast<long long>(kMgsThreads) * kMgsK;  // 147 KB of w per block

__device__ __forceinline__ double warp_sum(double v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ c64 warp_sum(c64 v) {
  for (int off = 16; off > 0; off >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, off);
    v.y += __shfl_down_sync(0xffffffffu, v.y, off);
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T block_sum_mgs(T v, T* sh) {  // result valid in thread 0
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T t = zero_v<T>();
  if (threadIdx.x < 32) {
    t = threadIdx.x < kMgsThreads / 32 ? sh[threadIdx.x] : zero_v<T>();
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// bulk prefetch of `count` complex values into L2 (no registers, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const c64* p, int count) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(static_cast<unsigned>(count * sizeof(c64)))
               : "memory");
}

__global__ void __launch_bounds__(kMgsThreads, 1)
mgs_fused_kernel(c64* __restrict__ w, const c64* __restrict__ V, long long ld, int j, long long n, long long chunk,
                 c64* __restrict__ h_out, double* __restrict__ norms, int* __restrict__ nonfinite,
                 c64* __restrict__ part_c, double* __restrict__ part_d, int do_pre, c64* __restrict__ hc_out) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  c64* ws = reinterpret_cast<c64*>(smem_raw);
  __shared__ c64 shc[32];
  __shared__ double shd[32];
  __shared__ c64 bcast_c;
  __shared__ double bcast_d;
  const int G = gridDim.x, tid = threadIdx.x;
  const long long start = blockIdx.x * chunk;
  const int len = static_cast<int>(max(0LL, min(chunk, n - start)));
  for (int e = tid; e < len; e += kMgsThreads) ws[e] = w[start + e];
  __syncthreads();

  auto fold_d = [&](double v, double* slot) -> double {  // block partial -> grid total
    const double b = block_sum_mgs(v, shd);
    if (tid == 0) slot[blockIdx.x] = b;
    grid.sync();
    if (tid < 32) {
      double acc = 0.0;
      for (int i = tid; i < G; i += 32) acc += slot[i];
      acc = warp_sum(acc);
      if (tid == 0) bcast_d = acc;
    }
    __syncthreads();
    return bcast_d;
  };
  auto fold_c = [&](c64 partial, int i) -> c64 {
    const c64 b = block_sum_mgs(partial, shc);
    c64* slot = part_c + (i & 1) * G;
    if (tid == 0) slot[blockIdx.x] = b;
    grid.sync();
    if (tid < 32) {
      c64 acc = cmk(0.0, 0.0);
      for (int q = tid; q < G; q += 32) acc = cadd(acc, slot[q]);
      acc = warp_sum(acc);
      if (tid == 0) bcast_c = acc;
    }
    __syncthreads();
    return bcast_c;
  };

  double pre = 0.0;
  if (do_pre) {
    double s = 0.0;
    bool bad = false;
    for (int e = tid; e < len; e += kMgsThreads) {
      const c64 v = ws[e];
      bad |= !isfinite(v.x) || !isfinite(v.y);
      s = fma(v.x, v.x, s);
      s = fma(v.y, v.y, s);
    }
    if (bad) atomicOr(nonfinite, 1);
    pre = fold_d(s, part_d);
    if (blockIdx.x == 0 && tid == 0) norms[0] = pre;
  }

  // one MGS pass over v_0..v_j on the chunk in shared memory: projections to
  // hout[0..j], returns ||w||^2 after the pass
  auto pass = [&](c64* __restrict__ hout) -> double {
    c64 vc[kMgsK];  // this thread's slice of v_i
    {
      const c64* v = V + start;
#pragma unroll
      for (int k = 0; k < kMgsK; ++k) {
        const int e = tid + k * kMgsThreads;
        vc[k] = e < len ? v[e] : cmk(0.0, 0.0);
      }
    }
    c64 s = cmk(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kMgsK; ++k) {
      const int e = tid + k * kMgsThreads;
      if (e < len) s = cfma_conj(vc[k], ws[e], s);
    }
    if (tid == 0 && j >= 1 && len > 0) prefetch_l2(V + ld + start, len);
    c64 h = fold_c(s, 0);
    if (blockIdx.x == 0 && tid == 0) hout[0] = h;
    for (int i = 0; i < j; ++i) {
      // w -= h_i v_i (v_i from registers) and the partial <v_{i+1}, w> in one pass;
      // v_{i+1} is read from HBM once and stays in registers for the next step
      const c64* v = V + static_cast<long long>(i + 1) * ld + start;
      // v_{i+2}'s chunk is pulled into L2 while this pass and the grid-wide fold
      // of h_{i+1} run, so the next pass's loads hit L2 instead of waiting on HBM
      if (tid == 0 && i + 2 <= j && len > 0) prefetch_l2(V + static_cast<long long>(i + 2) * ld + start, len);
      s = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < kMgsK; ++k) {
        const int e = tid + k * kMgsThreads;
        if (e < len) {
          const c64 nx = v[e];
          const c64 wv = csub(ws[e], cmul(h, vc[k]));
          ws[e] = wv;
          s = cfma_conj(nx, wv, s);
          vc[k] = nx;
        }
      }
      h = fold_c(s, i + 1);
      if (blockIdx.x == 0 && tid == 0) hout[i + 1] = h;
    }
    double q = 0.0;  // the last update, w -= h_j v_j, then ||w||^2
#pragma unroll
    for (int k = 0; k < kMgsK; ++k) {
      const int e = tid + k * kMgsThreads;
      if (e < len) {
        const c64 wv = csub(ws[e], cmul(h, vc[k]));
        q = fma(wv.x, wv.x, q);
        q = fma(wv.y, wv.y, q);
        ws[e] = wv;
      }
    }
    return fold_d(q, part_d + G);
  };

  const double post = pass(h_out);
  if (blockIdx.x == 0 && tid == 0) norms[1] = post;
  if (hc_out) {
    // the whole Arnoldi step (src/solver.cpp:58-73): the conditional second pass
    // when ||w|| < 0.5 ||w||_pre (the same arithmetic as a second launch on the
    // written-back w), then h_{j+1,j} = ||w|| and w / h_{j+1,j} (as div_kernel)
    double wn2 = post;
    const bool reorth = sqrt(post) < 0.5 * sqrt(pre);
    if (reorth) wn2 = pass(hc_out);
    const double hl = sqrt(wn2);
    if (blockIdx.x == 0 && tid == 0) {
      norms[2] = wn2;
      norms[4] = reorth ? 1.0 : 0.0;
      norms[5] = hl;
    }
    if (hl > 0.0)
      for (int e = tid; e < len; e += kMgsThreads) ws[e] = cmk(ws[e].x / hl, ws[e].y / hl);
    __syncthreads();
  }
  for (int e = tid; e < len; e += kMgsThreads) w[start + e] = ws[e];
}

// ---------------------------------------------------------------------------
// Batched (lockstep multi-RHS) variants: blockIdx.y = right-hand side r, the
// vectors of RHS r at base + r * ld; per-RHS deterministic reductions
// (partials[r * gridDim.x + b], counter[r]); RHS with mask[r] == 0 are skipped.

template <typename T>
__device__ void finish_reduce_b(T block_sum, T* partials, unsigned* counter, T* result, T* sh) {
  __shared__ bool last;
  const int r = blockIdx.y;
  if (threadIdx.x == 0) {
    partials[r * gridDim.x + blockIdx.x] = block_sum;
    __threadfence();
    const unsigned done = atomicAdd(counter + r, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  T v = zero_v<T>();
  for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += RT) v = add_v(v, partials[r * gridDim.x + i]);
  T total = block_reduce(v, sh);
  if (threadIdx.x == 0) {
    result[r] = total;
    counter[r] = 0u;
  }
}

#define RHS_GUARD()                       \
  const int r_ = blockIdx.y;              \
  if (mask && !mask[r_]) return;          \
  const long long off_ = r_ * ld;

__global__ void __launch_bounds__(RT) b_sqnorm_kernel(const c64* __restrict__ w, long long ld, long long n,
                                                      const int* __restrict__ mask, double* partials,
                                                      unsigned* counter, double* result, int* nonfinite) {
  RHS_GUARD();
  __shared__ double sh[RT];
  double s = 0.0;
  bool bad = false;
  const c64* wr = w + off_;
  GRID_STRIDE_4(i, n, {
    c64 v = wr[i];
    bad |= !isfinite(v.x) || !isfinite(v.y);
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  })
  if (bad && nonfinite) atomicOr(nonfinite + r_, 1);
  double b = block_reduce(s, sh);
  finish_reduce_b(b, partials, counter, result, sh);
}

__global__ void __launch_bounds__(RT) b_dotc_kernel(const c64* __restrict__ a, const c64* __restrict__ b, long long ld,
                                                    long long n, const int* __restrict__ mask, c64* partials,
                                                    unsigned* counter, c64* result) {
  RHS_GUARD();
  __shared__ c64 sh[RT];
  c64 s = cmk(0.0, 0.0);
  const c64* ar = a + off_;
  const c64* br = b + off_;
  GRID_STRIDE_4(i, n, { s = cfma_conj(ar[i], br[i], s); })
  c64 t = block_reduce(s, sh);
  finish_reduce_b(t, partials, counter, result, sh);
}

// w_r -= h[r] v_r ; result[r] = <vn_r, w_r>  (vn == null: result[r] = ||w_r||^2 into dres)
__global__ void __launch_bounds__(RT) b_axpy_dotc_kernel(c64* __restrict__ w, const c64* __restrict__ v,
                                                         const c64* __restrict__ h, const c64* __restrict__ vn,
                                                         long long ld, long long n, const int* __restrict__ mask,
                                                         c64* partials, unsigned* counter, c64* result) {
  RHS_GUARD();
  __shared__ c64 sh[RT];
  const c64 hh = h[r_];
  c64 s = cmk(0.0, 0.0);
  c64* wr = w + off_;
  const c64* vr = v + off_;
  const c64* vnr = vn + off_;
  GRID_STRIDE_4(i, n, {
    c64 wi = csub(wr[i], cmul(hh, vr[i]));
    wr[i] = wi;
    s = cfma_conj(vnr[i], wi, s);
  })
  c64 t = block_reduce(s, sh);
  finish_reduce_b(t, partials, counter, result, sh);
}

__global__ void __launch_bounds__(RT) b_axpy_sqnorm_kernel(c64* __restrict__ w, const c64* __restrict__ v,
                                                           const c64* __restrict__ h, long long ld, long long n,
                                                           const int* __restrict__ mask, double* partials,
                                                           unsigned* counter, double* result) {
  RHS_GUARD();
  __shared__ double sh[RT];
  const c64 hh = h[r_];
  double s = 0.0;
  c64* wr = w + off_;
  const c64* vr = v + off_;
  GRID_STRIDE_4(i, n, {
    c64 wi = csub(wr[i], cmul(hh, vr[i]));
    wr[i] = wi;
    s = fma(wi.x, wi.x, s);
    s = fma(wi.y, wi.y, s);
  })
  double t = block_reduce(s, sh);
  finish_reduce_b(t, partials, counter, result, sh);
}

// out_r = in_r / d[r]
__global__ void b_div_kernel(const c64* __restrict__ in, c64* __restrict__ out, long long ld, long long n,
                             const int* __restrict__ mask, const double* __restrict__ d) {
  RHS_GUARD();
  const double dr = d[r_];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const c64 v = in[off_ + i];
    out[off_ + i] = cmk(v.x / dr, v.y / dr);
  }
}

// x_r += sum_{i < jr[r]} V[i][r] y[r][i]; V column i of RHS r at basis + (i * G + r) * n
__global__ void b_update_x_kernel(c64* __restrict__ x, const c64* __restrict__ basis, int G, long long ld,
                                  const c64* __restrict__ y, int ystride, const int* __restrict__ jr, long long n,
                                  const int* __restrict__ mask) {
  RHS_GUARD();
  const int j = jr[r_];
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    c64 acc = cmk(0.0, 0.0);
    for (int i = 0; i < j; ++i)
      acc = cfma(basis[(static_cast<long long>(i) * G + r_) * ld + k], __ldg(y + r_ * ystride + i), acc);
    x[off_ + k] = cadd(x[off_ + k], acc);
  }
}

// r_r = b_r - ax_r ; result[r] = ||r_r||^2 (+ non-finite flag of ax_r)
__global__ void __launch_bounds__(RT) b_residual_kernel(const c64* __restrict__ b, const c64* __restrict__ ax,
                                                        c64* __restrict__ res, long long ld, long long n,
                                                        const int* __restrict__ mask, double* partials,
                                                        unsigned* counter, double* result, int* nonfinite) {
  RHS_GUARD();
  __shared__ double sh[RT];
  double s = 0.0;
  bool bad = false;
  GRID_STRIDE_4(i, n, {
    const c64 a = ax[off_ + i];
    bad |= !isfinite(a.x) || !isfinite(a.y);
    c64 v = csub(b[off_ + i], a);
    res[off_ + i] = v;
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  })
  if (bad && nonfinite) atomicOr(nonfinite + r_, 1);
  double t = block_reduce(s, sh);
  finish_reduce_b(t, partials, counter, result, sh);
}

// dst[q] = src[idx[q]] (gather = 1) or dst[idx[q]] = src[q] (gather = 0), vectors of length n
__global__ void b_pack_kernel(const c64* __restrict__ src, c64* __restrict__ dst, const int* __restrict__ idx,
                              long long n, int gather) {
  const int q = blockIdx.y;
  const long long from = (gather ? idx[q] : q) * n, to = (gather ? q : idx[q]) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[to + i] = src[from + i];
}

int b_grid(long long n) {  // blocks per RHS
  long long blocks = (n + 4 * 256 - 1) / (4 * 256);
  if (blocks > 64) blocks = 64;
  return static_cast<int>(blocks < 1 ? 1 : blocks);
}

int ew_grid(long long n) {
  long long blocks = (n + 255) / 256;
  const long long cap = static_cast<long long>(kNumSMs) * 8;
  if (blocks > cap) blocks = cap;
  return static_cast<int>(blocks < 1 ? 1 : blocks);
}

}  // namespace

cudaError_t launch_sqnorm(const c64* w, long long n, const RedScratch& rs, double* result, int* nonfinite,
                          cudaStream_t s) {
  sqnorm_kernel<<<kRedBlocks, RT, 0, s>>>(w, n, rs.partial_d, rs.counter, result, nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_dotc(const c64* a, const c64* b, long long n, const RedScratch& rs, c64* result,
                        cudaStream_t s) {
  dotc_kernel<<<kRedBlocks, RT, 0, s>>>(a, b, n, rs.partial_c, rs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_axpy_dotc(c64* w, const c64* v, const c64* h, const c64* vn, long long n, const RedScratch& rs,
                             c64* result, cudaStream_t s) {
  axpy_dotc_kernel<<<kRedBlocks, RT, 0, s>>>(w, v, h, vn, n, rs.partial_c, rs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_axpy_sqnorm(c64* w, const c64* v, const c64* h, long long n, const RedScratch& rs,
                               double* result, cudaStream_t s) {
  axpy_sqnorm_kernel<<<kRedBlocks, RT, 0, s>>>(w, v, h, n, rs.partial_d, rs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_div(const c64* in, c64* out, long long n, double d, cudaStream_t s) {
  div_kernel<<<ew_grid(n), 256, 0, s>>>(in, out, n, d);
  return cudaGetLastError();
}
cudaError_t launch_update_x(c64* x, const c64* basis, long long ld, const c64* y, int j, long long n,
                            cudaStream_t s) {
  update_x_kernel<<<ew_grid(n), 256, 0, s>>>(x, basis, ld, y, j, n);
  return cudaGetLastError();
}
namespace {
}

cudaError_t launch_b_sqnorm(const c64* w, long long ld, long long n, int G, const int* mask, const BatchScratch& bs,
                            double* result, int* nonfinite, cudaStream_t s) {
  b_sqnorm_kernel<<<dim3(b_grid(n), G), RT, 0, s>>>(w, ld, n, mask, bs.partial_d, bs.counter, result, nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_b_dotc(const c64* a, const c64* b, long long ld, long long n, int G, const int* mask,
                          const BatchScratch& bs, c64* result, cudaStream_t s) {
  b_dotc_kernel<<<dim3(b_grid(n), G), RT, 0, s>>>(a, b, ld, n, mask, bs.partial_c, bs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_b_axpy_dotc(c64* w, const c64* v, const c64* h, const c64* vn, long long ld, long long n, int G,
                               const int* mask, const BatchScratch& bs, c64* result, cudaStream_t s) {
  b_axpy_dotc_kernel<<<dim3(b_grid(n), G), RT, 0, s>>>(w, v, h, vn, ld, n, mask, bs.partial_c, bs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_b_axpy_sqnorm(c64* w, const c64* v, const c64* h, long long ld, long long n, int G,
                                 const int* mask, const BatchScratch& bs, double* result, cudaStream_t s) {
  b_axpy_sqnorm_kernel<<<dim3(b_grid(n), G), RT, 0, s>>>(w, v, h, ld, n, mask, bs.partial_d, bs.counter, result);
  return cudaGetLastError();
}
cudaError_t launch_b_div(const c64* in, c64* out, long long ld, long long n, int G, const int* mask, const double* d,
                         cudaStream_t s) {
  b_div_kernel<<<dim3(b_grid(n), G), 256, 0, s>>>(in, out, ld, n, mask, d);
  return cudaGetLastError();
}
cudaError_t launch_b_update_x(c64* x, const c64* basis, int G, long long ld, const c64* y, int ystride,
                              const int* jr, long long n, const int* mask, cudaStream_t s) {
  b_update_x_kernel<<<dim3(b_grid(n), G), 256, 0, s>>>(x, basis, G, ld, y, ystride, jr, n, mask);
  return cudaGetLastError();
}
cudaError_t launch_b_residual(const c64* b, const c64* ax, c64* res, long long ld, long long n, int G, const int* mask,
                              const BatchScratch& bs, double* result, int* nonfinite, cudaStream_t s) {
  b_residual_kernel<<<dim3(b_grid(n), G), RT, 0, s>>>(b, ax, res, ld, n, mask, bs.partial_d, bs.counter, result,
                                                      nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_b_pack(const c64* src, c64* dst, const int* idx, int count, long long n, bool gather,
                          cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  b_pack_kernel<<<dim3(b_grid(n), count), 256, 0, s>>>(src, dst, idx, n, gather ? 1 : 0);
  return cudaGetLastError();
}

// the cooperative grid needs every block co-resident: at most one per SM of the
// current device, and the occupancy calculator must agree at the largest chunk
bool mgs_fused_supported(long long n) {
  static std::atomic<unsigned long long> configured{0};
  if (ensure_max_smem(configured, reinterpret_cast<const void*>(&mgs_fused_kernel),
                      static_cast<int>(kMgsMaxChunk * sizeof(c64))) != cudaSuccess)
    return false;
  const int sms = device_sms();
  if (n > static_cast<long long>(sms) * kMgsMaxChunk) return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgs_fused_kernel, kMgsThreads,
                                                    kMgsMaxChunk * sizeof(c64)) != cudaSuccess)
    return false;
  return per_sm >= 1;
}

cudaError_t launch_mgs_fused(c64* w, const c64* V, long long ld, int j, long long n, c64* h_out, double* norms,
                             int* nonfinite, const RedScratch& rs, bool do_pre, cudaStream_t s, c64* hc_out) {
  // cooperative launch: every block co-resident (one per SM)
  static const long long per_block = [] {  // elements per block before using more SMs (FPBEM_MGS_PER_BLOCK, A/B)
    const char* v = std::getenv("FPBEM_MGS_PER_BLOCK");
    return v ? std::max(1LL, std::atoll(v)) : 1024LL;
  }();
  long long blocks = (n + per_block - 1) / per_block;
  if (blocks > device_sms()) blocks = device_sms();
  if (blocks < 1) blocks = 1;
  long long chunk = (n + blocks - 1) / blocks;
  if (chunk > kMgsMaxChunk) return cudaErrorInvalidValue;
  size_t smem = static_cast<size_t>(chunk) * sizeof(c64);
  static std::atomic<unsigned long long> configured{0};
  cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&mgs_fused_kernel),
                                  static_cast<int>(kMgsMaxChunk * sizeof(c64)));
  if (e != cudaSuccess) return e;
  int pre = do_pre ? 1 : 0;
  c64* pc = rs.partial_c;
  double* pd = rs.partial_d;
  void* args[] = {&w, const_cast<c64**>(&V), &ld, &j, &n, &chunk, &h_out, &norms, &nonfinite, &pc, &pd, &pre, &hc_out};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&mgs_fused_kernel), dim3(static_cast<unsigned>(blocks)),
                                     dim3(kMgsThreads), args, smem, s);
}

int cgs_blocks(long long n) {
  const long long tiles = (n + RT * kCgsR - 1) / (RT * kCgsR);
  return static_cast<int>(tiles < 1 ? 1 : (tiles > kCgsMaxBlocks ? kCgsMaxBlocks : tiles));
}

cudaError_t launch_cgs_dots(const c64* V, long long ld, int cols, const c64* w, long long n, c64* partials,
                            unsigned* counter, c64* out, cudaStream_t s) {
  if (cols < 0 || cols >= kCgsMaxCols) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(cols + 1) * kCgsWarps * sizeof(c64);
  static std::atomic<unsigned long long> configured{0};
  if (smem > 48 * 1024) {
    const size_t cap = static_cast<size_t>(kCgsMaxCols) * kCgsWarps * sizeof(c64);
    cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&cgs_dots_kernel),
                                    static_cast<int>(cap));
    if (e != cudaSuccess) return e;
  }
  cgs_dots_kernel<<<cgs_blocks(n), RT, smem, s>>>(V, ld, cols, w, n, partials, counter, out);
  return cudaGetLastError();
}

cudaError_t launch_cgs_update(c64* w, const c64* V, long long ld, int cols, const c64* h, long long n,
                              double* partials, unsigned* counter, double* result, cudaStream_t s) {
  cgs_update_kernel<<<cgs_blocks(n), RT, 0, s>>>(w, V, ld, cols, h, n, partials, counter, result);
  return cudaGetLastError();
}

cudaError_t launch_residual(const c64* b, const c64* ax, c64* r, long long n, const RedScratch& rs,
                            double* result, cudaStream_t s) {
  residual_kernel<<<kRedBlocks, RT, 0, s>>>(b, ax, r, n, rs.partial_d, rs.counter, result);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
