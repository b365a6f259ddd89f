// GMRES vector operations on the device (src/solver.cpp:56-72, 109-112).
//
// All reductions are deterministic: a fixed grid of kRedBlocks blocks strides
// over the vector, each block reduces in a fixed shared-memory tree, and the
// last block to finish (counter) sums the per-block partials in index order.
// The MGS step is fused so that the update w -= h_i v_i and the next
// projection <v_{i+1}, w> (or the norm ||w|| after the last one) are one pass.
#include "common.cuh"
#include "kernels.cuh"

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

// result = ||w||^2 ; flag |= non-finite entry present
__global__ void __launch_bounds__(RT) sqnorm_kernel(const c64* __restrict__ w, long long n, double* partials,
                                                    unsigned* counter, double* result, int* nonfinite) {
  __shared__ double sh[RT];
  double s = 0.0;
  bool bad = false;
  for (long long i = blockIdx.x * static_cast<long long>(RT) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * RT) {
    c64 v = w[i];
    bad |= !isfinite(v.x) || !isfinite(v.y);
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  double b = block_reduce(s, sh);
  finish_reduce(b, partials, counter, result, sh);
}

// result = <a, b> = sum conj(a) b
__global__ void __launch_bounds__(RT) dotc_kernel(const c64* __restrict__ a, const c64* __restrict__ b,
                                                  long long n, c64* partials, unsigned* counter, c64* result) {
  __shared__ c64 sh[RT];
  c64 s = cmk(0.0, 0.0);
  for (long long i = blockIdx.x * static_cast<long long>(RT) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * RT)
    s = cfma_conj(a[i], b[i], s);
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
  for (long long i = blockIdx.x * static_cast<long long>(RT) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * RT) {
    c64 wi = csub(w[i], cmul(hh, v[i]));
    w[i] = wi;
    s = cfma_conj(vn[i], wi, s);
  }
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
  for (long long i = blockIdx.x * static_cast<long long>(RT) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * RT) {
    c64 wi = csub(w[i], cmul(hh, v[i]));
    w[i] = wi;
    s = fma(wi.x, wi.x, s);
    s = fma(wi.y, wi.y, s);
  }
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
  for (long long i = blockIdx.x * static_cast<long long>(RT) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * RT) {
    c64 v = csub(b[i], ax[i]);
    r[i] = v;
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  double t = block_reduce(s, sh);
  finish_reduce(t, partials, counter, result, sh);
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
cudaError_t launch_residual(const c64* b, const c64* ax, c64* r, long long n, const RedScratch& rs,
                            double* result, cudaStream_t s) {
  residual_kernel<<<kRedBlocks, RT, 0, s>>>(b, ax, r, n, rs.partial_d, rs.counter, result);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
