// Far-field M2L as a circulant convolution over the cell lattice, and the
// shared P2M expansion.
//
// Reference: CirculantSpectrum::matvec (src/structured.cpp:122-166) zero-pads
// the cell-major moments into an L_x x L_y x L_z field, runs FFTW forward over
// all b coefficient fields, multiplies every Fourier mode by its b x b block
// Λ_q, runs FFTW backward and keeps the first M cells per axis scaled by 1/q.
// Here the lattice DFT is separable and pruned: the forward pass along an
// axis reads only the M nonzero inputs, the backward pass writes only the M
// kept outputs, so padded zeros are never touched. Each axis pass is a
// streaming kernel over [outer][axis][inner][fields] with the fields
// (nrhs x b, contiguous) innermost, so every warp access is coalesced. The
// per-mode product streams Λ once per apply (the HBM-bound part).
// P2M (src/fmm.cpp:256-259) runs as a job list of the DMMA block GEMM (near_field.cu).
#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {

// out[a][qo][bi][e] = scale * sum_{j < n_in} tw[(j*qo*sign) mod L] * in[a][j][bi][e]
// with tw[k] = exp(-2 pi i k / L); sign = +1 forward, -1 backward (conjugate).
__global__ void dft_axis_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ tw,
                                long long n_a, int n_in, int n_out, long long n_inner, int L, int backward,
                                double scale) {
  const long long total = n_a * n_out * n_inner;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long inner = g % n_inner;
    const long long rest = g / n_inner;
    const int qo = static_cast<int>(rest % n_out);
    const long long a = rest / n_out;
    const c64* src = in + (a * n_in) * n_inner + inner;
    c64 acc = cmk(0.0, 0.0);
    int idx = 0;  // (j * qo) mod L, advanced incrementally
    for (int j = 0; j < n_in; ++j) {
      c64 w = tw[idx];
      if (backward) w.y = -w.y;
      acc = cfma(w, src[static_cast<long long>(j) * n_inner], acc);
      idx += qo;
      if (idx >= L) idx -= L;
    }
    out[g] = cscale(acc, scale);
  }
}

// image[q][r][i] = sum_j Λ_q[i + b j] field[q][r][j]; one thread per (q, r, i)
__global__ void mode_product_kernel(const c64* __restrict__ lambda, const c64* __restrict__ field,
                                    c64* __restrict__ image, long long q_total, int b, int nrhs) {
  const long long per_q = static_cast<long long>(nrhs) * b;
  const long long total = q_total * per_q;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = g / per_q;
    const int ri = static_cast<int>(g % per_q);
    const int r = ri / b, i = ri % b;
    const c64* lam = lambda + q * b * b + i;
    const c64* f = field + q * per_q + static_cast<long long>(r) * b;
    c64 acc = cmk(0.0, 0.0);
#pragma unroll 5
    for (int j = 0; j < b; ++j) acc = cfma(__ldg(lam + static_cast<long long>(j) * b), f[j], acc);
    image[g] = acc;
  }
}

// zero the embedded field and place each K_o at slot (o mod L) (src/structured.cpp:73-86)
__global__ void scatter_bank_kernel(const c64* __restrict__ blocks, const int* __restrict__ offsets, int n_blk,
                                    int b2, int lx, int ly, int lz, c64* __restrict__ field) {
  const long long total = static_cast<long long>(n_blk) * b2;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(g / b2);
    const int e = static_cast<int>(g % b2);
    int qx = offsets[3 * s], qy = offsets[3 * s + 1], qz = offsets[3 * s + 2];
    if (qx < 0) qx += lx;
    if (qy < 0) qy += ly;
    if (qz < 0) qz += lz;
    const long long q = (static_cast<long long>(qz) * ly + qy) * lx + qx;
    field[q * b2 + e] = blocks[g];
  }
}

int grid_for(long long total, int threads) {
  long long blocks = (total + threads - 1) / threads;
  const long long cap = static_cast<long long>(kNumSMs) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

}  // namespace

cudaError_t launch_dft_axis(const c64* in, c64* out, const c64* tw, long long n_a, int n_in, int n_out,
                            long long n_inner, int L, bool backward, double scale, cudaStream_t stream) {
  const long long total = n_a * n_out * n_inner;
  if (total == 0) return cudaSuccess;
  dft_axis_kernel<<<grid_for(total, 256), 256, 0, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L,
                                                            backward ? 1 : 0, scale);
  return cudaGetLastError();
}

cudaError_t launch_mode_product(const c64* lambda, const c64* field, c64* image, long long q_total, int b,
                                int nrhs, cudaStream_t stream) {
  const long long total = q_total * b * nrhs;
  mode_product_kernel<<<grid_for(total, 256), 256, 0, stream>>>(lambda, field, image, q_total, b, nrhs);
  return cudaGetLastError();
}

cudaError_t launch_scatter_bank(const c64* blocks, const int* offsets, int n_blk, int b2, int lx, int ly, int lz,
                                c64* field, cudaStream_t stream) {
  const long long total = static_cast<long long>(n_blk) * b2;
  if (total == 0) return cudaSuccess;
  scatter_bank_kernel<<<grid_for(total, 256), 256, 0, stream>>>(blocks, offsets, n_blk, b2, lx, ly, lz, field);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
