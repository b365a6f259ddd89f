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
    int j = 0;
    // batches of 8 independent loads, accumulated in j order
    for (; j + 8 <= n_in; j += 8) {
      c64 v[8], w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = src[static_cast<long long>(j + u) * n_inner];
        w[u] = __ldg(tw + idx);
        idx += qo;
        if (idx >= L) idx -= L;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (backward) w[u].y = -w[u].y;
        acc = cfma(w[u], v[u], acc);
      }
    }
    for (; j < n_in; ++j) {
      c64 w = __ldg(tw + idx);
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

// Last-axis fusion: forward DFT along z (Mz nonzero inputs -> Lz modes), the
// per-mode product with Λ_q, and the pruned inverse along z (Lz modes -> Mz
// kept outputs), for one (qy, qx) column per CTA. The z-extended field never
// touches HBM; Λ is streamed once.
//   in  : F2[iz][plane][E]   (iz < Mz)      out: H2[iz][plane][E] (iz < Mz)
//   E = nrhs * b fields, plane = Ly * Lx columns, lambda[q][b*b], q = qz*plane + column
__global__ void __launch_bounds__(256)
m2l_zfused_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ lambda,
                  const c64* __restrict__ tw, int Mz, int Lz, long long plane, int E, int b, double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  c64* f_in = reinterpret_cast<c64*>(smem_raw);  // Mz x E
  c64* f_z = f_in + Mz * E;                       // Lz x E  (forward along z)
  c64* g_z = f_z + Lz * E;                        // Lz x E  (after the mode product)
  const long long col = blockIdx.x;
  const int tid = threadIdx.x;
  for (int e = tid; e < Mz * E; e += blockDim.x) {
    const int iz = e / E, f = e % E;
    f_in[e] = in[(static_cast<long long>(iz) * plane + col) * E + f];
  }
  __syncthreads();
  for (int e = tid; e < Lz * E; e += blockDim.x) {
    const int qz = e / E, f = e % E;
    c64 acc = cmk(0.0, 0.0);
    int idx = 0;
    for (int iz = 0; iz < Mz; ++iz) {
      acc = cfma(__ldg(tw + idx), f_in[iz * E + f], acc);
      idx += qz;
      if (idx >= Lz) idx -= Lz;
    }
    f_z[e] = acc;
  }
  __syncthreads();
  // mode product: g[qz][r*b + i] = sum_c Λ_q[i + b c] f[qz][r*b + c]; lanes over i read Λ contiguously
  const int nrhs = E / b;
  for (int e = tid; e < Lz * E; e += blockDim.x) {
    const int qz = e / E, ri = e % E;
    const int r = ri / b, i = ri % b;
    const c64* lam = lambda + (static_cast<long long>(qz) * plane + col) * b * b + i;
    const c64* f = f_z + qz * E + r * b;
    c64 acc = cmk(0.0, 0.0);
    int c = 0;
    for (; c + 5 <= b; c += 5) {
      c64 l[5];
#pragma unroll
      for (int u = 0; u < 5; ++u) l[u] = __ldg(lam + static_cast<long long>(c + u) * b);
#pragma unroll
      for (int u = 0; u < 5; ++u) acc = cfma(l[u], f[c + u], acc);
    }
    for (; c < b; ++c) acc = cfma(__ldg(lam + static_cast<long long>(c) * b), f[c], acc);
    g_z[e] = acc;
  }
  (void)nrhs;
  __syncthreads();
  for (int e = tid; e < Mz * E; e += blockDim.x) {
    const int iz = e / E, f = e % E;
    c64 acc = cmk(0.0, 0.0);
    int idx = 0;
    for (int qz = 0; qz < Lz; ++qz) {
      c64 w = __ldg(tw + idx);
      w.y = -w.y;
      acc = cfma(w, g_z[qz * E + f], acc);
      idx += iz;
      if (idx >= Lz) idx -= Lz;
    }
    out[(static_cast<long long>(iz) * plane + col) * E + f] = cscale(acc, scale);
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

// out[cell'] = in[cell] with the cell index reversed along `level`
// (mirror_permute, src/structured.cpp:168-183); E fields per cell
__global__ void mirror_permute_kernel(const c64* __restrict__ in, c64* __restrict__ out, int mx, int my, int mz,
                                      int level, long long E) {
  const long long total = static_cast<long long>(mx) * my * mz * E;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long cell = g / E, f = g % E;
    int c[3] = {static_cast<int>(cell % mx), static_cast<int>((cell / mx) % my), static_cast<int>(cell / (static_cast<long long>(mx) * my))};
    const int m[3] = {mx, my, mz};
    c[level] = m[level] - 1 - c[level];
    const long long from = c[0] + static_cast<long long>(mx) * (c[1] + static_cast<long long>(my) * c[2]);
    out[g] = in[from * E + f];
  }
}

__global__ void add_kernel(c64* __restrict__ acc, const c64* __restrict__ v, long long n) {
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<long long>(gridDim.x) * blockDim.x)
    acc[g] = cadd(acc[g], v[g]);
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

cudaError_t launch_mirror_permute(const c64* in, c64* out, const int counts[3], int level, long long E,
                                  cudaStream_t stream) {
  const long long total = static_cast<long long>(counts[0]) * counts[1] * counts[2] * E;
  mirror_permute_kernel<<<grid_for(total, 256), 256, 0, stream>>>(in, out, counts[0], counts[1], counts[2], level, E);
  return cudaGetLastError();
}

cudaError_t launch_add(c64* acc, const c64* v, long long n, cudaStream_t stream) {
  add_kernel<<<grid_for(n, 256), 256, 0, stream>>>(acc, v, n);
  return cudaGetLastError();
}

size_t m2l_zfused_smem(int Mz, int Lz, int E) { return sizeof(c64) * static_cast<size_t>(Mz + 2 * Lz) * E; }

cudaError_t launch_m2l_zfused(const c64* in, c64* out, const c64* lambda, const c64* tw, int Mz, int Lz,
                              long long plane, int E, int b, double scale, cudaStream_t stream) {
  const size_t smem = m2l_zfused_smem(Mz, Lz, E);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(m2l_zfused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  m2l_zfused_kernel<<<static_cast<unsigned>(plane), 256, smem, stream>>>(in, out, lambda, tw, Mz, Lz, plane, E, b,
                                                                         scale);
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
