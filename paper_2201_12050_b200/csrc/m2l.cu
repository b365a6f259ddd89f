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
// P2M (src/fmm.cpp:256-259) runs as the per-cell DMMA GEMM with V0 resident in
// shared memory (cellwise_gemm_kernel, cellwise.cu), else p2m_kernel below.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {



// out[a][qo][bi][e] = scale * sum_{j < n_in} tw[(j*qo*sign) mod L] * in[a][j][bi][e]
// with tw[k] = exp(-2 pi i k / L); sign = +1 forward, -1 backward (conjugate).
// One thread owns kQG consecutive outputs qo of one (a, inner) column, so each
// input is read once per kQG outputs (not once per output); consecutive
// threads take consecutive inner indices (coalesced loads and stores). Each
// output is still summed in j order.
template <int kQG>
__global__ void __launch_bounds__(256)
dft_axis_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ tw, long long n_a,
                int n_in, int n_out, long long n_inner, int L, int backward, double scale) {
  extern __shared__ __align__(16) unsigned char dft_smem[];
  c64* tw_s = reinterpret_cast<c64*>(dft_smem);  // the L twiddles, conjugated for the backward pass
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    c64 w = tw[k];
    if (backward) w.y = -w.y;
    tw_s[k] = w;
  }
  __syncthreads();
  const int n_grp = (n_out + kQG - 1) / kQG;
  const long long total = n_a * n_grp * n_inner;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long inner = g % n_inner;
    const long long rest = g / n_inner;
    const int q0 = static_cast<int>(rest % n_grp) * kQG;
    const long long a = rest / n_grp;
    const c64* src = in + (a * n_in) * n_inner + inner;
    c64 acc[kQG];
    int idx[kQG], step[kQG];  // (j * qo) mod L per output, advanced incrementally
#pragma unroll
    for (int o = 0; o < kQG; ++o) {
      acc[o] = cmk(0.0, 0.0);
      idx[o] = 0;
      step[o] = (q0 + o) % L;  // padded outputs (q0 + o >= n_out) may exceed L
    }
    // kB inputs and their twiddles are loaded before the FMAs (latency of the
    // dependent loads otherwise dominates; 8 deep when a thread owns few
    // outputs, e.g. the 256-term lines of a 1 x 256 lattice); zero-padded
    // tail: fma(w, 0, acc) == acc
    constexpr int kB = kQG <= 2 ? 8 : 4;
    for (int j0 = 0; j0 < n_in; j0 += kB) {
      c64 v[kB], w[kQG][kB];
#pragma unroll
      for (int u = 0; u < kB; ++u)
        v[u] = (j0 + u < n_in) ? src[static_cast<long long>(j0 + u) * n_inner] : cmk(0.0, 0.0);
#pragma unroll
      for (int o = 0; o < kQG; ++o)
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          w[o][u] = tw_s[idx[o]];
          idx[o] += step[o];
          if (idx[o] >= L) idx[o] -= L;
        }
#pragma unroll
      for (int u = 0; u < kB; ++u)
#pragma unroll
        for (int o = 0; o < kQG; ++o) acc[o] = cfma(w[o][u], v[u], acc[o]);
    }
    c64* dst = out + (a * n_out + q0) * n_inner + inner;
#pragma unroll
    for (int o = 0; o < kQG; ++o)
      if (q0 + o < n_out) dst[static_cast<long long>(o) * n_inner] = cscale(acc[o], scale);
  }
}

// x and y lattice DFTs of one z-plane and one field in shared memory (the two
// per-axis passes fused; pruned as they are).
//   forward : in = moments [iz][iy][ix][E] (iy < My, ix < Mx)
//             X[iy][qx] = sum_ix Wx[qx][ix] in[iy][ix]            (all My x Lx)
//             out[iz][qy][qx][E] = sum_iy Wy[qy][iy] X[iy][qx]     (this CTA's qy range)
//   inverse : in = [iz][qy][qx][E] (all Ly x Lx)
//             Y[iy][qx] = sum_qy conj Wy[qy][iy] in[qy][qx]        (this CTA's iy range)
//             out[iz][iy][ix][E] = scale sum_qx conj Wx[qx][ix] Y[iy][qx]
// with W[q][j] = exp(-2 pi i (j q mod L) / L) expanded once per CTA into
// shared matrices (odd row pitch), and both phases run as small complex GEMMs
// on the FP64 tensor cores (DMMA m8n8k4, Gauss 3M): two fragment loads per
// three MMAs instead of two shared loads per complex FMA, which made the
// DFMA version shared-memory bound. CTA (iz * E + e, part): the second
// (forward) or first (inverse) phase is split over `parts` CTAs to fill the GPU.
__device__ __forceinline__ int odd_pitch(int n) { return n | 1; }

template <bool kInverse>
__global__ void __launch_bounds__(256)
xy_plane_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ twx,
                const c64* __restrict__ twy, int Mx, int My, int Lx, int Ly, int E, int parts, double scale) {
  extern __shared__ __align__(16) unsigned char xy_smem[];
  // matrices indexed [output index][summation index]
  //   forward: A1 = Wx (Lx x Mx), A2 = Wy (Ly x My); inverse: A1 = conj Wy^T (My x Ly), A2 = conj Wx^T (Mx x Lx)
  const int r1 = kInverse ? My : Lx, c1 = kInverse ? Ly : Mx, L1 = kInverse ? Ly : Lx;
  const int r2 = kInverse ? Mx : Ly, c2 = kInverse ? Lx : My, L2 = kInverse ? Lx : Ly;
  const int p1 = odd_pitch(c1), p2 = odd_pitch(c2);
  c64* A1 = reinterpret_cast<c64*>(xy_smem);
  c64* A2 = A1 + r1 * p1;
  c64* a = A2 + r2 * p2;  // input plane: forward My x Mx, inverse Ly x Lx
  const int rows_in = kInverse ? Ly : My, cols_in = kInverse ? Lx : Mx;
  c64* mid = a + rows_in * cols_in;  // forward X (My x Lx); inverse Y (this CTA's iy rows x Lx)
  const int iz = blockIdx.x / E, e = blockIdx.x - iz * E, part = blockIdx.y;
  const c64* t1 = kInverse ? twy : twx;
  const c64* t2 = kInverse ? twx : twy;
  for (int k = threadIdx.x; k < r1 * c1; k += blockDim.x) {
    const int q = k / c1, j = k - q * c1;
    c64 w = t1[(j * q) % L1];
    if (kInverse) w.y = -w.y;
    A1[q * p1 + j] = w;
  }
  for (int k = threadIdx.x; k < r2 * c2; k += blockDim.x) {
    const int q = k / c2, j = k - q * c2;
    c64 w = t2[(j * q) % L2];
    if (kInverse) w.y = -w.y;
    A2[q * p2 + j] = w;
  }
  const long long plane_in = static_cast<long long>(iz) * rows_in * cols_in;
  for (int k = threadIdx.x; k < rows_in * cols_in; k += blockDim.x) a[k] = in[(plane_in + k) * E + e];
  const int split_n = kInverse ? My : Ly;
  const int s0 = static_cast<int>(static_cast<long long>(split_n) * part / parts);
  const int s1 = static_cast<int>(static_cast<long long>(split_n) * (part + 1) / parts);
  __syncthreads();

  // C = A B on the FP64 tensor cores (complex, Gauss 3M as in near_field.cu),
  // 8 x 8 output tiles over the warps, k in steps of 4; out-of-range rows,
  // columns and k are zero-filled
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  auto cgemm = [&](int M, int N, int K, auto a_at, auto b_at, auto store) {
    const int tn_count = (N + 7) / 8, tiles = ((M + 7) / 8) * tn_count;
    for (int t = warp; t < tiles; t += n_warps) {
      const int tm = t / tn_count, tn = t - tm * tn_count;
      double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
      const int am = tm * 8 + fr, bn = tn * 8 + fr;
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int k = k0 + fk;
        const c64 av = (am < M && k < K) ? a_at(am, k) : cmk(0.0, 0.0);
        const c64 bv = (k < K && bn < N) ? b_at(k, bn) : cmk(0.0, 0.0);
        dmma884(t1[0], t1[1], av.x, bv.x);
        dmma884(t2[0], t2[1], av.y, bv.y);
        dmma884(t3[0], t3[1], av.x + av.y, bv.x + bv.y);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = tn * 8 + 2 * fk + j;
        if (am < M && n < N) store(am, n, cmk(t1[j] - t2[j], t3[j] - t1[j] - t2[j]));
      }
    }
  };

  if (!kInverse) {
    // X[iy][qx] = sum_ix in[iy][ix] Wx[qx][ix]      (M = My, N = Lx, K = Mx)
    cgemm(My, Lx, Mx, [&](int m, int k) { return a[m * Mx + k]; }, [&](int k, int n) { return A1[n * p1 + k]; },
          [&](int m, int n, c64 v) { mid[m * Lx + n] = v; });
    __syncthreads();
    // out[qy][qx] = sum_iy Wy[qy][iy] X[iy][qx]     (M = this CTA's qy, N = Lx, K = My)
    cgemm(s1 - s0, Lx, My, [&](int m, int k) { return A2[(s0 + m) * p2 + k]; },
          [&](int k, int n) { return mid[k * Lx + n]; },
          [&](int m, int n, c64 v) { out[((static_cast<long long>(iz) * Ly + s0 + m) * Lx + n) * E + e] = v; });
  } else {
    // Y[iy][qx] = sum_qy conj Wy[qy][iy] in[qy][qx] (M = this CTA's iy, N = Lx, K = Ly)
    cgemm(s1 - s0, Lx, Ly, [&](int m, int k) { return A1[(s0 + m) * p1 + k]; },
          [&](int k, int n) { return a[k * Lx + n]; }, [&](int m, int n, c64 v) { mid[m * Lx + n] = v; });
    __syncthreads();
    // out[iy][ix] = scale sum_qx Y[iy][qx] conj Wx[qx][ix]   (M = this CTA's iy, N = Mx, K = Lx)
    cgemm(s1 - s0, Mx, Lx, [&](int m, int k) { return mid[m * Lx + k]; }, [&](int k, int n) { return A2[n * p2 + k]; },
          [&](int m, int n, c64 v) {
            out[((static_cast<long long>(iz) * My + s0 + m) * Mx + n) * E + e] = cscale(v, scale);
          });
  }
}

// P2M: mom[(cell * nrhs + r) * b + c] = sum_j V0[c][j] x[r * N + cell * n + j]
// (src/fmm.cpp:256-259). CTA (cell * nrhs + r, coefficient group g of 8 CPW):
// warp w carries the coefficients c = 8 CPW g + w + 8 u, u < CPW (independent
// partial sums sharing every x load) over lane-strided j, four j per step with
// all loads issued before the FMAs, reading rows of V0^T (v0t[c * n + j],
// contiguous); fixed-order shuffle reductions. CPW = 4 when there are enough
// (cell, rhs) pairs to fill the GPU, else 1 (more CTAs per cell).
template <int CPW>
__global__ void __launch_bounds__(256)
p2m_kernel(const c64* __restrict__ v0t, const c64* __restrict__ x, c64* __restrict__ mom, int n, int b,
           long long N, int nrhs) {
  const int cr = blockIdx.x;
  const int cell = cr / nrhs, r = cr - cell * nrhs;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.y * 8 * CPW + w;
  const int nc = min(CPW, (b - c0 + 7) / 8);  // this warp's coefficients
  if (nc <= 0) return;
  const c64* xv = x + static_cast<long long>(r) * N + static_cast<long long>(cell) * n;
  const c64* vr = v0t + static_cast<long long>(c0) * n;
  c64 acc[CPW];
#pragma unroll
  for (int u = 0; u < CPW; ++u) acc[u] = cmk(0.0, 0.0);
  int j = lane;
  for (; j + 96 < n; j += 128) {
    c64 xj[4], v[CPW][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) xj[t] = xv[j + 32 * t];
#pragma unroll
    for (int u = 0; u < CPW; ++u)
#pragma unroll
      for (int t = 0; t < 4; ++t)
        v[u][t] = u < nc ? __ldg(vr + static_cast<long long>(8 * u) * n + j + 32 * t) : cmk(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int u = 0; u < CPW; ++u) acc[u] = cfma(v[u][t], xj[t], acc[u]);
  }
  for (; j < n; j += 32) {
    const c64 xj = xv[j];
#pragma unroll
    for (int u = 0; u < CPW; ++u)
      if (u < nc) acc[u] = cfma(__ldg(vr + static_cast<long long>(8 * u) * n + j), xj, acc[u]);
  }
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    c64 t = acc[u];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      t.x += __shfl_xor_sync(0xffffffffu, t.x, off);
      t.y += __shfl_xor_sync(0xffffffffu, t.y, off);
    }
    if (lane == 0 && u < nc) mom[static_cast<long long>(cr) * b + c0 + 8 * u] = t;
  }
}

// The same axis pass as a batched complex GEMM on the FP64 tensor cores:
// per line a, C (n_out x n_inner) = W (n_out x n_in) B (n_in x n_inner) with
// W[q][j] = tw[(j q) mod L] (conjugated backward) and B the line's inputs. One
// warp per (a, 8 consecutive inner indices): the line's inputs for those 8
// columns are loaded once into registers as m8n8k4 B fragments (8 consecutive
// inner values per k row: 128-byte coalesced), then every 8-row block of W runs
// its k steps from fragment-ordered shared memory (conflict-free, expanded once
// per CTA) in the Gauss 3-multiplication form (T1 = Wr Br, T2 = Wi Bi,
// T3 = (Wr + Wi)(Br + Bi); C = (T1 - T2, T3 - T1 - T2)). Each output is a fixed-
// order sum (deterministic). n_in, n_out <= kDftMmaMax.
constexpr int kDftMmaMax = 64;
constexpr int kDftMmaWarps = 4;

// EPI: the L2P of the lattice near field fused into its last inverse pass (the
// x axis: line a = r * cpl + (z My + y), output q = cell x index, inner = row i
// of the cell): out += U0 L_cell (src/fmm.cpp:265-267) as a second small DMMA
// product per tile, C[q][i] += sum_m L[cell(q)][r][m] U0[i][m], unscaled and
// added after the scaled transform (y = S p, then y += U0 L).
struct L2pEpi {
  const c64* u0 = nullptr;   // n x b column-major: u0[m n + i]
  const c64* loc = nullptr;  // [cell][rhs][b]
  int b = 0, nrhs = 1;
  long long cpl = 1;  // lines per right-hand side (My Mz)
};

template <int KTM, bool EPI = false>
__global__ void __launch_bounds__(kDftMmaWarps * 32)
dft_axis_dmma_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ tw, long long n_a,
                     int n_in, int n_out, long long n_inner, int L, int backward, double scale, L2pEpi epi = {}) {
  extern __shared__ __align__(16) unsigned char dmma_smem[];
  pdl_trigger();
  const int MT = (n_out + 7) / 8, KT = (n_in + 3) / 4;
  double* wr = reinterpret_cast<double*>(dmma_smem);  // [mt][kt][lane]
  double* wi = wr + MT * KT * 32;
  double* ws = wi + MT * KT * 32;
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  const long long n_et = (n_inner + 7) / 8, tiles = n_a * n_et;
  // a lone last input (n_in = 4k + 1, e.g. the 17 modes of a 16-cell near lattice)
  // or a lone last output (n_out = 8k + 1) would cost a whole k step / row block of
  // DMMAs for one useful term: it is added with FMAs instead (xcol: the input
  // j = n_in - 1 into every output of the lane; xrow: output n_out - 1 as a sum
  // over the B fragments, reduced across the 4 lanes of a column)
  const bool xcol = n_in % 4 == 1 && n_in > 4;
  const bool xrow = !EPI && !xcol && n_out % 8 == 1 && n_out > 8;
  const int KTd = xcol ? KT - 1 : KT, MTd = xrow ? MT - 1 : MT;
  const long long warp0 = blockIdx.x * static_cast<long long>(kDftMmaWarps) + (threadIdx.x >> 5);
  const long long nwarps = static_cast<long long>(gridDim.x) * kDftMmaWarps;
  // B fragments of the next tile are loaded before the current tile's MMAs
  c64 nb[KTM];
  auto load = [&](long long t) {
    const long long a = t / n_et, col = (t % n_et) * 8 + fr;
    const bool ok = t < tiles && col < n_inner;
    const c64* src = in + a * n_in * n_inner + col;
#pragma unroll
    for (int kt = 0; kt < KTM; ++kt) {
      const int j = kt * 4 + fk;
      nb[kt] = (ok && kt < KTd && j < n_in) ? src[static_cast<long long>(j) * n_inner] : cmk(0.0, 0.0);
    }
  };
  // the first tile's loads are in flight while the twiddle table is expanded (both are
  // L2 round trips of about a microsecond; in series they cost every short pass both)
  pdl_wait();  // `in` is the previous kernel's output, `out` may be its input
  load(warp0);
  for (int e = threadIdx.x; e < MT * KT * 32; e += blockDim.x) {
    const int ln = e & 31, f = e >> 5, kt = f % KT, mt = f / KT;
    const int q = mt * 8 + (ln >> 2), j = kt * 4 + (ln & 3);
    c64 w = cmk(0.0, 0.0);
    if (q < n_out && j < n_in) {
      w = tw[(j * q) % L];
      if (backward) w.y = -w.y;
    }
    wr[e] = w.x;
    wi[e] = w.y;
    ws[e] = w.x + w.y;
  }
  __syncthreads();
  for (long long t = warp0; t < tiles; t += nwarps) {
    double br[KTM], bi[KTM];  // (br + bi is formed at each use: fewer live registers)
#pragma unroll
    for (int kt = 0; kt < KTM; ++kt) {
      br[kt] = nb[kt].x;
      bi[kt] = nb[kt].y;
    }
    const long long a = t / n_et, e0 = (t % n_et) * 8;
    c64 xc[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};  // xcol: input n_in - 1 at the lane's two output columns
    if (xcol)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long c = e0 + 2 * fk + h;
        if (c < n_inner) xc[h] = in[(a * n_in + n_in - 1) * n_inner + c];
      }
    load(t + nwarps);
    c64* dst = out + a * n_out * n_inner;
    constexpr int KB = 8;  // L2P k steps (b <= 32)
    c64 ub[EPI ? KB : 1];  // U0 B fragments of this tile's 8 rows i
    long long lbase = 0;
    int kb_n = 0;
    if constexpr (EPI) {
      kb_n = (epi.b + 3) / 4;
      const long long r = a / epi.cpl, line = a - r * epi.cpl;
      lbase = (line * n_out * epi.nrhs + r) * epi.b;  // loc of cell (line, q = 0), rhs r
      const long long i = e0 + fr;
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        const int m = kb * 4 + fk;
        ub[kb] = (kb < kb_n && m < epi.b && i < n_inner) ? __ldg(epi.u0 + static_cast<long long>(m) * n_inner + i)
                                                         : cmk(0.0, 0.0);
      }
    }
    for (int mt = 0; mt < MTd; mt += 2) {  // two row blocks per pass: independent accumulator chains
      double t1[2][2] = {}, t2[2][2] = {}, t3[2][2] = {};
      const bool two = mt + 1 < MTd;
      c64 la[EPI ? 2 : 1][EPI ? KB : 1];
      if constexpr (EPI) {  // L A fragments: row q = cell, k = coefficient m
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int q = (mt + u) * 8 + fr;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            const int m = kb * 4 + fk;
            la[u][kb] = (kb < kb_n && m < epi.b && q < n_out)
                            ? __ldg(epi.loc + lbase + static_cast<long long>(q) * epi.nrhs * epi.b + m)
                            : cmk(0.0, 0.0);
          }
        }
      }
#pragma unroll
      for (int kt = 0; kt < KTM; ++kt) {
        if (kt < KTd) {
          const int o0 = (mt * KT + kt) * 32 + lane, o1 = o0 + KT * 32;
          dmma884(t1[0][0], t1[0][1], wr[o0], br[kt]);
          dmma884(t2[0][0], t2[0][1], wi[o0], bi[kt]);
          const double bsum = br[kt] + bi[kt];
          dmma884(t3[0][0], t3[0][1], ws[o0], bsum);
          if (two) {
            dmma884(t1[1][0], t1[1][1], wr[o1], br[kt]);
            dmma884(t2[1][0], t2[1][1], wi[o1], bi[kt]);
            dmma884(t3[1][0], t3[1][1], ws[o1], bsum);
          }
        }
      }
      double s1[2][2] = {}, s2[2][2] = {}, s3[2][2] = {};
      if constexpr (EPI) {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          if (kb < kb_n) {
            const double usum = ub[kb].x + ub[kb].y;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              dmma884(s1[u][0], s1[u][1], la[u][kb].x, ub[kb].x);
              dmma884(s2[u][0], s2[u][1], la[u][kb].y, ub[kb].y);
              dmma884(s3[u][0], s3[u][1], la[u][kb].x + la[u][kb].y, usum);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = (mt + u) * 8 + fr;
        if (q >= n_out) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long c = e0 + 2 * fk + h;
          if (c < n_inner) {
            c64 d = cmk(t1[u][h] - t2[u][h], t3[u][h] - t1[u][h] - t2[u][h]);
            if (xcol) {  // + W[q][n_in - 1] x[n_in - 1][c]: W at (row block, last k step, k lane 0)
              const int ow = ((mt + u) * KT + KT - 1) * 32 + fr * 4;
              d = cfma(cmk(wr[ow], wi[ow]), xc[h], d);
            }
            c64 v = cmk(d.x * scale, d.y * scale);
            if constexpr (EPI) v = cadd(v, cmk(s1[u][h] - s2[u][h], s3[u][h] - s1[u][h] - s2[u][h]));
            dst[static_cast<long long>(q) * n_inner + c] = v;
          }
        }
      }
    }
    if (xrow) {  // output n_out - 1 = 8 (MT - 1): row 0 of the last row block of W, column fr
      c64 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int kt = 0; kt < KTM; ++kt)
        if (kt < KTd) {
          const int ow = ((MT - 1) * KT + kt) * 32 + fk;
          acc = cfma(cmk(wr[ow], wi[ow]), cmk(br[kt], bi[kt]), acc);
        }
      // fixed tree over the column's four k lanes (deterministic)
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
      const long long c = e0 + fr;
      if (fk == 0 && c < n_inner) dst[static_cast<long long>(n_out - 1) * n_inner + c] = cmk(acc.x * scale, acc.y * scale);
    }
  }
}

// Long lines with few outputs (e.g. the 256 -> 512 line of a 1 x 256 lattice):
// one warp per output (a, qo, inner); lane l sums the terms j = l, l + 32, ...
// then a fixed shuffle tree combines the lanes (deterministic).
__global__ void __launch_bounds__(256)
dft_axis_warp_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ tw, long long n_a,
                     int n_in, int n_out, long long n_inner, int L, int backward, double scale) {
  const long long total = n_a * n_out * n_inner;
  const int lane = threadIdx.x & 31;
  for (long long g = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; g < total;
       g += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const long long inner = g % n_inner;
    const long long rest = g / n_inner;
    const int qo = static_cast<int>(rest % n_out);
    const long long a = rest / n_out;
    const c64* src = in + (a * n_in) * n_inner + inner;
    const int step = static_cast<int>((32LL * qo) % L);
    int idx = static_cast<int>((static_cast<long long>(lane) * qo) % L);
    c64 acc0 = cmk(0.0, 0.0), acc1 = cmk(0.0, 0.0);
    int j = lane;
    for (; j + 32 < n_in; j += 64) {
      c64 w0 = __ldg(tw + idx);
      int idx1 = idx + step;
      if (idx1 >= L) idx1 -= L;
      c64 w1 = __ldg(tw + idx1);
      const c64 v0 = src[static_cast<long long>(j) * n_inner], v1 = src[static_cast<long long>(j + 32) * n_inner];
      if (backward) {
        w0.y = -w0.y;
        w1.y = -w1.y;
      }
      acc0 = cfma(w0, v0, acc0);
      acc1 = cfma(w1, v1, acc1);
      idx = idx1 + step;
      if (idx >= L) idx -= L;
    }
    if (j < n_in) {
      c64 w = __ldg(tw + idx);
      if (backward) w.y = -w.y;
      acc0 = cfma(w, src[static_cast<long long>(j) * n_inner], acc0);
    }
    c64 t = cadd(acc0, acc1);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      t.x += __shfl_xor_sync(0xffffffffu, t.x, off);
      t.y += __shfl_xor_sync(0xffffffffu, t.y, off);
    }
    if (lane == 0) out[(a * n_out + qo) * n_inner + inner] = cscale(t, scale);
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

// Multi-RHS mode product on the FP64 tensor cores: per mode q the field block
// F_q (nrhs x b, rhs-major, contiguous) times Λ_q^T,
//   image[q][r][i] = sum_j Λ_q(i, j) F_q[r][j]      (C = F Λ^T: M = rhs, N = K = b),
// the dense contraction of src/structured.cpp:148-152 batched over right-hand
// sides. One CTA per (mode, block of kModeRows right-hand sides); Λ_q (one
// contiguous b x b block) and the F_q rows are staged in shared memory, the
// product runs as 8 x 8 x 4 DMMA tiles with the complex Gauss 3M split.
constexpr int kModeRows = 64;

__global__ void __launch_bounds__(256)
mode_gemm_kernel(const c64* __restrict__ lambda, const c64* __restrict__ field, c64* __restrict__ image, int b,
                 int nrhs) {
  extern __shared__ __align__(16) unsigned char mg_smem[];
  const int pf = odd_pitch(b);
  c64* lam = reinterpret_cast<c64*>(mg_smem);  // [j * b + i] = Λ(i, j), as stored
  c64* f = lam + b * b;                        // rows x pf
  const long long q = blockIdx.x;
  const int r0 = blockIdx.y * kModeRows, rows = min(kModeRows, nrhs - r0);
  const c64* lq = lambda + q * b * b;
  for (int k = threadIdx.x; k < b * b; k += blockDim.x) lam[k] = lq[k];
  const c64* fq = field + (q * nrhs + r0) * b;
  for (int k = threadIdx.x; k < rows * b; k += blockDim.x) {
    const int r = k / b;
    f[r * pf + (k - r * b)] = fq[k];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int tn_count = (b + 7) / 8, tiles = ((rows + 7) / 8) * tn_count;
  c64* out = image + (q * nrhs + r0) * b;
  for (int t = warp; t < tiles; t += n_warps) {
    const int tm = t / tn_count, tn = t - tm * tn_count;
    double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
    const int am = tm * 8 + fr, bn = tn * 8 + fr;
    for (int k0 = 0; k0 < b; k0 += 4) {
      const int k = k0 + fk;
      const c64 av = (am < rows && k < b) ? f[am * pf + k] : cmk(0.0, 0.0);
      const c64 bv = (k < b && bn < b) ? lam[k * b + bn] : cmk(0.0, 0.0);
      dmma884(t1[0], t1[1], av.x, bv.x);
      dmma884(t2[0], t2[1], av.y, bv.y);
      dmma884(t3[0], t3[1], av.x + av.y, bv.x + bv.y);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tn * 8 + 2 * fk + j;
      if (am < rows && n < b) out[am * b + n] = cmk(t1[j] - t2[j], t3[j] - t1[j] - t2[j]);
    }
  }
}

// Multi-RHS P2M on the FP64 tensor cores: all right-hand sides and cells are
// one skinny GEMM sharing V0,
//   mom[cell nrhs + r][c] = sum_j x[r N + cell n + j] V0[c][j]   (M = cells nrhs, N = b, K = n).
// Persistent CTAs (one per SM) hold V0^T in shared memory (row pitch = 4 mod 8
// complex: the 8 x 4 fragment loads hit distinct 16-byte slots); each warp
// takes 8-row tiles in turn, streams its x rows from HBM in 8 x 4 fragments and
// keeps four 8 x 8 coefficient tiles in registers (Gauss 3M as in mode_gemm_kernel).
constexpr int kP2mWarps = 16;

__host__ __device__ inline int p2m_pitch(int n) { return ((n + 3) / 8) * 8 + 4; }

__global__ void __launch_bounds__(kP2mWarps * 32, 1)
p2m_gemm_kernel(const c64* __restrict__ v0t, const c64* __restrict__ x, c64* __restrict__ mom, int n, int b,
                long long N, int nrhs, int cells) {
  extern __shared__ __align__(16) unsigned char p2m_smem[];
  c64* vs = reinterpret_cast<c64*>(p2m_smem);
  const int pk = p2m_pitch(n);
  for (int k = threadIdx.x; k < b * n; k += blockDim.x) {
    const int c = k / n;
    vs[c * pk + (k - c * n)] = v0t[k];
  }
  __syncthreads();
  const long long rows = static_cast<long long>(cells) * nrhs, tiles = (rows + 7) / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  for (long long t = static_cast<long long>(blockIdx.x) * kP2mWarps + warp; t < tiles;
       t += static_cast<long long>(gridDim.x) * kP2mWarps) {
    const long long rho = t * 8 + fr;  // output row cell * nrhs + r
    const bool row_ok = rho < rows;
    const long long cell = row_ok ? rho / nrhs : 0, r = row_ok ? rho - cell * nrhs : 0;
    const c64* xr = x + r * N + cell * n;
    for (int tn0 = 0; tn0 < b; tn0 += 32) {  // four 8-wide coefficient tiles at a time
      double t1[4][2] = {}, t2[4][2] = {}, t3[4][2] = {};
      for (int k0 = 0; k0 < n; k0 += 16) {
        c64 av[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int k = k0 + 4 * s + fk;
          av[s] = (row_ok && k < n) ? __ldcs(xr + k) : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int k = k0 + 4 * s + fk;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = tn0 + 8 * u + fr;
            const c64 bv = (c < b && k < n) ? vs[c * pk + k] : cmk(0.0, 0.0);
            dmma884(t1[u][0], t1[u][1], av[s].x, bv.x);
            dmma884(t2[u][0], t2[u][1], av[s].y, bv.y);
            dmma884(t3[u][0], t3[u][1], av[s].x + av[s].y, bv.x + bv.y);
          }
        }
      }
      // D fragment: lane (fr, fk) holds row fr, columns 2 fk and 2 fk + 1 of each tile
      if (row_ok) {
        c64* out = mom + rho * b;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = tn0 + 8 * u + 2 * fk + j;
            if (c < b) out[c] = cmk(t1[u][j] - t2[u][j], t3[u][j] - t1[u][j] - t2[u][j]);
          }
      }
    }
  }
}

constexpr size_t kZfSmemMax = 225 * 1024;  // dynamic; static barriers + driver share take the rest

// One z-DFT phase of the fused kernel, over the consumer threads:
//   dst[o][f] = scale * sum_{j < n_in} w(j*o mod L) src[j][f],  o < n_out
// w = tw (forward) or conj(tw) (backward; results go to global `out` rows
// (o*plane + col)*E). A thread owns G consecutive outputs of one field
// (independent chains sharing each input load); G = 1 uses two partial sums.
__device__ __forceinline__ int zdft_group(int outputs, int threads) {
  return outputs >= 3 * threads ? 4 : (outputs >= 3 * threads / 2 ? 2 : 1);
}

template <int G, bool kBack>
__device__ __forceinline__ void zdft(const c64* __restrict__ src, c64* __restrict__ dst, const c64* __restrict__ tw_s,
                                     int n_in, int n_out, int L, int E, int ct, int n_ct, double scale,
                                     c64* __restrict__ out, long long plane, long long col) {
  // shared-load latency (~60 cycles) dominates a naive loop: inputs and
  // twiddles of 4 terms are loaded before their FMAs, and even / odd terms
  // feed separate partial sums
  const int n_g = (n_out + G - 1) / G;
  for (int e = ct; e < n_g * E; e += n_ct) {
    const int g = e / E, f = e - g * E, o0 = g * G;
    c64 acc[G][2];
    int idx[G], step[G];
#pragma unroll
    for (int o = 0; o < G; ++o) {
      acc[o][0] = acc[o][1] = cmk(0.0, 0.0);
      idx[o] = 0;
      step[o] = (o0 + o) % L;  // padded outputs (o0 + o >= n_out) may exceed L
    }
    int j = 0;
    for (; j + 4 <= n_in; j += 4) {
      c64 v[4], w[G][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = src[(j + u) * E + f];
#pragma unroll
      for (int o = 0; o < G; ++o)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w[o][u] = tw_s[idx[o]];
          idx[o] += step[o];
          if (idx[o] >= L) idx[o] -= L;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int o = 0; o < G; ++o) {
          c64 t = w[o][u];
          if (kBack) t.y = -t.y;
          acc[o][u & 1] = cfma(t, v[u], acc[o][u & 1]);
        }
    }
    for (; j < n_in; ++j) {
      const c64 v = src[j * E + f];
#pragma unroll
      for (int o = 0; o < G; ++o) {
        c64 t = tw_s[idx[o]];
        if (kBack) t.y = -t.y;
        acc[o][0] = cfma(t, v, acc[o][0]);
        idx[o] += step[o];
        if (idx[o] >= L) idx[o] -= L;
      }
    }
#pragma unroll
    for (int o = 0; o < G; ++o) {
      if (o0 + o >= n_out) continue;
      const c64 r = cadd(acc[o][0], acc[o][1]);
      if (kBack)
        out[(static_cast<long long>(o0 + o) * plane + col) * E + f] = cscale(r, scale);
      else
        dst[(o0 + o) * E + f] = r;
    }
  }
}

// The same z-DFT of the item's columns as small complex GEMMs on DMMA (the
// FMA form above spends its time on shared-memory twiddle / input loads and
// dependent FMA chains): per column C[n_out][E] = W[n_out][n_in] B[n_in][E] with
// W[q][j] = tw[(q j) mod L] (conjugated backward), tiles of 8 outputs x 8
// fields over the DFT warps, A fragments formed from the twiddle table, Gauss
// 3-multiplication form. Forward: C into f_z (shared); backward: C * scale
// into the global output of column col. The tile sums run in a fixed order.
template <bool kBack>
__device__ __forceinline__ void zdft_mma(const c64* const* src, c64* const* dst, const long long* cols, int nc,
                                         const c64* __restrict__ tw_s, int n_in, int n_out, int L, int E, int w,
                                         int n_w, int lane, double scale, c64* __restrict__ out, long long plane) {
  const int fr = lane >> 2, fk = lane & 3;
  const int MT = (n_out + 7) / 8, NT = (E + 7) / 8, KT = (n_in + 3) / 4;
  const int per_col = MT * NT;
  for (int t = w; t < nc * per_col; t += n_w) {
    const int s = t / per_col, r = t - s * per_col, mt = r / NT, nt = r - mt * NT;
    const c64* B = src[s];
    const int q = mt * 8 + fr, cb = nt * 8 + fr;
    double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
    for (int kt = 0; kt < KT; ++kt) {
      const int j = kt * 4 + fk;
      c64 a = cmk(0.0, 0.0), bv = cmk(0.0, 0.0);
      if (j < n_in) {
        if (q < n_out) {
          a = tw_s[(q * j) % L];
          if (kBack) a.y = -a.y;
        }
        if (cb < E) bv = B[j * E + cb];
      }
      dmma884(t1[0], t1[1], a.x, bv.x);
      dmma884(t2[0], t2[1], a.y, bv.y);
      dmma884(t3[0], t3[1], a.x + a.y, bv.x + bv.y);
    }
    if (q >= n_out) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = nt * 8 + 2 * fk + h;
      if (c >= E) continue;
      const c64 v = cmk(t1[h] - t2[h], t3[h] - t1[h] - t2[h]);
      if (kBack)
        out[(static_cast<long long>(q) * plane + cols[s]) * E + c] = cscale(v, scale);
      else
        dst[s][q * E + c] = v;
    }
  }
}

// one mode's product for the lanes of a warp: g[ri] = sum_c lam[i + b c] f[r b + c]
__device__ __forceinline__ void mode_product_warp(const c64* __restrict__ lam_blk, const c64* __restrict__ f_mode,
                                                  c64* __restrict__ g_mode, int E, int b, int lane) {
  for (int ri = lane; ri < E; ri += 32) {
    const int r = ri / b, i = ri - r * b;
    const c64* lam = lam_blk + i;
    const c64* f = f_mode + r * b;
    c64 acc0 = cmk(0.0, 0.0), acc1 = cmk(0.0, 0.0);
    int c = 0;
    for (; c + 4 <= b; c += 4) {
      c64 l[4], v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        l[u] = lam[(c + u) * b];
        v[u] = f[c + u];
      }
      acc0 = cfma(l[0], v[0], acc0);
      acc1 = cfma(l[1], v[1], acc1);
      acc0 = cfma(l[2], v[2], acc0);
      acc1 = cfma(l[3], v[3], acc1);
    }
    for (; c < b; ++c) acc0 = cfma(lam[c * b], f[c], acc0);
    g_mode[ri] = cadd(acc0, acc1);
  }
}

// Last-axis fusion: forward DFT along z (Mz nonzero inputs -> Lz modes), the
// per-mode product with Λ_q, and the pruned inverse along z (Lz modes -> Mz
// kept outputs) per (qy, qx) column; the z-extended field never touches HBM.
// Persistent (one CTA per SM walking columns blockIdx.x + k gridDim.x) and
// warp-specialised in three roles, so the Λ stream (the only large operand,
// read exactly once) never waits on a DFT phase:
//   warp 0 lane 0      producer: each mode's b x b Λ block (contiguous) with one
//                      cp.async.bulk into a ring of `ring` shared-memory slots
//                      (full / empty mbarriers), refilled as soon as a slot is
//                      released, running on across columns; input columns (Mz
//                      rows of E contiguous values) the same way, double-buffered
//   n_mw mode warps    stream column after column: warp w owns ring slots w and
//                      w + n_mw and takes the modes g = w (mod n_mw); reads
//                      f_z[k%2], writes g_z[k%2]
//   n_dw DFT warps     iteration k: forward DFT of column k into f_z[k%2], then
//                      inverse DFT of column k-1 from g_z[(k-1)%2]
// Hand-offs (mbarriers, phases by column parity):
//   fwd_done[c%2]  DFT -> mode   f_z of column c ready          (count 1)
//   col_done[c%2]  mode -> DFT   modes of column c finished:    (count n_mw)
//                                g_z complete, f_z free again
//   inv_done[c%2]  DFT -> mode   inverse of column c read g_z   (count 1)
// While the mode warps stream column k, the DFT warps compute column k+1's
// forward pass and column k-1's inverse. A warp owning fixed ring slots never
// waits more than one phase ahead on a slot.
//   in  : F2[iz][plane][E]   (iz < Mz)      out: H2[iz][plane][E] (iz < Mz)
//   E = nrhs * b fields, plane = Ly * Lx columns, lambda[q][b*b], q = qz*plane + column
// Measured route (profiles/r01_m2l_probes.md): producer/consumer mbarriers
// instead of barrier-separated refills (3.5 -> 6.7 TB/s in the probe) and the
// z-DFTs on their own warps.
constexpr int kPipeMaxModeWarps = 8;
constexpr int kPipeMaxRing = 16;
constexpr int kPipeMaxDftWarps = 8;

__device__ __forceinline__ void dft_sync(int n_threads) {
  asm volatile("bar.sync 2, %0;\n" ::"r"(n_threads) : "memory");
}

// In-place mode product on the E = nrhs * b fields of one mode:
//   f <- Λ f,  or  f <- D Λ D f  (conj: the mirror column's mode, see below)
// with D = diag((-1)^n) over the coefficients (n, m). Each right-hand side's b
// outputs are formed in registers before any is written back.
__device__ __forceinline__ void mode_inplace(const c64* __restrict__ lam_blk, c64* __restrict__ f_mode, int E, int b,
                                             int lane, bool conj, const double* __restrict__ dsg) {
  constexpr int kMaxPerLane = 8;  // b <= 256
  for (int r0 = 0; r0 < E; r0 += b) {
    c64* f = f_mode + r0;
    c64 res[kMaxPerLane];
#pragma unroll
    for (int k = 0; k < kMaxPerLane; ++k) {
      const int i = lane + 32 * k;
      res[k] = cmk(0.0, 0.0);
      if (i >= b) continue;
      const c64* lam = lam_blk + i;
      c64 acc0 = cmk(0.0, 0.0), acc1 = cmk(0.0, 0.0);
      int c = 0;
      for (; c + 4 <= b; c += 4) {
        c64 l[4], v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          l[u] = lam[(c + u) * b];
          v[u] = f[c + u];
          if (conj) v[u] = cscale(v[u], dsg[c + u]);
        }
        acc0 = cfma(l[0], v[0], acc0);
        acc1 = cfma(l[1], v[1], acc1);
        acc0 = cfma(l[2], v[2], acc0);
        acc1 = cfma(l[3], v[3], acc1);
      }
      for (; c < b; ++c) acc0 = cfma(lam[c * b], conj ? cscale(f[c], dsg[c]) : f[c], acc0);
      res[k] = cadd(acc0, acc1);
      if (conj) res[k] = cscale(res[k], dsg[i]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kMaxPerLane; ++k)
      if (lane + 32 * k < b) f[lane + 32 * k] = res[k];
    __syncwarp();
  }
}

// The common case b <= 32 (n_t <= 4): one output per lane. f1 <- Λ f1 and, when
// f2 is given, f2 <- D Λ D f2 in the same pass, the two sums sharing every Λ load.
template <bool kPair>
__device__ __forceinline__ void mode_pair_small(const c64* __restrict__ lam_blk, c64* __restrict__ f1,
                                                c64* __restrict__ f2, int E, int b, int lane,
                                                const double* __restrict__ dsg) {
  const bool active = lane < b;
  const c64* lam = lam_blk + (active ? lane : 0);
  for (int r0 = 0; r0 < E; r0 += b) {
    c64 a0 = cmk(0.0, 0.0), a1 = cmk(0.0, 0.0), p0 = cmk(0.0, 0.0), p1 = cmk(0.0, 0.0);
    const c64* x1 = f1 + r0;
    const c64* x2 = kPair ? f2 + r0 : nullptr;
    int c = 0;
    for (; c + 2 <= b; c += 2) {
      const c64 l0 = lam[c * b], l1 = lam[(c + 1) * b];
      a0 = cfma(l0, x1[c], a0);
      a1 = cfma(l1, x1[c + 1], a1);
      if (kPair) {
        p0 = cfma(l0, cscale(x2[c], dsg[c]), p0);
        p1 = cfma(l1, cscale(x2[c + 1], dsg[c + 1]), p1);
      }
    }
    if (c < b) {
      const c64 l0 = lam[c * b];
      a0 = cfma(l0, x1[c], a0);
      if (kPair) p0 = cfma(l0, cscale(x2[c], dsg[c]), p0);
    }
    __syncwarp();  // every lane has read f1 / f2 of this right-hand side
    if (active) {
      f1[r0 + lane] = cadd(a0, a1);
      if (kPair) f2[r0 + lane] = cscale(cadd(p0, p1), dsg[lane]);
    }
    __syncwarp();
  }
}

// Work items: one column (qy, qx), or a column and its mirror (-qy, -qx) when
// Λ has the K-bank parity Λ(-q) = D Λ(q) D (K(-δ) = D K(δ) D: solid harmonics
// of degree l change sign by (-1)^l and the Gaunt rule makes n + n' + l even;
// the far offsets are symmetric). Then each Λ block (qz, c) is streamed once
// and used for mode qz of c and, conjugated by D, for mode -qz of the mirror:
// half the Λ bytes. items[k] = (c, mirror or -1).
__global__ void __launch_bounds__(32 * (1 + kPipeMaxModeWarps + kPipeMaxDftWarps), 1)
m2l_zpipe_kernel(const c64* __restrict__ in, c64* __restrict__ out, const c64* __restrict__ lambda,
                 const c64* __restrict__ tw, int Mz, int Lz, long long plane, int E, int b, int n_mw,
                 int ring, int n_dw, double scale, const int2* __restrict__ items, int n_items_total,
                 int use_mma) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b2 = b * b;
  c64* ring_buf = reinterpret_cast<c64*>(smem_raw);  // ring x b2
  c64* f_in0 = ring_buf + ring * b2;                  // [buffer 2][column 2][Mz][E]
  c64* f_z0 = f_in0 + 4 * Mz * E;                     // [buffer 2][column 2][Lz][E] (g in place)
  c64* tw_s = f_z0 + 4 * Lz * E;                      // Lz twiddles
  __shared__ double dsg[256];                         // (-1)^n of coefficient (n, m)
  __shared__ __align__(8) unsigned long long full[kPipeMaxRing], empty[kPipeMaxRing];
  __shared__ __align__(8) unsigned long long in_full[2], in_empty[2];
  __shared__ __align__(8) unsigned long long fwd_done[2], col_done[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = static_cast<int>((n_items_total - blockIdx.x + gridDim.x - 1) / gridDim.x);
  auto item = [&](int k) { return items[blockIdx.x + static_cast<long long>(k) * gridDim.x]; };
  if (tid == 0) {
    for (int s = 0; s < ring; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&in_full[s]), 1);
      mbar_init(smem_u32(&in_empty[s]), 1);
      mbar_init(smem_u32(&fwd_done[s]), 1);
      mbar_init(smem_u32(&col_done[s]), n_mw);
    }
    mbar_fence_init();
  }
  for (int k = tid; k < Lz; k += blockDim.x) tw_s[k] = tw[k];
  for (int i = tid; i < b; i += blockDim.x) {
    int n = 0;
    while ((n + 1) * (n + 1) <= i) ++n;
    dsg[i] = (n & 1) ? -1.0 : 1.0;
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      const unsigned lam_bytes = static_cast<unsigned>(b2 * sizeof(c64));
      const unsigned row_bytes = static_cast<unsigned>(E * sizeof(c64));
      auto issue_input = [&](int k) {  // both columns of item k -> buffer k % 2
        if (k >= n_items) return;
        const int buf = k & 1;
        if (k >= 2) mbar_wait(smem_u32(&in_empty[buf]), static_cast<unsigned>((k / 2 - 1) & 1));
        const int2 it = item(k);
        const int nc = it.y >= 0 ? 2 : 1;
        const unsigned bar = smem_u32(&in_full[buf]);
        mbar_arrive_expect_tx(bar, row_bytes * Mz * nc);
        for (int s = 0; s < nc; ++s) {
          const long long col = s ? it.y : it.x;
          c64* dst = f_in0 + (buf * 2 + s) * Mz * E;
          for (int iz = 0; iz < Mz; ++iz)
            bulk_g2s(smem_u32(dst + iz * E), in + (iz * plane + col) * E, row_bytes, bar);
        }
      };
      issue_input(0);
      issue_input(1);
      int slot = 0;
      unsigned phase = 0;
      long long g = 0;
      const long long mode_step = plane * b2;
      for (int k = 0; k < n_items; ++k) {
        if (k > 0) issue_input(k + 1);  // buffer of item k - 1: its forward pass is done by now
        const c64* col_lam = lambda + static_cast<long long>(item(k).x) * b2;
        for (int qz = 0; qz < Lz; ++qz, ++g) {
          if (g >= ring) mbar_wait(smem_u32(&empty[slot]), phase ^ 1u);
          const unsigned bar = smem_u32(&full[slot]);
          mbar_arrive_expect_tx(bar, lam_bytes);
          bulk_g2s(smem_u32(ring_buf + slot * b2), col_lam + qz * mode_step, lam_bytes, bar);
          if (++slot == ring) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp <= n_mw) {  // ---- mode warps
    const int w = warp - 1;
    // this warp's modes are the global g = w, w + n_mw, ... (ring = spw * n_mw):
    // the j-th lands in slot w + (j % spw) n_mw, phase (j / spw) & 1
    const int spw = ring / n_mw;
    long long g = w;
    int jm = 0;
    unsigned jphase = 0;
    for (int k = 0; k < n_items; ++k) {
      const int buf = k & 1;
      const bool pair = item(k).y >= 0;
      mbar_wait(smem_u32(&fwd_done[buf]), static_cast<unsigned>((k >> 1) & 1));  // f_z[buf] holds item k
      c64* fz = f_z0 + buf * 2 * Lz * E;
      const long long g_end = static_cast<long long>(k + 1) * Lz;
      for (; g < g_end; g += n_mw) {
        const int qz = static_cast<int>(g - static_cast<long long>(k) * Lz);
        const int slot = w + jm * n_mw;
        mbar_wait(smem_u32(&full[slot]), jphase);
        if (++jm == spw) {
          jm = 0;
          jphase ^= 1u;
        }
        const c64* blk = ring_buf + slot * b2;
        c64* m1 = fz + qz * E;
        c64* m2 = fz + (Lz + (qz ? Lz - qz : 0)) * E;  // the mirror column's mode -qz
        if (use_mma & 2) {
          // FPBEM_ZF_PROBE=1 (diagnostic, wrong results): the Λ stream without the mode products
        } else if (b <= 32) {
          if (pair)
            mode_pair_small<true>(blk, m1, m2, E, b, lane, dsg);
          else
            mode_pair_small<false>(blk, m1, nullptr, E, b, lane, dsg);
        } else {
          mode_inplace(blk, m1, E, b, lane, false, dsg);
          if (pair) mode_inplace(blk, m2, E, b, lane, true, dsg);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&col_done[buf]));
    }
  } else {  // ---- DFT warps
    const int dt = tid - 32 * (1 + n_mw), n_dt = 32 * n_dw;
    const bool mma = (use_mma & 1) != 0;  // the z-DFTs on DMMA (FPBEM_ZF_DFT=fma: the FMA form, A/B)
    const bool skip = (use_mma & 4) != 0;  // FPBEM_ZF_PROBE=2 (diagnostic, wrong results): no z-DFT work
    auto inverse = [&](int c) {  // inverse z of item c (its modes are finished)
      const int buf = c & 1;
      mbar_wait(smem_u32(&col_done[buf]), static_cast<unsigned>((c >> 1) & 1));
      const int2 it = item(c);
      if (skip) {
        dft_sync(n_dt);
        return;
      }
      if (mma) {
        const c64* srcs[2] = {f_z0 + (buf * 2) * Lz * E, f_z0 + (buf * 2 + 1) * Lz * E};
        const long long cols[2] = {it.x, it.y};
        zdft_mma<true>(srcs, nullptr, cols, it.y >= 0 ? 2 : 1, tw_s, Lz, Mz, Lz, E, dt >> 5, n_dw, lane, scale, out,
                       plane);
        dft_sync(n_dt);
        return;
      }
      for (int s = 0; s < (it.y >= 0 ? 2 : 1); ++s) {
        const long long col = s ? it.y : it.x;
        const c64* g_z = f_z0 + (buf * 2 + s) * Lz * E;
        const int G = zdft_group(Mz * E, n_dt);
        if (G == 4) zdft<4, true>(g_z, nullptr, tw_s, Lz, Mz, Lz, E, dt, n_dt, scale, out, plane, col);
        else if (G == 2) zdft<2, true>(g_z, nullptr, tw_s, Lz, Mz, Lz, E, dt, n_dt, scale, out, plane, col);
        else zdft<1, true>(g_z, nullptr, tw_s, Lz, Mz, Lz, E, dt, n_dt, scale, out, plane, col);
      }
      dft_sync(n_dt);
    };
    for (int k = 0; k < n_items; ++k) {
      const int buf = k & 1;
      // f_z[buf] was last used by item k - 2: its modes finished (col_done waited
      // in inverse(k - 2)) and its inverse ran before this forward pass
      mbar_wait(smem_u32(&in_full[buf]), static_cast<unsigned>((k >> 1) & 1));
      const int nc = item(k).y >= 0 ? 2 : 1;
      if (mma && !skip) {
        const c64* srcs[2] = {f_in0 + (buf * 2) * Mz * E, f_in0 + (buf * 2 + 1) * Mz * E};
        c64* dsts[2] = {f_z0 + (buf * 2) * Lz * E, f_z0 + (buf * 2 + 1) * Lz * E};
        zdft_mma<false>(srcs, dsts, nullptr, nc, tw_s, Mz, Lz, Lz, E, dt >> 5, n_dw, lane, 1.0, nullptr, 0);
      }
      for (int s = 0; s < (mma || skip ? 0 : nc); ++s) {
        c64* f_z = f_z0 + (buf * 2 + s) * Lz * E;
        const c64* f_in = f_in0 + (buf * 2 + s) * Mz * E;
        const int G = zdft_group(Lz * E, n_dt);
        if (G == 4) zdft<4, false>(f_in, f_z, tw_s, Mz, Lz, Lz, E, dt, n_dt, 1.0, nullptr, 0, 0);
        else if (G == 2) zdft<2, false>(f_in, f_z, tw_s, Mz, Lz, Lz, E, dt, n_dt, 1.0, nullptr, 0, 0);
        else zdft<1, false>(f_in, f_z, tw_s, Mz, Lz, Lz, E, dt, n_dt, 1.0, nullptr, 0, 0);
      }
      dft_sync(n_dt);
      if (dt == 0) {
        mbar_arrive(smem_u32(&fwd_done[buf]));
        mbar_arrive(smem_u32(&in_empty[buf]));
      }
      if (k >= 1) inverse(k - 1);
    }
    if (n_items >= 1) inverse(n_items - 1);
  }
  __syncthreads();  // the producer stays resident until every copy it issued has landed
}

// The per-mode products of the far field as ONE FLAT STREAM over Λ, in place on
// the z-extended field (the unfused form of the z kernel above: the z-DFTs run
// as axis passes before and after, and the 2 x 13 MB field of cfg3 stays in the
// 126 MB L2). Unit u = qz * n_items + k: the Λ block of mode qz of column
// c = items[k].x, used for every mode whose block it determines
// (src/structured.cpp:148-152, one block read for up to four modes):
//   (qz, c)     Λ
//   (-qz, c')   D Λ D          c' = items[k].y the mirror column, D = diag((-1)^n)
//                              (Λ(-q) = D Λ(q) D, the pairing of the z kernel)
//   (-qz, c)    Dz Λ Dz        quad only: Dz = diag((-1)^(n+m)), the reflection z -> -z
//   (qz, c')    (D Dz) Λ (Dz D)   (K(Rz δ) = Dz K(δ) Dz and far offsets symmetric in z;
//                              checked on the spectrum actually built, lambda_parity_kernel)
// so quad streams only qz <= Lz/2: a quarter of Λ. The signs are applied to the
// vectors when they are staged and when they are written back; the products
// themselves share every Λ load (mode_multi). CTA c takes the units c, c + G,
// c + 2G, ...: at any time the CTAs read neighbouring blocks, the access order
// that reached the copy bandwidth in the stream probe (profiles/r01_m2l_probes.md;
// the per-column walk of the fused kernel ran at 4 TB/s). Warp 0 lane 0 is the
// producer (one cp.async.bulk per block into a ring, full / empty mbarriers);
// consumer warp w takes the CTA's units j = w (mod n_w): the fields of its next
// unit are loaded into registers before the wait on the current block, staged
// in a warp-private shared buffer, multiplied in place and written back coalesced.
// ring is a multiple of n_w, so a slot's successive blocks go to ONE warp in
// order: it waits for a slot's phase only after it consumed the phase before
// (a parity wait two phases ahead would pass at once on the stale phase).
constexpr int kStreamWarps = 11;  // most consumer warps (12 warps with the producer: 168 registers each)
constexpr int kStreamMaxRing = 32;
constexpr int kStreamRegs = 2;  // E <= 32 * kStreamRegs

// s[v] <- Λ s[v] for NV staged vectors of E = nrhs x b fields (b <= 32: one output per lane).
// BC > 0: b = BC at compile time (the reference's default order n_t = 4, b = 25: the column loop
// is unrolled by 4 pairs — a full unroll spills — so its shared-memory loads run ahead of the FMA
// chains); BC = 0: any b.
template <int NV, int BC>
__device__ __forceinline__ void mode_multi(const c64* __restrict__ lam_blk, c64* __restrict__ s0, int E, int b_rt,
                                           int lane) {
  const int b = BC > 0 ? BC : b_rt;
  const c64* lam = lam_blk + (lane < b ? lane : 0);
  for (int r0 = 0; r0 < E; r0 += b) {
    c64 a0[NV], a1[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) a0[v] = a1[v] = cmk(0.0, 0.0);
    int c = 0;
#pragma unroll(BC > 0 ? 4 : 1)
    for (; c + 2 <= b; c += 2) {
      const c64 l0 = lam[c * b], l1 = lam[(c + 1) * b];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const c64* x = s0 + v * E + r0 + c;
        a0[v] = cfma(l0, x[0], a0[v]);
        a1[v] = cfma(l1, x[1], a1[v]);
      }
    }
    if (c < b) {
      const c64 l0 = lam[c * b];
#pragma unroll
      for (int v = 0; v < NV; ++v) a0[v] = cfma(l0, s0[v * E + r0 + c], a0[v]);
    }
    __syncwarp();  // every lane has read this right-hand side's inputs
    if (lane < b) {
#pragma unroll
      for (int v = 0; v < NV; ++v) s0[v * E + r0 + lane] = cadd(a0[v], a1[v]);
    }
    __syncwarp();
  }
}

template <int BC>
__device__ __forceinline__ void mode_multi_nv(int nv, const c64* __restrict__ blk, c64* __restrict__ st, int E, int b,
                                              int lane) {
  if (nv == 4)
    mode_multi<4, BC>(blk, st, E, b, lane);
  else if (nv == 2)
    mode_multi<2, BC>(blk, st, E, b, lane);
  else
    mode_multi<1, BC>(blk, st, E, b, lane);
}

__global__ void __launch_bounds__(32 * (1 + kStreamWarps), 1)
mode_stream_kernel(c64* __restrict__ field, const c64* __restrict__ lambda, int Lz, int qz_count, long long plane,
                   int E, int b, int ring, const int2* __restrict__ items, int n_items, int quad, int probe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b2 = b * b;
  c64* ring_buf = reinterpret_cast<c64*>(smem_raw);  // ring x b2
  c64* stage0 = ring_buf + ring * b2;                 // [warp][4][E]
  __shared__ double sgn[4][32];  // sign of coefficient i under: none, D, Dz, D Dz
  __shared__ __align__(8) unsigned long long full[kStreamMaxRing], empty[kStreamMaxRing];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_w = (blockDim.x >> 5) - 1;  // consumer warps; ring % n_w == 0
  const long long total = static_cast<long long>(n_items) * qz_count;
  const int n_units = static_cast<int>((total - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < ring; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_fence_init();
  }
  if (tid < 32) {  // coefficient i = n^2 + n + m: (-1)^n, (-1)^(n+m) = (-1)^(i - n^2)
    int n = 0;
    while ((n + 1) * (n + 1) <= tid) ++n;
    const double d = (n & 1) ? -1.0 : 1.0, dz = ((tid - n * n) & 1) ? -1.0 : 1.0;
    sgn[0][tid] = 1.0;
    sgn[1][tid] = d;
    sgn[2][tid] = dz;
    sgn[3][tid] = d * dz;
  }
  __syncthreads();
  const unsigned g = gridDim.x, ni = static_cast<unsigned>(n_items);
  if (warp == 0) {
    // ---- producer (lane 0): the items[] load and index arithmetic of one unit take longer than
    // its 10 KB copy takes to stream, so the block addresses are looked up four units ahead
    // of the copies (four independent loads in flight while four copies are issued)
    if (lane == 0) {
      const unsigned lam_bytes = static_cast<unsigned>(b2 * sizeof(c64));
      auto lookup = [&](int j) -> long long {  // element offset of unit j's Λ block (units < 2^31)
        if (j >= n_units) return 0;
        const unsigned u = blockIdx.x + static_cast<unsigned>(j) * g;
        const unsigned qz = u / ni, k = u - qz * ni;
        return (static_cast<long long>(qz) * plane + items[k].x) * b2;
      };
      long long nxt[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) nxt[i] = lookup(i);
      int slot = 0;
      unsigned phase = 0;
      for (int j0 = 0; j0 < n_units; j0 += 4) {
        long long cur[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) nxt[i] = lookup(j0 + 4 + i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (j0 + i >= n_units) break;
          if (j0 + i >= ring) mbar_wait(smem_u32(&empty[slot]), phase ^ 1u);
          const unsigned bar = smem_u32(&full[slot]);
          mbar_arrive_expect_tx(bar, lam_bytes);
          bulk_g2s(smem_u32(ring_buf + slot * b2), lambda + cur[i], lam_bytes, bar);
          if (++slot == ring) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {  // ---- consumers
    const int w = warp - 1;
    c64* st = stage0 + static_cast<long long>(w) * 4 * E;
    // the unit in registers: its vectors' addresses (null: absent) and values. Vector 0 is mode
    // (qz, c) [sign type 0]; vector 1 the mirror column's (-qz, c') [type 1] or, for a column that
    // is its own mirror, the z-reflected (-qz, c) [type 2]; vectors 2, 3 are (-qz, c) [2] and
    // (qz, c') [3]: a unit has 1, 2 or 4 vectors
    c64* ptr[4] = {nullptr, nullptr, nullptr, nullptr};
    int typ1 = 1;
    c64 reg[4][kStreamRegs];
    // items[] of a unit is loaded one unit ahead of its fields (two dependent loads in a row
    // would leave their latencies exposed in front of every unit)
    int2 it_ahead = make_int2(0, -1);
    auto item_of = [&](int j) {
      if (j >= n_units) return;
      const unsigned u = blockIdx.x + static_cast<unsigned>(j) * g;
      it_ahead = items[u % ni];
    };
    auto fetch = [&](int j) {  // fields of unit j (its item is in it_ahead); then the next unit's item
      const unsigned u = blockIdx.x + static_cast<unsigned>(j) * g;
      const int qz = static_cast<int>(u / ni);
      const int zm = qz ? Lz - qz : 0;
      const int2 it = it_ahead;
      item_of(j + n_w);
      const bool zpair = quad && zm != qz;
      ptr[0] = field + (qz * plane + it.x) * E;
      ptr[1] = ptr[2] = ptr[3] = nullptr;
      typ1 = 1;
      if (it.y >= 0) {
        ptr[1] = field + (zm * plane + it.y) * E;
        if (zpair) {
          ptr[2] = field + (zm * plane + it.x) * E;
          ptr[3] = field + (qz * plane + it.y) * E;
        }
      } else if (zpair) {
        ptr[1] = field + (zm * plane + it.x) * E;
        typ1 = 2;
      }
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (ptr[v]) {
#pragma unroll
          for (int t = 0; t < kStreamRegs; ++t) {
            const int i = lane + 32 * t;
            if (i < E) reg[v][t] = ptr[v][i];
          }
        }
    };
    item_of(w);
    if (w < n_units) fetch(w);
    for (int j = w; j < n_units; j += n_w) {
      c64* q[4];
      const int ty[4] = {0, typ1, 2, 3};
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        q[v] = ptr[v];
        if (ptr[v]) {
#pragma unroll
          for (int t = 0; t < kStreamRegs; ++t) {
            const int i = lane + 32 * t;
            if (i < E) st[v * E + i] = cscale(reg[v][t], sgn[ty[v]][E == b ? i : i % b]);
          }
        }
      }
      const int nv = q[2] ? 4 : (q[1] ? 2 : 1);
      if (j + n_w < n_units) fetch(j + n_w);
      __syncwarp();
      const int slot = j % ring;
      mbar_wait(smem_u32(&full[slot]), static_cast<unsigned>((j / ring) & 1));
      const c64* blk = ring_buf + slot * b2;
      if (probe & 1) {
        // FPBEM_MS_PROBE=1 (diagnostic, wrong results): the stream without the products
      } else if (b == 25) {
        mode_multi_nv<25>(nv, blk, st, E, b, lane);
      } else {
        mode_multi_nv<0>(nv, blk, st, E, b, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      if (!(probe & 2)) {  // FPBEM_MS_PROBE=2 (diagnostic): no write-back
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (q[v])
            for (int i = lane; i < E; i += 32) q[v][i] = cscale(st[v * E + i], sgn[ty[v]][E == b ? i : i % b]);
      }
      __syncwarp();  // the staging buffer is rewritten at the top of the next unit
    }
  }
  __syncthreads();  // the producer stays resident until every copy it issued has landed
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
  if (n_a * n_out * n_inner == 0) return cudaSuccess;
  // short lines: the tensor-core form (FPBEM_DFT=fma keeps the DFMA kernels, A/B)
  static const bool dft_mma = [] {
    const char* v = std::getenv("FPBEM_DFT");
    return !(v && std::strcmp(v, "fma") == 0);
  }();
  if (dft_mma && n_in <= kDftMmaMax && n_out <= kDftMmaMax) {
    const int MT = (n_out + 7) / 8, KT = (n_in + 3) / 4;
    const int KTd = (n_in % 4 == 1 && n_in > 4) ? KT - 1 : KT;  // the kernel's DMMA k steps (xcol)
    const size_t smem = sizeof(double) * 3 * MT * KT * 32;
    static std::atomic<unsigned long long> raised[4];
    {
      int i = 0;
      for (auto fn : {dft_axis_dmma_kernel<4>, dft_axis_dmma_kernel<8>, dft_axis_dmma_kernel<12>,
                      dft_axis_dmma_kernel<16>}) {
        cudaError_t e = ensure_max_smem(raised[i++], reinterpret_cast<const void*>(fn),
                                        static_cast<int>(sizeof(double) * 3 * 8 * 16 * 32));
        if (e != cudaSuccess) return e;
      }
    }
    const long long tiles = n_a * ((n_inner + 7) / 8);
    long long blocks = (tiles + kDftMmaWarps - 1) / kDftMmaWarps;
    // one resident wave (W expanded once per CTA), as many CTAs per SM as fit
    static int occ[4] = {0, 0, 0, 0};
    const int which = KTd <= 4 ? 0 : KTd <= 8 ? 1 : KTd <= 12 ? 2 : 3;
    if (occ[which] == 0) {
      const void* fn = which == 0   ? reinterpret_cast<const void*>(dft_axis_dmma_kernel<4>)
                       : which == 1 ? reinterpret_cast<const void*>(dft_axis_dmma_kernel<8>)
                       : which == 2 ? reinterpret_cast<const void*>(dft_axis_dmma_kernel<12>)
                                    : reinterpret_cast<const void*>(dft_axis_dmma_kernel<16>);
      int per_sm = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kDftMmaWarps * 32,
                                                                    sizeof(double) * 3 * 4 * 8 * 32);
      if (e != cudaSuccess) return e;
      occ[which] = per_sm > 0 ? per_sm : 1;
    }
    const long long cap = static_cast<long long>(kNumSMs) * occ[which];
    if (blocks > cap) blocks = cap;
    const int bw = backward ? 1 : 0;
    const bool pdl = pdl_enabled(stream);
    const dim3 g(static_cast<unsigned>(blocks)), blk(kDftMmaWarps * 32);
    if (KTd <= 4)
      return launch_ex(dft_axis_dmma_kernel<4>, g, blk, smem, stream, pdl, in, out, tw, n_a, n_in, n_out, n_inner, L, bw,
                       scale, L2pEpi{});
    if (KTd <= 8)
      return launch_ex(dft_axis_dmma_kernel<8>, g, blk, smem, stream, pdl, in, out, tw, n_a, n_in, n_out, n_inner, L, bw,
                       scale, L2pEpi{});
    if (KTd <= 12)
      return launch_ex(dft_axis_dmma_kernel<12>, g, blk, smem, stream, pdl, in, out, tw, n_a, n_in, n_out, n_inner, L,
                       bw, scale, L2pEpi{});
    return launch_ex(dft_axis_dmma_kernel<16>, g, blk, smem, stream, pdl, in, out, tw, n_a, n_in, n_out, n_inner, L, bw,
                     scale, L2pEpi{});
    return cudaGetLastError();
  }
  // widest output group that still gives >= 2 x 256 threads per SM
  const long long want = 2LL * kNumSMs * 256;
  if (n_in >= 64 && n_a * n_out * n_inner < want) {  // long lines, few outputs: a warp per output
    const long long warps = n_a * n_out * n_inner;
    long long blocks = (warps * 32 + 255) / 256;
    if (blocks > 16LL * kNumSMs) blocks = 16LL * kNumSMs;
    dft_axis_warp_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L,
                                                                       backward ? 1 : 0, scale);
    return cudaGetLastError();
  }
  int qg = 8;
  while (qg > 1 && n_a * ((n_out + qg - 1) / qg) * n_inner < want) qg /= 2;
  static const int qg_env = [] {  // FPBEM_DFT_QG: force the outputs per thread (A/B)
    const char* v = std::getenv("FPBEM_DFT_QG");
    return v ? std::atoi(v) : 0;
  }();
  if (qg_env == 1 || qg_env == 2 || qg_env == 4 || qg_env == 8) qg = qg_env;
  const long long total = n_a * ((n_out + qg - 1) / qg) * n_inner;
  const int grid = grid_for(total, 256), bw = backward ? 1 : 0;
  const size_t smem = sizeof(c64) * static_cast<size_t>(L);
  if (smem > 48 * 1024) {  // L > 3072: raise the dynamic shared-memory limit once per instantiation
    static std::atomic<unsigned long long> raised[4];
    int i = 0;
    for (auto fn : {dft_axis_kernel<8>, dft_axis_kernel<4>, dft_axis_kernel<2>, dft_axis_kernel<1>}) {
      cudaError_t e = ensure_max_smem(raised[i++], reinterpret_cast<const void*>(fn), 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
  }
  switch (qg) {
    case 8: dft_axis_kernel<8><<<grid, 256, smem, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L, bw, scale); break;
    case 4: dft_axis_kernel<4><<<grid, 256, smem, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L, bw, scale); break;
    case 2: dft_axis_kernel<2><<<grid, 256, smem, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L, bw, scale); break;
    default: dft_axis_kernel<1><<<grid, 256, smem, stream>>>(in, out, tw, n_a, n_in, n_out, n_inner, L, bw, scale); break;
  }
  return cudaGetLastError();
}

bool dft_l2p_supported(int n_in, int n_out, int b) {
  static const bool dft_mma = [] {
    const char* v = std::getenv("FPBEM_DFT");
    return !(v && std::strcmp(v, "fma") == 0);
  }();
  return dft_mma && n_in <= 32 && n_out <= kDftMmaMax && b >= 1 && b <= 32;
}

cudaError_t launch_dft_axis_l2p(const c64* in, c64* out, const c64* tw, long long n_a, int n_in, int n_out,
                                long long n_inner, int L, double scale, const c64* u0, const c64* loc, int b, int nrhs,
                                cudaStream_t stream) {
  if (n_a * n_out * n_inner == 0) return cudaSuccess;
  if (!dft_l2p_supported(n_in, n_out, b) || n_a % nrhs) return cudaErrorInvalidValue;
  const int MT = (n_out + 7) / 8, KT = (n_in + 3) / 4;
  const size_t smem = sizeof(double) * 3 * MT * KT * 32;
  static std::atomic<unsigned long long> raised[2];
  cudaError_t e = ensure_max_smem(raised[0], reinterpret_cast<const void*>(&dft_axis_dmma_kernel<4, true>),
                                  static_cast<int>(sizeof(double) * 3 * 8 * 16 * 32));
  if (e != cudaSuccess) return e;
  e = ensure_max_smem(raised[1], reinterpret_cast<const void*>(&dft_axis_dmma_kernel<8, true>),
                      static_cast<int>(sizeof(double) * 3 * 8 * 16 * 32));
  if (e != cudaSuccess) return e;
  L2pEpi epi;
  epi.u0 = u0;
  epi.loc = loc;
  epi.b = b;
  epi.nrhs = nrhs;
  epi.cpl = n_a / nrhs;
  const long long tiles = n_a * ((n_inner + 7) / 8);
  long long blocks = (tiles + kDftMmaWarps - 1) / kDftMmaWarps;
  const int KTd = (n_in % 4 == 1 && n_in > 4) ? KT - 1 : KT;  // the kernel's DMMA k steps (xcol)
  // one resident wave: as many CTAs per SM as the kernel's registers allow (a fixed 4 per SM left
  // a second, thin wave once the epilogue's registers brought the kernel to 3 CTAs per SM);
  // FPBEM_L2P_CTAS forces the CTAs per SM (A/B)
  static int occ[2] = {0, 0};
  const int which = KTd <= 4 ? 0 : 1;
  if (occ[which] == 0) {
    static const int occ_env = [] {
      const char* v = std::getenv("FPBEM_L2P_CTAS");
      return v ? std::atoi(v) : 0;
    }();
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm,
        which == 0 ? reinterpret_cast<const void*>(&dft_axis_dmma_kernel<4, true>)
                   : reinterpret_cast<const void*>(&dft_axis_dmma_kernel<8, true>),
        kDftMmaWarps * 32, smem);
    if (e != cudaSuccess) return e;
    occ[which] = occ_env > 0 ? occ_env : (per_sm > 0 ? per_sm : 1);
  }
  const long long cap = static_cast<long long>(device_sms()) * occ[which];
  if (blocks > cap) blocks = cap;
  if (KTd <= 4)
    dft_axis_dmma_kernel<4, true><<<static_cast<int>(blocks), kDftMmaWarps * 32, smem, stream>>>(
        in, out, tw, n_a, n_in, n_out, n_inner, L, 1, scale, epi);
  else
    dft_axis_dmma_kernel<8, true><<<static_cast<int>(blocks), kDftMmaWarps * 32, smem, stream>>>(
        in, out, tw, n_a, n_in, n_out, n_inner, L, 1, scale, epi);
  return cudaGetLastError();
}

size_t xy_plane_smem(int Mx, int My, int Lx, int Ly, bool inverse) {
  const size_t r1 = inverse ? My : Lx, c1 = inverse ? Ly : Mx, r2 = inverse ? Mx : Ly, c2 = inverse ? Lx : My;
  const size_t plane = inverse ? static_cast<size_t>(Ly) * Lx : static_cast<size_t>(My) * Mx;
  const size_t c = r1 * (c1 | 1) + r2 * (c2 | 1) + plane + static_cast<size_t>(My) * Lx;
  return c * sizeof(c64);
}

cudaError_t launch_xy_plane(const c64* in, c64* out, const c64* twx, const c64* twy, int Mx, int My, int Lx, int Ly,
                            int Mz, int E, bool inverse, double scale, cudaStream_t stream) {
  const size_t smem = xy_plane_smem(Mx, My, Lx, Ly, inverse);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> raised[2];
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_max_smem(raised[inverse ? 1 : 0],
                                    inverse ? reinterpret_cast<const void*>(&xy_plane_kernel<true>)
                                            : reinterpret_cast<const void*>(&xy_plane_kernel<false>),
                                    200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const long long planes = static_cast<long long>(Mz) * E;
  if (planes > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int split_n = inverse ? My : Ly;
  long long parts = (2LL * kNumSMs + planes - 1) / planes;  // fill >= 2 CTAs per SM
  if (parts > split_n) parts = split_n;
  if (parts < 1) parts = 1;
  const dim3 grid(static_cast<unsigned>(planes), static_cast<unsigned>(parts));
  if (inverse)
    xy_plane_kernel<true><<<grid, 256, smem, stream>>>(in, out, twx, twy, Mx, My, Lx, Ly, E, static_cast<int>(parts),
                                                       scale);
  else
    xy_plane_kernel<false><<<grid, 256, smem, stream>>>(in, out, twx, twy, Mx, My, Lx, Ly, E, static_cast<int>(parts),
                                                        scale);
  return cudaGetLastError();
}

cudaError_t launch_p2m(const c64* v0t, const c64* x, c64* mom, int n, int b, long long N, int nrhs, int cells,
                       cudaStream_t stream) {
  if (cells == 0 || nrhs == 0) return cudaSuccess;
  static const int gemm_mode = [] {  // FPBEM_P2M_GEMM=0: the FMA kernel for every rhs count; =2: GEMM for all
    const char* v = std::getenv("FPBEM_P2M_GEMM");
    return v ? std::atoi(v) : 1;
  }();
  const size_t smem = sizeof(c64) * static_cast<size_t>(b) * p2m_pitch(n);
  if (gemm_mode != 0 && (nrhs >= 4 || gemm_mode == 2) && smem <= 200 * 1024) {
    static std::atomic<unsigned long long> configured{0};
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&p2m_gemm_kernel), 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    const long long tiles = (static_cast<long long>(cells) * nrhs + 7) / 8;
    const int grid = static_cast<int>(std::min<long long>(kNumSMs, (tiles + kP2mWarps - 1) / kP2mWarps));
    p2m_gemm_kernel<<<grid, kP2mWarps * 32, smem, stream>>>(v0t, x, mom, n, b, N, nrhs, cells);
    return cudaGetLastError();
  }
  const long long blocks = static_cast<long long>(cells) * nrhs;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (blocks >= 4LL * kNumSMs) {
    p2m_kernel<4><<<dim3(static_cast<unsigned>(blocks), (b + 31) / 32), 256, 0, stream>>>(v0t, x, mom, n, b, N, nrhs);
  } else {
    p2m_kernel<1><<<dim3(static_cast<unsigned>(blocks), (b + 7) / 8), 256, 0, stream>>>(v0t, x, mom, n, b, N, nrhs);
  }
  return cudaGetLastError();
}

cudaError_t launch_mode_product(const c64* lambda, const c64* field, c64* image, long long q_total, int b,
                                int nrhs, cudaStream_t stream) {
  // the tensor-core contraction from 4 right-hand sides on (FPBEM_MODE_GEMM=0 disables)
  static const bool gemm_on = [] {
    const char* v = std::getenv("FPBEM_MODE_GEMM");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const size_t smem = sizeof(c64) * (static_cast<size_t>(b) * b + static_cast<size_t>(kModeRows) * (b | 1));
  if (gemm_on && nrhs >= 4 && smem <= 200 * 1024) {
    static std::atomic<unsigned long long> configured{0};
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&mode_gemm_kernel), 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    const dim3 grid(static_cast<unsigned>(q_total), static_cast<unsigned>((nrhs + kModeRows - 1) / kModeRows));
    mode_gemm_kernel<<<grid, 256, smem, stream>>>(lambda, field, image, b, nrhs);
    return cudaGetLastError();
  }
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

namespace {
size_t zpipe_fields_bytes(int Mz, int Lz, int E) {
  return sizeof(c64) * (static_cast<size_t>(4 * Mz + 4 * Lz) * E + Lz);  // inputs and f_z: 2 buffers x 2 columns
}
int zpipe_max_ring(int Mz, int Lz, int E, int b) {
  const size_t fields = zpipe_fields_bytes(Mz, Lz, E), per_mode = sizeof(c64) * static_cast<size_t>(b) * b;
  if (fields >= kZfSmemMax) return 0;
  long long r = static_cast<long long>((kZfSmemMax - fields) / per_mode);
  return static_cast<int>(r > kPipeMaxRing ? kPipeMaxRing : r);
}
// mode warps: FPBEM_ZF_MW (default 7); ring = the largest multiple of it that
// fits, at least two slots per warp (0: the fused kernel does not fit)
int zpipe_mode_warps(int Mz, int Lz, int E, int b) {
  static const int want = [] {
    const char* s = std::getenv("FPBEM_ZF_MW");
    const int v = s ? std::atoi(s) : 7;  // measured best on cfg3 / cfg5 (profiles/r01_m2l_probes.md)
    return v < 2 ? 2 : (v > kPipeMaxModeWarps ? kPipeMaxModeWarps : v);
  }();
  const int r = zpipe_max_ring(Mz, Lz, E, b);
  for (int w = want; w >= 2; --w)
    if (r >= 2 * w) return w;
  return 0;
}
}  // namespace

int m2l_zfused_ring(int Mz, int Lz, int E, int b) {
  const int w = zpipe_mode_warps(Mz, Lz, E, b);
  return w ? (zpipe_max_ring(Mz, Lz, E, b) / w) * w : 0;
}

cudaError_t launch_m2l_zfused(const c64* in, c64* out, const c64* lambda, const c64* tw, int Mz, int Lz,
                              long long plane, int E, int b, double scale, const int2* items, int n_items,
                              cudaStream_t stream) {
  const int n_mw = zpipe_mode_warps(Mz, Lz, E, b);
  if (n_mw == 0 || b > 256) return cudaErrorInvalidValue;
  const int ring = m2l_zfused_ring(Mz, Lz, E, b);
  const size_t smem = zpipe_fields_bytes(Mz, Lz, E) + sizeof(c64) * static_cast<size_t>(ring) * b * b;
  static std::atomic<unsigned long long> configured{0};
  if (smem > 48 * 1024) {
    if (smem > static_cast<size_t>(kMaxDynSmem)) return cudaErrorInvalidValue;
    cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&m2l_zpipe_kernel), kMaxDynSmem);
    if (e != cudaSuccess) return e;
  }
  const int grid = n_items < kNumSMs ? n_items : kNumSMs;  // persistent: one CTA per SM
  if (grid == 0) return cudaSuccess;
  static const int use_mma = [] {
    const char* v = std::getenv("FPBEM_ZF_DFT");
    const char* pr = std::getenv("FPBEM_ZF_PROBE");
    const int probe = pr ? std::atoi(pr) : 0;
    return ((v && std::strcmp(v, "fma") == 0) ? 0 : 1) | (probe == 1 ? 2 : 0) | (probe == 2 ? 4 : 0);
  }();
  m2l_zpipe_kernel<<<grid, 32 * (1 + n_mw + kPipeMaxDftWarps), smem, stream>>>(
      in, out, lambda, tw, Mz, Lz, plane, E, b, n_mw, ring, kPipeMaxDftWarps, scale, items, n_items, use_mma);
  return cudaGetLastError();
}

// consumer warps and ring of the flat mode stream: the most warps (FPBEM_MS_WARPS, default 11)
// that still get FPBEM_MS_SPW (default 1) slots each, ring = the largest multiple that fits.
// Measured on cfg3 (M2L stage, serial): 9 warps x 2 slots 84.6 us, 9 x 1 84.5, 11 x 1 78.4 —
// with four products per block the consumers bind, not the ring depth (0: shape not
// supported — b > 32 or too many fields per mode)
namespace {
void mode_stream_shape(int E, int b, int* n_w, int* ring) {
  *n_w = *ring = 0;
  if (b < 1 || b > 32 || E > 32 * kStreamRegs) return;
  static const int want = [] {
    const char* v = std::getenv("FPBEM_MS_WARPS");
    const int w = v ? std::atoi(v) : kStreamWarps;
    return w < 1 ? 1 : (w > kStreamWarps ? kStreamWarps : w);
  }();
  static const int spw_min = [] {  // FPBEM_MS_SPW: least slots per warp (A/B)
    const char* v = std::getenv("FPBEM_MS_SPW");
    const int w = v ? std::atoi(v) : 1;
    return w < 1 ? 1 : w;
  }();
  static const int ring_cap = [] {  // FPBEM_MS_RING: most ring slots (a small ring lets the kernel share an SM)
    const char* v = std::getenv("FPBEM_MS_RING");
    return v ? std::atoi(v) : 0;
  }();
  const size_t per_mode = sizeof(c64) * static_cast<size_t>(b) * b;
  for (int w = want; w >= 1; --w) {
    const size_t stage = sizeof(c64) * static_cast<size_t>(w) * 4 * E;
    long long r = static_cast<long long>((200 * 1024 - stage) / per_mode);
    if (r > kStreamMaxRing) r = kStreamMaxRing;
    if (ring_cap > 0 && r > ring_cap) r = ring_cap;
    if (r >= static_cast<long long>(spw_min) * w || (w == 1 && r >= 2)) {
      *n_w = w;
      *ring = static_cast<int>(r / w) * w;
      return;
    }
  }
}
}  // namespace

int mode_stream_ring(int E, int b) {
  int n_w, ring;
  mode_stream_shape(E, b, &n_w, &ring);
  return ring;
}

cudaError_t launch_mode_stream(c64* field, const c64* lambda, int Lz, long long plane, int E, int b,
                               const int2* items, int n_items, bool quad, cudaStream_t stream) {
  int n_w, ring;
  mode_stream_shape(E, b, &n_w, &ring);
  if (ring < 2) return cudaErrorInvalidValue;
  const int qz_count = quad ? Lz / 2 + 1 : Lz;  // quad: the modes qz <= Lz/2 determine the rest
  const long long total = static_cast<long long>(n_items) * qz_count;
  if (total == 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidValue;  // 32-bit unit arithmetic in the kernel
  const size_t smem = sizeof(c64) * (static_cast<size_t>(ring) * b * b + static_cast<size_t>(n_w) * 4 * E);
  static std::atomic<unsigned long long> configured{0};
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&mode_stream_kernel), kMaxDynSmem);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sms();
  const int grid = static_cast<int>(total < sms ? total : sms);  // persistent: one CTA per SM
  static const int probe = [] {
    const char* v = std::getenv("FPBEM_MS_PROBE");
    return v ? std::atoi(v) : 0;
  }();
  if (probe & 8) return cudaSuccess;  // FPBEM_MS_PROBE=8 (diagnostic, wrong results): the DFT passes alone
  mode_stream_kernel<<<grid, 32 * (1 + n_w), smem, stream>>>(field, lambda, Lz, qz_count, plane, E, b, ring, items,
                                                              n_items, quad ? 1 : 0, probe);
  return cudaGetLastError();
}

// max |Λ(-q) - D Λ(q) D| and max |Λ| (component-wise, as bit patterns of
// non-negative doubles) over the whole spectrum; zflip: the reflection parity
// max |Λ(qx, qy, -qz) - Dz Λ(q) Dz| with Dz = diag((-1)^(n+m)) instead
__global__ void lambda_parity_kernel(const c64* __restrict__ lam, int Lx, int Ly, int Lz, int b, int zflip,
                                     unsigned long long* __restrict__ out) {
  const long long q_total = static_cast<long long>(Lx) * Ly * Lz, b2 = static_cast<long long>(b) * b;
  double dmax = 0.0, amax = 0.0;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < q_total * b2;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = g / b2, e = g - q * b2;
    const int qx = static_cast<int>(q % Lx), qy = static_cast<int>((q / Lx) % Ly), qz = static_cast<int>(q / Lx / Ly);
    const long long qm = zflip ? (static_cast<long long>((Lz - qz) % Lz) * Ly + qy) * Lx + qx
                               : (static_cast<long long>((Lz - qz) % Lz) * Ly + (Ly - qy) % Ly) * Lx + (Lx - qx) % Lx;
    const int i = static_cast<int>(e % b), j = static_cast<int>(e / b);  // column-major block
    int ni = 0, nj = 0;
    while ((ni + 1) * (ni + 1) <= i) ++ni;
    while ((nj + 1) * (nj + 1) <= j) ++nj;
    // coefficient i = n^2 + n + m: n + m = i - n^2
    const int par = zflip ? (i - ni * ni) + (j - nj * nj) : ni + nj;
    const double sg = (par & 1) ? -1.0 : 1.0;
    const c64 a = lam[q * b2 + e], m = lam[qm * b2 + e];
    dmax = fmax(dmax, fmax(fabs(m.x - sg * a.x), fabs(m.y - sg * a.y)));
    amax = fmax(amax, fmax(fabs(a.x), fabs(a.y)));
  }
  atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(dmax)));
  atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
}

cudaError_t launch_lambda_parity(const c64* lam, const int L[3], int b, bool zflip, unsigned long long* out2,
                                 cudaStream_t stream) {
  const long long total = static_cast<long long>(L[0]) * L[1] * L[2] * b * b;
  lambda_parity_kernel<<<grid_for(total, 256), 256, 0, stream>>>(lam, L[0], L[1], L[2], b, zflip ? 1 : 0, out2);
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
