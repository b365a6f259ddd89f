// Near-field block-Toeplitz product on FP64 tensor cores (DMMA), plus the
// fixed-order offset reduction fused with the L2P epilogue.
//
// Reference: BlockToeplitzMatrix::matvec (src/assembly.cpp:62-84) computes,
// for every target cell t and every stored offset o (insertion order),
// y_t += S_o p_{t-o} as one GEMV per (t, o) pair — each S_o is re-streamed
// per pair. Here each offset is one GEMM over all of its valid target cells
// (and right-hand sides): W[:, pairs(o)] = S_o * P[:, sources(o)], so S_o is
// read from HBM once per column tile instead of once per pair. The partial
// products land in a pair-major workspace W and are summed per target in the
// reference's offset order by near_reduce_l2p_kernel, which also adds the
// L2P term U0 * L_t (src/fmm.cpp:265-267) — no atomics, deterministic.
//
// Complex arithmetic: C_re += A_re B_re - A_im B_im, C_im += A_re B_im + A_im B_re,
// four real m8n8k4 DMMAs per complex 8x8x4 tile.
#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {

constexpr int BM = 64;   // rows of S (targets' collocation points) per CTA
constexpr int BN = 64;   // (pair, rhs) columns per CTA
constexpr int BK = 16;   // complex k per pipeline stage
constexpr int STAGES = 3;
constexpr int AP = BM + 2;  // smem pitch (complex) of the [k][m] A tile: 16B-bank conflict free
constexpr int BP = BK + 4;  // smem pitch (complex) of the [n][k] B tile
constexpr int THREADS = 256;

constexpr size_t kSmemA = sizeof(c64) * STAGES * BK * AP;
constexpr size_t kSmemB = sizeof(c64) * STAGES * BN * BP;

__global__ void __launch_bounds__(THREADS, 2)
near_gemm_dmma_kernel(const c64* __restrict__ S, const c64* __restrict__ x, c64* __restrict__ W,
                      const int* __restrict__ pair_src, const int4* __restrict__ jobs, int n,
                      long long N, int nrhs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  c64* As = reinterpret_cast<c64*>(smem_raw);
  c64* Bs = reinterpret_cast<c64*>(smem_raw + kSmemA);
  __shared__ long long col_src[BN];
  __shared__ long long col_out[BN];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * BM;
  const int4 job = jobs[blockIdx.y];  // (offset slot, first column, column count, pair base)
  const int s = job.x, col0 = job.y, ncols = job.z, pair_base = job.w;

  if (tid < BN) {
    if (tid < ncols) {
      const int gc = col0 + tid;
      const int pair = pair_base + gc / nrhs;
      const int r = gc % nrhs;
      col_src[tid] = static_cast<long long>(r) * N + static_cast<long long>(pair_src[pair]) * n;
      col_out[tid] = (static_cast<long long>(pair_base) * nrhs + gc) * n;
    } else {
      col_src[tid] = -1;
      col_out[tid] = -1;
    }
  }
  __syncthreads();

  const c64* Sblk = S + static_cast<size_t>(s) * n * n;
  const int nk = (n + BK - 1) / BK;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    c64* as = As + stage * BK * AP;
    c64* bs = Bs + stage * BN * BP;
#pragma unroll
    for (int i = 0; i < (BM * BK) / THREADS; ++i) {
      const int e = tid + i * THREADS;
      const int kk = e / BM, mm = e % BM;
      const int gk = k0 + kk, gm = m0 + mm;
      const bool ok = gk < n && gm < n;
      cp_async16(as + kk * AP + mm, ok ? Sblk + static_cast<size_t>(gk) * n + gm : Sblk, ok);
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / THREADS; ++i) {
      const int e = tid + i * THREADS;
      const int c = e / BK, kk = e % BK;
      const long long src = col_src[c];
      const bool ok = src >= 0 && (k0 + kk) < n;
      cp_async16(bs + c * BP + kk, ok ? x + src + k0 + kk : x, ok);
    }
  };

  double cre[4][2][2], cim[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      cre[mi][ni][0] = cre[mi][ni][1] = 0.0;
      cim[mi][ni][0] = cim[mi][ni][1] = 0.0;
    }

  const int wm = warp & 1;   // 32-row slab
  const int wn = warp >> 1;  // 16-column slab
  const int fr = lane >> 2, fk = lane & 3;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load_stage(st, st);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < nk) load_stage(pf % STAGES, pf);
    cp_async_commit();

    const c64* as = As + (kt % STAGES) * BK * AP;
    const c64* bs = Bs + (kt % STAGES) * BN * BP;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      c64 a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = as[(k4 * 4 + fk) * AP + wm * 32 + mi * 8 + fr];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = bs[(wn * 16 + ni * 8 + fr) * BP + k4 * 4 + fk];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma884(cre[mi][ni][0], cre[mi][ni][1], a[mi].x, b[ni].x);
          dmma884(cre[mi][ni][0], cre[mi][ni][1], a[mi].y, -b[ni].y);
          dmma884(cim[mi][ni][0], cim[mi][ni][1], a[mi].x, b[ni].y);
          dmma884(cim[mi][ni][0], cim[mi][ni][1], a[mi].y, b[ni].x);
        }
    }
  }
  cp_async_wait<0>();

  // epilogue: accumulator (row fr, cols 2*fk + {0,1}) of each 8x8 tile
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int gm = m0 + wm * 32 + mi * 8 + fr;
    if (gm >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = wn * 16 + ni * 8 + 2 * fk + j;
        const long long out = col_out[c];
        if (out >= 0) W[out + gm] = cmk(cre[mi][ni][j], cim[mi][ni][j]);
      }
  }
}

// y[r,t,i] = sum_{pairs of t, offset order} W[pair, r, i]  +  sum_m U0[i, m] L[t, r, m]
// One thread per row i; grid (row tiles, target cells * nrhs).
constexpr int RED_THREADS = 128;
constexpr int MAX_COEF = 64;

__global__ void __launch_bounds__(RED_THREADS)
near_reduce_l2p_kernel(const c64* __restrict__ W, const int* __restrict__ tgt_ptr,
                       const int* __restrict__ tgt_pairs, const c64* __restrict__ u0,
                       const c64* __restrict__ local, c64* __restrict__ y, int n, int n_coef,
                       long long N, int nrhs, int accumulate) {
  __shared__ c64 loc[MAX_COEF];
  const int tr = blockIdx.y;  // t * nrhs + r
  const int t = tr / nrhs, r = tr % nrhs;
  if (local != nullptr && threadIdx.x < n_coef)
    loc[threadIdx.x] = local[static_cast<size_t>(tr) * n_coef + threadIdx.x];
  __syncthreads();
  const int i = blockIdx.x * RED_THREADS + threadIdx.x;
  if (i >= n) return;
  const int p0 = tgt_ptr[t], p1 = tgt_ptr[t + 1];
  c64 acc = cmk(0.0, 0.0);
  int p = p0;
  // batches of independent loads, summed in offset order
  for (; p + 8 <= p1; p += 8) {
    c64 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long pr = tgt_pairs[p + u];
      v[u] = W[(pr * nrhs + r) * n + i];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = cadd(acc, v[u]);
  }
  for (; p < p1; ++p) {
    const long long pr = tgt_pairs[p];
    acc = cadd(acc, W[(pr * nrhs + r) * n + i]);
  }
  if (local != nullptr) {
    c64 l2p = cmk(0.0, 0.0);
    for (int m = 0; m < n_coef; ++m) l2p = cfma(u0[static_cast<size_t>(m) * n + i], loc[m], l2p);
    acc = cadd(acc, l2p);
  }
  c64* dst = y + static_cast<size_t>(r) * N + static_cast<size_t>(t) * n + i;
  if (accumulate) acc = cadd(*dst, acc);
  *dst = acc;
}

}  // namespace

size_t near_gemm_smem_bytes() { return kSmemA + kSmemB; }
int near_gemm_tile_cols() { return BN; }
int near_gemm_tile_rows() { return BM; }

cudaError_t launch_near_gemm(const c64* S, const c64* x, c64* W, const int* pair_src, const int4* jobs,
                             int n_jobs, int n, long long N, int nrhs, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(near_gemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemA + kSmemB));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_jobs == 0) return cudaSuccess;
  dim3 grid((n + BM - 1) / BM, n_jobs);
  near_gemm_dmma_kernel<<<grid, THREADS, kSmemA + kSmemB, stream>>>(S, x, W, pair_src, jobs, n, N, nrhs);
  return cudaGetLastError();
}

cudaError_t launch_near_reduce_l2p(const c64* W, const int* tgt_ptr, const int* tgt_pairs, const c64* u0,
                                   const c64* local, c64* y, int n, int n_coef, int n_cells, long long N,
                                   int nrhs, bool accumulate, cudaStream_t stream) {
  if (n_coef > MAX_COEF) return cudaErrorInvalidValue;
  dim3 grid((n + RED_THREADS - 1) / RED_THREADS, n_cells * nrhs);
  near_reduce_l2p_kernel<<<grid, RED_THREADS, 0, stream>>>(W, tgt_ptr, tgt_pairs, u0, local, y, n, n_coef, N,
                                                           nrhs, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
