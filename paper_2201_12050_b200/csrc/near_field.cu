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
// Complex arithmetic: the Gauss 3-multiplication form (three real m8n8k4
// DMMAs per complex 8x8x4 tile instead of four); the algorithmic count stays
// 8 real flops per complex multiply-add.
#include <algorithm>
#include <cstdlib>
#include <cstring>

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

// K loop + epilogue of one CTA tile. Gauss 3-multiplication complex product
// on the FP64 tensor cores: T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi);
// Cr = T1 - T2, Ci = T3 - T1 - T2. A warp owns MI x NI 8x8 tiles: warps form
// (8 / MI) row groups of 8 MI rows x MI column groups of 8 NI columns, covering
// 64 rows x 8 MI NI columns. Per 4-deep k step a warp loads MI + NI fragments
// from shared memory for 3 MI NI DMMAs (NI = 2 halves the A re-reads of NI = 1,
// where every warp loaded all 64 rows: shared-memory bandwidth was the limiter).
template <int MI, int NI, typename Loader>
__device__ __forceinline__ void gemm_main(const c64* As, const c64* Bs, Loader& load_stage, int nk, int warp, int lane,
                                          int ncols, int m0, int M, const long long* col_out, c64* __restrict__ out,
                                          const int* col_g, const int* __restrict__ perm) {
  constexpr int G = 8 / MI;  // row groups
  const int wm = warp % G, wn = warp / G;
  const int fr = lane >> 2, fk = lane & 3;
  const bool active = wn * 8 * NI < ncols;
  double t1[MI][NI][2], t2[MI][NI][2], t3[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      t1[mi][ni][0] = t1[mi][ni][1] = 0.0;
      t2[mi][ni][0] = t2[mi][ni][1] = 0.0;
      t3[mi][ni][0] = t3[mi][ni][1] = 0.0;
    }

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
    if (!active) continue;

    const c64* as = As + (kt % STAGES) * BK * AP + wm * (8 * MI);
    const c64* bs = Bs + (kt % STAGES) * BN * BP + wn * (8 * NI) * BP;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      c64 b[NI], a[MI];
      double bsum[NI], asum[MI];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        b[ni] = bs[(ni * 8 + fr) * BP + k4 * 4 + fk];
        bsum[ni] = b[ni].x + b[ni].y;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        a[mi] = as[(k4 * 4 + fk) * AP + mi * 8 + fr];
        asum[mi] = a[mi].x + a[mi].y;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          dmma884(t1[mi][ni][0], t1[mi][ni][1], a[mi].x, b[ni].x);
          dmma884(t2[mi][ni][0], t2[mi][ni][1], a[mi].y, b[ni].y);
          dmma884(t3[mi][ni][0], t3[mi][ni][1], asum[mi], bsum[ni]);
        }
    }
  }
  cp_async_wait<0>();
  if (!active) return;

  // epilogue: accumulator (row fr, cols 2*fk + {0,1}) of each 8x8 tile
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int gm = m0 + wm * (8 * MI) + mi * 8 + fr;
    if (gm >= M) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = wn * 8 * NI + ni * 8 + 2 * fk + j;
        const long long o = col_out[c];
        const int g = col_g[c];  // image column: its rows land at P_g[row]
        if (o >= 0)
          out[o + (g ? __ldg(perm + static_cast<size_t>(g - 1) * M + gm) : gm)] =
              cmk(t1[mi][ni][j] - t2[mi][ni][j], t3[mi][ni][j] - t1[mi][ni][j] - t2[mi][ni][j]);
      }
  }
}

// Batched block GEMM over (block, column-tile) jobs:
//   out[col_out(c) + m] = sum_k A_s[m + lda k] * x[col_src(c) + k],  m < M, k < K
// Near field: A_s = S_s (lda = M = K = n), columns = (pair, rhs) of offset s,
//   col_src = rhs*N + pair_src[pair]*n, col_out = (pair*nrhs + rhs)*ldo;
// with pair_src == nullptr the columns are (cell, rhs) of one block.
// Warps whose 8-column slab lies beyond the job's column count skip the MMA
// loop, so partial column tiles cost (almost) only their useful work.
// 2 CTAs per SM (128 registers): measured 15-17 % faster than one CTA with the
// 154 registers the compiler takes when uncapped
__global__ void __launch_bounds__(THREADS, 2)
near_gemm_dmma_kernel(const c64* __restrict__ A, long long a_stride, int lda, int M, const c64* __restrict__ x,
                      c64* __restrict__ out, int ldo, const int* __restrict__ pair_src, const int4* __restrict__ jobs,
                      int K, int n, long long N, int nrhs, long long out_rhs_stride, const int* __restrict__ perm,
                      const int* __restrict__ items, long long n_items) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  c64* As = reinterpret_cast<c64*>(smem_raw);
  c64* Bs = reinterpret_cast<c64*>(smem_raw + kSmemA);
  __shared__ long long col_src[BN];
  __shared__ long long col_out[BN];
  __shared__ int col_g[BN];  // symmetry map of the column (0: none)

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int m_tiles = (M + BM - 1) / BM;
  const int m0 = static_cast<int>(blockIdx.x % m_tiles) * BM;
  const int4 job = jobs[blockIdx.x / m_tiles];  // (block slot, first column, count | class << 8, pair base)
  const int s = job.x, col0 = job.y, ncols = job.z & 0xff, cls = (job.z >> 8) & 0xf, pair_base = job.w;
  // image-mode tile of the lattice near field: rows of B gathered and rows of
  // the output scattered through the symmetry permutation P_g (g = bits 12-14)
  const int gsym = (job.z >> 12) & 7;
  // bit 15: the columns are (image, rhs) pairs of stored block s's whole orbit
  // (items[s]: its up-to-8 image modes and maps), so the block is read once
  // for every image instead of once per image
  const bool orbit = (job.z >> 15) & 1;

  if (tid < BN) {
    if (tid < ncols) {
      const int gc = col0 + tid;
      const int r = gc % nrhs;
      if (orbit) {
        const int v = gc / nrhs;  // the v-th image of the orbit with a mode
        int q = -1, g = 0;
        for (int i = 0, cnt = 0; i < 8; ++i) {
          const int qi = items[static_cast<long long>(s) * 8 + i];
          if (qi < 0) continue;
          if (cnt++ == v) {
            q = qi;
            g = items[(n_items + s) * 8 + i];
            break;
          }
        }
        col_src[tid] = static_cast<long long>(r) * N + static_cast<long long>(q) * n;
        col_out[tid] = r * out_rhs_stride + static_cast<long long>(q) * ldo;
        col_g[tid] = g;
      } else {
        const int unit = pair_base + gc / nrhs;  // pair (near field) or cell (P2M)
        const long long cell = pair_src ? pair_src[unit] : unit;
        col_src[tid] = static_cast<long long>(r) * N + cell * n;
        col_out[tid] = out_rhs_stride > 0 ? r * out_rhs_stride + static_cast<long long>(unit) * ldo
                                          : (static_cast<long long>(pair_base) * nrhs + gc) * ldo;
        col_g[tid] = gsym;
      }
    } else {
      col_src[tid] = -1;
      col_out[tid] = -1;
      col_g[tid] = 0;
    }
  }
  __syncthreads();

  const c64* Ablk = A + static_cast<size_t>(s) * a_stride;
  const int nk = (K + BK - 1) / BK;

  // per-thread load coordinates: A rows (tid % BM) of k-columns tid / BM + 4 i,
  // B k-entries (tid % BK) of columns tid / BK + 16 i
  const int a_m = tid % BM, a_k = tid / BM;
  const bool a_row_ok = m0 + a_m < M;
  const c64* a_src = Ablk + static_cast<size_t>(a_k) * lda + m0 + a_m;
  const int b_k = tid % BK, b_c = tid / BK;
  const unsigned smem_a = static_cast<unsigned>(__cvta_generic_to_shared(As + a_k * AP + a_m));
  const unsigned smem_b = static_cast<unsigned>(__cvta_generic_to_shared(Bs + b_c * BP + b_k));

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
#pragma unroll
    for (int i = 0; i < (BM * BK) / THREADS; ++i) {
      const int kk = a_k + i * (THREADS / BM);
      const bool ok = a_row_ok && k0 + kk < K;
      const c64* src = ok ? a_src + static_cast<size_t>(k0 + i * (THREADS / BM)) * lda : Ablk;
      const unsigned dst = smem_a + sizeof(c64) * (stage * BK * AP + i * (THREADS / BM) * AP);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / THREADS; ++i) {
      const long long src_off = col_src[b_c + i * (THREADS / BK)];
      const int g = col_g[b_c + i * (THREADS / BK)];  // B rows gathered through P_g
      const bool ok = src_off >= 0 && (k0 + b_k) < K;
      const c64* src = ok ? x + src_off + (g ? __ldg(perm + static_cast<size_t>(g - 1) * K + k0 + b_k) : k0 + b_k) : x;
      const unsigned dst = smem_b + sizeof(c64) * (stage * BN * BP + i * (THREADS / BK) * BP);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
    }
  };

  // width class of the column tile: 0 -> 64 columns (warps 32 rows x 16),
  // 1 -> 32 columns (16 x 16), 2 -> 16 columns (8 x 16): narrow tiles keep
  // all 8 warps busy instead of idling most of them
  switch (cls) {
    case 0: gemm_main<4, 2>(As, Bs, load_stage, nk, warp, lane, ncols, m0, M, col_out, out, col_g, perm); break;
    case 1: gemm_main<2, 2>(As, Bs, load_stage, nk, warp, lane, ncols, m0, M, col_out, out, col_g, perm); break;
    default: gemm_main<1, 2>(As, Bs, load_stage, nk, warp, lane, ncols, m0, M, col_out, out, col_g, perm); break;
  }
}

// Near field as a lattice convolution: per Fourier mode q of
// the near-field embedding, yh[r][q] = Shat_q xh[r][q] with Shat_q the n x n
// column-major block of the lattice DFT of the embedded S_o (the same circulant
// embedding CirculantSpectrum uses for K, src/structured.cpp:63-108, applied to
// the Toeplitz blocks of BlockToeplitzMatrix, src/assembly.cpp:62-84). For a few
// right-hand sides this is a streaming complex GEMV over all modes: one thread
// per row, the k loop in fixed ascending order (deterministic), the block read
// once with 8 independent 16-byte loads in flight per thread, the RHS chunk
// staged in shared memory. HBM-bound: 16 n^2 bytes per stored block.
// Work item t = an orbit of modes under the cell's verified symmetries: block
// t of the stored spectrum is Shat(q_0), and image mode q_i = A_g q_0 has
// Shat(q_i) = P_g Shat(q_0) P_g, so the same stream also gives
// yh[q_i] = P_g Shat(q_0) P_g xh[q_i]: image i's accumulators read xh[q_i]
// gathered through P_g and its rows land at P_g[row].
constexpr int GEMV_THREADS = 128;
constexpr int GEMV_KC = 256;  // k chunk of xh staged in shared memory
constexpr int GEMV_U = 8;     // independent Shat loads per thread

template <int R, int NI>
__global__ void __launch_bounds__(GEMV_THREADS)
near_mode_gemv_kernel(const c64* __restrict__ shat, const int* __restrict__ items, long long n_items,
                      const int* __restrict__ perm, const c64* __restrict__ xh, c64* __restrict__ yh, int n,
                      long long t_lo, long long q_stride, int row_tiles) {
  constexpr int A = NI * R;  // accumulators per thread
  __shared__ c64 xs[A][GEMV_KC];
  __shared__ int iq[8], ig[8];
  const long long t = t_lo + blockIdx.x / row_tiles;
  if (threadIdx.x < 8) {
    iq[threadIdx.x] = items[t * 8 + threadIdx.x];
    ig[threadIdx.x] = items[(n_items + t) * 8 + threadIdx.x];
  }
  const int i = (blockIdx.x % row_tiles) * GEMV_THREADS + threadIdx.x;
  const bool row_ok = i < n;
  const size_t nn = static_cast<size_t>(n) * n;
  const c64* a = shat + static_cast<size_t>(t) * nn + (row_ok ? i : 0);
  c64 acc[A];
#pragma unroll
  for (int r = 0; r < A; ++r) acc[r] = cmk(0.0, 0.0);
  for (int k0 = 0; k0 < n; k0 += GEMV_KC) {
    const int kc = min(GEMV_KC, n - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < A * GEMV_KC; e += GEMV_THREADS) {
      const int slot = e / GEMV_KC, k = e % GEMV_KC;
      const int img = slot / R, r = slot % R;
      const int q = iq[img];
      c64 v = cmk(0.0, 0.0);
      if (k < kc && q >= 0) {
        const int g = ig[img];
        const int kk = g ? __ldg(perm + static_cast<size_t>(g - 1) * n + k0 + k) : k0 + k;
        v = xh[r * q_stride * n + static_cast<long long>(q) * n + kk];
      }
      xs[slot][k] = v;
    }
    __syncthreads();
    int k = 0;
    for (; k + GEMV_U <= kc; k += GEMV_U) {
      c64 v[GEMV_U];
#pragma unroll
      for (int u = 0; u < GEMV_U; ++u) v[u] = __ldcs(a + static_cast<size_t>(k0 + k + u) * n);
#pragma unroll
      for (int u = 0; u < GEMV_U; ++u)
#pragma unroll
        for (int r = 0; r < A; ++r) acc[r] = cfma(v[u], xs[r][k + u], acc[r]);
    }
    for (; k < kc; ++k) {
      const c64 v = __ldcs(a + static_cast<size_t>(k0 + k) * n);
#pragma unroll
      for (int r = 0; r < A; ++r) acc[r] = cfma(v, xs[r][k], acc[r]);
    }
  }
  if (!row_ok) return;
#pragma unroll
  for (int img = 0; img < NI; ++img) {
    const int q = iq[img];
    if (q < 0) continue;
    const int g = ig[img];
    const int row = g ? __ldg(perm + static_cast<size_t>(g - 1) * n + i) : i;
#pragma unroll
    for (int r = 0; r < R; ++r) yh[r * q_stride * n + static_cast<long long>(q) * n + row] = acc[img * R + r];
  }
}

// Same product as near_mode_gemv_kernel on the FP64 tensor cores, for up to 8
// columns per stored block (right-hand sides x images, e.g. the 8 images of
// an orbit under the icosphere's axis-sign group on cfg3/cfg5). The GEMV's
// 8 complex FMAs per streamed element left it bound between the FP64 pipe and
// load latency at ~0.5 of HBM. Here:
//   * persistent CTAs, one per SM, walking the stored blocks t = blockIdx.x,
//     blockIdx.x + gridDim.x, ...;
//   * a producer warp streams each block column by column with
//     cp.async.bulk (evict-first: the 1.2 GB stream must not push x_hat out of
//     L2) into a ring of KC-column stages (full / empty mbarriers), running
//     ahead across block boundaries, so HBM never waits on the math;
//   * NW consumer warps own n / 8 / NW row tiles each: per 4-deep k step one
//     A fragment per row tile from the ring (column pitch n + 2 complex:
//     conflict-free 16-byte fragment loads), one B fragment of the block's
//     8 columns, and the Gauss 3-multiplication complex product on
//     mma.sync.m8n8k4.f64 (3 DMMAs per complex 8x8x4 tile);
//   * the block's columns X[c][k] = xh[r][q_img][P_g k] are gathered from L2
//     into shared memory at the block's start, and the epilogue scatters the
//     rows through P_g into yh[r][q_img].
// Fixed summation order (k ascending in groups of 4): bitwise repeatable.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void cp_async16_zfill(unsigned dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
// arrive on `bar` when all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

template <int MT, int NW>
__global__ void __launch_bounds__(32 * (NW + 2), 1)
near_mode_mma_kernel(const c64* __restrict__ shat, const int* __restrict__ items, long long n_items,
                     const int* __restrict__ perm, const c64* __restrict__ xh, c64* __restrict__ yh, int n,
                     long long t_lo, long long t_hi, long long q_stride, int nrhs, int ncols, int KC, int ring,
                     int rsplit, int nxb) {
  // work unit u = (stored block t, row part h): rsplit parts of the block's row
  // tiles per block, so that few blocks (a slab rank's share) still fill every SM
  extern __shared__ __align__(128) unsigned char mm_smem[];
  const int AP = n + 2, XP = n + 4;  // complex pitches: A columns, X columns
  c64* As = reinterpret_cast<c64*>(mm_smem);
  c64* Xs = As + static_cast<size_t>(ring) * KC * AP;  // two X buffers of 8 columns
  // barriers: full[ring], empty[ring], xfull[2], xempty[2]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(Xs + nxb * 8 * XP);  // nxb X buffers
  __shared__ int iq[2][8], ig[2][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + ring), xfull0 = smem_u32(bars + 2 * ring),
                 xempty0 = smem_u32(bars + 2 * ring + 2);
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, NW);
    }
    for (int i = 0; i < 2; ++i) {
      // the producer warp's 32 lanes through cp.async.mbarrier.arrive.noinc (their gathers
      // landed) + one plain release arrive after the block's (iq, ig) were written
      mbar_init(xfull0 + 8 * i, 33);
      mbar_init(xempty0 + 8 * i, NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int stages = (n + KC - 1) / KC;  // per stored block
  const size_t nn = static_cast<size_t>(n) * n;
  const long long u_lo = t_lo * rsplit, u_hi = t_hi * rsplit;
  const int n_mt_all = n >> 3;
  auto part_rows = [&](long long u, int* m0, int* m1) {  // row tiles [m0, m1) of unit u
    const int h = static_cast<int>(u % rsplit);
    *m0 = h * n_mt_all / rsplit;
    *m1 = (h + 1) * n_mt_all / rsplit;
  };

  if (warp == NW + 1) {  // ---- X producer: the blocks' columns, up to two blocks ahead of the consumers
    // xh is the previous kernel's output (the block producer streams operator data and starts at
    // once; the consumers touch global memory only after an X buffer has arrived)
    pdl_wait();
    int it = 0;
    for (long long u = u_lo + blockIdx.x; u < u_hi; u += gridDim.x, ++it) {
      const long long t = u / rsplit;
      // X[c][k] = xh[r][q_img][P_g k] into X buffer it & 1, 16-byte cp.async per element
      const int xb = it % nxb;
      if (it >= nxb) mbar_wait(xempty0 + 8 * xb, ((it / nxb) - 1) & 1);
      int q8 = -1, g8 = 0;
      if (lane < 8) {
        q8 = items[t * 8 + lane];
        g8 = items[(n_items + t) * 8 + lane];
        iq[xb][lane] = q8;
        ig[xb][lane] = g8;
      }
      c64* xdst = Xs + xb * 8 * XP;
      for (int c = 0; c < 8; ++c) {
        const int img = c / nrhs, r = c - img * nrhs;
        const int q = __shfl_sync(0xffffffffu, q8, img), gg = __shfl_sync(0xffffffffu, g8, img);
        const bool ok = c < ncols && q >= 0;
        const c64* src = xh + (ok ? r * q_stride * n + static_cast<long long>(q) * n : 0);
        const int* pg = gg ? perm + static_cast<size_t>(gg - 1) * n : nullptr;
        constexpr int B = 8;  // permutation indices in flight per lane
        for (int k0 = 0; k0 < n; k0 += 32 * B) {
          int idx[B];
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const int k = k0 + lane + 32 * u;
            idx[u] = (k < n && pg) ? __ldg(pg + k) : k;
          }
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const int k = k0 + lane + 32 * u;
            if (k < n) cp_async16_zfill(smem_u32(xdst + c * XP + k), ok ? src + idx[u] : xh, ok);
          }
        }
      }
      cp_async_arrive_noinc(xfull0 + 8 * xb);
      __syncwarp();  // orders lanes 0-7's (iq, ig) stores before lane 0's release arrive
      if (lane == 0) mbar_arrive(xfull0 + 8 * xb);
    }
    return;
  }
  if (warp == NW) {  // ---- block producer: each stored block column by column into the ring
    if (lane == 0) {
      const unsigned long long pol = evict_first_policy();
      int slot = 0;
      unsigned ph = 0;
      for (long long u = u_lo + blockIdx.x; u < u_hi; u += gridDim.x) {
        int m0, m1;
        part_rows(u, &m0, &m1);
        const int rows = 8 * (m1 - m0);
        const c64* blk = shat + static_cast<size_t>(u / rsplit) * nn + 8 * m0;
        for (int st = 0; st < stages; ++st) {
          mbar_wait(empty0 + 8 * slot, ph ^ 1);
          const int k0 = st * KC, kc = min(KC, n - k0);
          mbar_arrive_expect_tx(full0 + 8 * slot, static_cast<unsigned>(kc * rows * sizeof(c64)));
          const unsigned dst = smem_u32(As + static_cast<size_t>(slot) * KC * AP);
          for (int c = 0; c < kc; ++c)
            bulk_g2s_hint(dst + static_cast<unsigned>(c * AP * sizeof(c64)), blk + static_cast<size_t>(k0 + c) * n,
                          static_cast<unsigned>(rows * sizeof(c64)), full0 + 8 * slot, pol);
          if (++slot == ring) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---- consumers
  const int fr = lane >> 2, fk = lane & 3;
  int slot = 0;
  unsigned ph = 0;
  int it = 0;
  for (long long u = u_lo + blockIdx.x; u < u_hi; u += gridDim.x, ++it) {
    int m0, m1;
    part_rows(u, &m0, &m1);
    const int n_mt = m1 - m0;  // this unit's row tiles; the ring holds rows 8 m0 ..
    const int xb = it % nxb;
    mbar_wait(xfull0 + 8 * xb, (it / nxb) & 1);
    const c64* xs = Xs + xb * 8 * XP + fr * XP + fk;

    double t1[MT][2], t2[MT][2], t3[MT][2];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) t1[mi][0] = t1[mi][1] = t2[mi][0] = t2[mi][1] = t3[mi][0] = t3[mi][1] = 0.0;
    for (int st = 0; st < stages; ++st) {
      mbar_wait(full0 + 8 * slot, ph);
      const c64* as = As + static_cast<size_t>(slot) * KC * AP + fk * AP + fr;
      const int k0 = st * KC, kc = min(KC, n - k0);
      for (int k4 = 0; k4 < kc; k4 += 4) {
        const c64 b = xs[k0 + k4];
        const double bsum = b.x + b.y;
        c64 a[MT];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
          const int mt = warp + mi * NW;
          a[mi] = mt < n_mt ? as[k4 * AP + mt * 8] : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
          if (warp + mi * NW < n_mt) {
            dmma884(t1[mi][0], t1[mi][1], a[mi].x, b.x);
            dmma884(t2[mi][0], t2[mi][1], a[mi].y, b.y);
            dmma884(t3[mi][0], t3[mi][1], a[mi].x + a[mi].y, bsum);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * slot);
      if (++slot == ring) {
        slot = 0;
        ph ^= 1;
      }
    }
    // epilogue: accumulator (row fr, columns 2 fk + {0, 1}) of each 8 x 8 tile
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      const int mt = warp + mi * NW;
      if (mt >= n_mt) continue;
      const int i = (m0 + mt) * 8 + fr;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = 2 * fk + j;
        if (c >= ncols) continue;
        const int img = c / nrhs, r = c - img * nrhs;
        const int q = iq[xb][img];
        if (q < 0) continue;
        const int gg = ig[xb][img];
        const int row = gg ? __ldg(perm + static_cast<size_t>(gg - 1) * n + i) : i;
        yh[r * q_stride * n + static_cast<long long>(q) * n + row] =
            cmk(t1[mi][j] - t2[mi][j], t3[mi][j] - t1[mi][j] - t2[mi][j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty0 + 8 * xb);  // X buffer and (iq, ig)[xb] free for block it + 2
  }
}

// y[r,t,i] = sum_{pairs of t, offset order} W[pair, r, i]  +  sum_m U0[i, m] L[t, r, m]
// One thread per row i; grid (row tiles, target cells * nrhs).
constexpr int RED_THREADS = 128;
constexpr int MAX_COEF = 256;  // n_t <= 15

__global__ void __launch_bounds__(RED_THREADS)
near_reduce_l2p_kernel(const c64* __restrict__ W, const int* __restrict__ tgt_ptr,
                       const int* __restrict__ tgt_pairs, const c64* __restrict__ u0,
                       const c64* __restrict__ local, c64* __restrict__ y, int n, int n_coef,
                       long long N, int nrhs, int accumulate) {
  __shared__ c64 loc[MAX_COEF];
  const int row_tiles = (n + RED_THREADS - 1) / RED_THREADS;
  const int tr = static_cast<int>(blockIdx.x / row_tiles);  // t * nrhs + r
  const int t = tr / nrhs, r = tr % nrhs;
  // strided: n_coef may exceed the CTA size (up to MAX_COEF = 256 for n_t <= 15)
  if (local != nullptr)
    for (int m = threadIdx.x; m < n_coef; m += RED_THREADS) loc[m] = local[static_cast<size_t>(tr) * n_coef + m];
  __syncthreads();
  const int i = static_cast<int>(blockIdx.x % row_tiles) * RED_THREADS + threadIdx.x;
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


cudaError_t launch_block_gemm(const c64* A, long long a_stride, int lda, int M, const c64* x, c64* out, int ldo,
                              const int* pair_src, const int4* jobs, int n_jobs, int K, int n, long long N, int nrhs,
                              cudaStream_t stream, long long out_rhs_stride, const int* perm, const int* items,
                              long long n_items) {
  static std::atomic<unsigned long long> configured{0};
  cudaError_t e = ensure_max_smem(configured, reinterpret_cast<const void*>(&near_gemm_dmma_kernel),
                                  static_cast<int>(kSmemA + kSmemB));
  if (e != cudaSuccess) return e;
  if (n_jobs == 0) return cudaSuccess;
  // 1-D grid, m-tiles of one job adjacent (they share the job's B columns in L2)
  const long long ctas = static_cast<long long>((M + BM - 1) / BM) * n_jobs;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(ctas));
  near_gemm_dmma_kernel<<<grid, THREADS, kSmemA + kSmemB, stream>>>(A, a_stride, lda, M, x, out, ldo, pair_src, jobs,
                                                                    K, n, N, nrhs, out_rhs_stride, perm, items,
                                                                    n_items);
  return cudaGetLastError();
}

cudaError_t launch_mode_gemv(const c64* shat, const int* items, long long n_items, const int* perm, const c64* xh,
                             c64* yh, int n, long long t_lo, long long t_hi, long long q_stride, int nrhs, int nimg,
                             cudaStream_t stream) {
  if (t_hi <= t_lo) return cudaSuccess;
  const int row_tiles = (n + GEMV_THREADS - 1) / GEMV_THREADS;
  const long long blocks = (t_hi - t_lo) * row_tiles;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const dim3 grid(static_cast<unsigned>(blocks));
  switch (nimg * 16 + nrhs) {
#define FPBEM_GEMV_CASE(R, NI)                                                                                   \
  case NI * 16 + R:                                                                                             \
    near_mode_gemv_kernel<R, NI><<<grid, GEMV_THREADS, 0, stream>>>(shat, items, n_items, perm, xh, yh, n, t_lo, \
                                                                    q_stride, row_tiles);                       \
    break;
    FPBEM_GEMV_CASE(1, 1)
    FPBEM_GEMV_CASE(2, 1)
    FPBEM_GEMV_CASE(3, 1)
    FPBEM_GEMV_CASE(4, 1)
    FPBEM_GEMV_CASE(5, 1)
    FPBEM_GEMV_CASE(6, 1)
    FPBEM_GEMV_CASE(7, 1)
    FPBEM_GEMV_CASE(8, 1)
    FPBEM_GEMV_CASE(1, 2)
    FPBEM_GEMV_CASE(2, 2)
    FPBEM_GEMV_CASE(3, 2)
    FPBEM_GEMV_CASE(4, 2)
    FPBEM_GEMV_CASE(1, 4)
    FPBEM_GEMV_CASE(2, 4)
    FPBEM_GEMV_CASE(1, 8)
#undef FPBEM_GEMV_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Shape of the tensor-core mode product for n rows and `ncols` columns per
// stored block: consumer warps, k columns per ring stage, ring depth and the
// dynamic shared memory; false when it does not apply (n % 8, > 8 columns,
// more than 8 row tiles per warp, or no 2-stage ring fits).
// X (image-column) buffers of the mode product: 2 lets the gather of the next block's
// columns run under the current block; 1 frees 41 KB (n = 320) for one more ring
// stage of the block stream (FPBEM_MMA_XBUF=1|2, A/B)
int mode_mma_xbufs() {
  static const int xb = [] {
    const char* v = std::getenv("FPBEM_MMA_XBUF");
    return (v && std::atoi(v) == 1) ? 1 : 2;
  }();
  return xb;
}

bool mode_mma_shape(int n, int ncols, int* nw, int* kc, int* ring, size_t* smem) {
  if (n <= 0 || n % 8 || ncols < 1 || ncols > 8) return false;
  // consumer warps of up to 8 row tiles each (n <= 512; larger blocks keep the
  // GEMV, which streams at the HBM roofline with few columns per block, cfg2):
  // 10 warps x 4 tiles where the rows split evenly that way (n = 320), else 8
  // (FPBEM_MMA_NW=8|10|20 forces one, A/B)
  static const int nw_env = [] {
    const char* v = std::getenv("FPBEM_MMA_NW");
    return v ? std::atoi(v) : 0;
  }();
  const int n_mt = n / 8;
  int NW = (n_mt % 10 == 0 && n_mt / 10 <= 8) ? 10 : 8;
  if (nw_env == 8 || nw_env == 10 || nw_env == 20) NW = nw_env;
  if ((n_mt + NW - 1) / NW > 8) NW = 8;
  if ((n_mt + NW - 1) / NW > 8) return false;
  static const int kc_env = [] {  // FPBEM_MMA_KC=4|8|16: columns per ring stage (A/B)
    const char* v = std::getenv("FPBEM_MMA_KC");
    const int k = v ? std::atoi(v) : 8;
    return (k == 4 || k == 8 || k == 16) ? k : 8;
  }();
  const int KC = kc_env;
  const int XB = mode_mma_xbufs();
  const size_t stage = sizeof(c64) * KC * static_cast<size_t>(n + 2);
  const size_t fixed = XB * sizeof(c64) * 8 * static_cast<size_t>(n + 4) + 4 * 8 * 16 + 128;
  const size_t budget = static_cast<size_t>(kMaxDynSmem) - 1024;  // the kernel's static shared memory
  if (fixed + 2 * stage > budget) return false;
  static const int ring_env = [] {  // FPBEM_MMA_RING: most ring stages (A/B: shared memory left to a co-resident kernel)
    const char* v = std::getenv("FPBEM_MMA_RING");
    return v ? std::atoi(v) : 0;
  }();
  int R = static_cast<int>(std::min<size_t>(16, (budget - fixed) / stage));
  if (ring_env >= 2 && R > ring_env) R = ring_env;
  *nw = NW;
  *kc = KC;
  *ring = R;
  *smem = sizeof(c64) * (static_cast<size_t>(R) * KC * (n + 2) + XB * 8 * static_cast<size_t>(n + 4)) +
          sizeof(unsigned long long) * (2 * R + 4);
  return true;
}

cudaError_t launch_mode_mma(const c64* shat, const int* items, long long n_items, const int* perm, const c64* xh,
                            c64* yh, int n, long long t_lo, long long t_hi, long long q_stride, int nrhs, int nimg,
                            cudaStream_t stream) {
  if (t_hi <= t_lo) return cudaSuccess;
  int NW, KC, R;
  size_t smem;
  const int ncols = nrhs * nimg;
  if (!mode_mma_shape(n, ncols, &NW, &KC, &R, &smem)) return cudaErrorInvalidValue;
  // FPBEM_MMA_RSPLIT=2|4 splits each block's row tiles over that many CTAs (A/B for
  // few blocks, e.g. a slab rank's share). Off by default: the per-block DMMA work
  // bounds an SM, so a split only pays when the units fill whole waves, and cfg3's
  // 8-rank share (99 blocks -> 198 units on 148 SMs) measured 46 -> 63 us
  static const int rsplit_env = [] {
    const char* v = std::getenv("FPBEM_MMA_RSPLIT");
    const int r = v ? std::atoi(v) : 1;
    return (r == 2 || r == 4) ? r : 1;
  }();
  const long long n_blk = t_hi - t_lo;
  const int sms = device_sms();
  const int rsplit = ((n / 8) / rsplit_env >= NW) ? rsplit_env : 1;
  const int MT = ((n / 8 + rsplit - 1) / rsplit + NW - 1) / NW;
  static std::atomic<unsigned long long> raised[18];
  using K = void (*)(const c64*, const int*, long long, const int*, const c64*, c64*, int, long long, long long,
                     long long, int, int, int, int, int, int);
  static const K fns[18] = {near_mode_mma_kernel<1, 8>,  near_mode_mma_kernel<2, 8>,  near_mode_mma_kernel<3, 8>,
                            near_mode_mma_kernel<4, 8>,  near_mode_mma_kernel<5, 8>,  near_mode_mma_kernel<6, 8>,
                            near_mode_mma_kernel<7, 8>,  near_mode_mma_kernel<8, 8>,  near_mode_mma_kernel<1, 10>,
                            near_mode_mma_kernel<2, 10>, near_mode_mma_kernel<3, 10>, near_mode_mma_kernel<4, 10>,
                            near_mode_mma_kernel<5, 10>, near_mode_mma_kernel<6, 10>, near_mode_mma_kernel<7, 10>,
                            near_mode_mma_kernel<8, 10>, near_mode_mma_kernel<1, 20>, near_mode_mma_kernel<2, 20>};
  if (NW == 20 && MT > 2) return cudaErrorInvalidValue;
  const int which = (NW == 8 ? 0 : NW == 10 ? 8 : 16) + MT - 1;
  cudaError_t e = ensure_max_smem(raised[which], reinterpret_cast<const void*>(fns[which]), kMaxDynSmem);
  if (e != cudaSuccess) return e;
  const long long units = n_blk * rsplit;
  const int grid = static_cast<int>(std::min<long long>(units, sms));
  return launch_ex(fns[which], dim3(grid), dim3(32 * (NW + 2)), smem, stream, pdl_enabled(stream, true), shat, items, n_items,
                   perm, xh, yh, n, t_lo, t_hi, q_stride, nrhs, ncols, KC, R, rsplit, mode_mma_xbufs());
}

// max |S_s'[P i + n P j] - S_s[i + n j]| over blocks s with image slot s' (the
// block of A_g o) and max |S|, as double bits (non-negative doubles order like
// their bit patterns): the device check of one cell symmetry g (mirror = slot of A_g o, perm = P_g)
__global__ void near_symmetry_kernel(const c64* __restrict__ S, int n, int n_blk, const int* __restrict__ mirror,
                                     const int* __restrict__ perm, unsigned long long* out2) {
  const long long nn = static_cast<long long>(n) * n, total = nn * n_blk;
  double dev = 0.0, amax = 0.0;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(g / nn);
    const long long e = g % nn;
    const int i = static_cast<int>(e % n), j = static_cast<int>(e / n);
    const c64 v = S[g];
    const c64 w = S[mirror[s] * nn + __ldg(perm + i) + static_cast<long long>(n) * __ldg(perm + j)];
    dev = fmax(dev, fmax(fabs(v.x - w.x), fabs(v.y - w.y)));
    amax = fmax(amax, fmax(fabs(v.x), fabs(v.y)));
  }
  for (int o = 16; o > 0; o >>= 1) {
    dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out2, static_cast<unsigned long long>(__double_as_longlong(dev)));
    atomicMax(out2 + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
  }
}

cudaError_t launch_near_symmetry(const c64* S, int n, int n_blk, const int* mirror, const int* perm,
                                 unsigned long long* out2, cudaStream_t stream) {
  const long long total = static_cast<long long>(n) * n * n_blk;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > 16LL * kNumSMs) blocks = 16LL * kNumSMs;
  near_symmetry_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(S, n, n_blk, mirror, perm, out2);
  return cudaGetLastError();
}

// y[r, t, i] += sum_m U0[i, m] L[t, r, m] (src/fmm.cpp:265-267) for the lattice
// near field, whose product already sits in y. CTA = (128 rows, kL2pCols (cell,
// rhs) columns): each U0 element is loaded once per CTA and used for all its
// columns (independent accumulators), the locals come from shared memory as
// broadcasts; every output sums m in ascending order from zero and is then
// added to y, the same arithmetic as the reduction kernel with no pairs.
constexpr int kL2pCols = 8;

__global__ void __launch_bounds__(128)
l2p_add_kernel(const c64* __restrict__ u0, const c64* __restrict__ local, c64* __restrict__ y, int n, int n_coef,
               long long n_cols, long long N, int nrhs, int row_tiles) {
  extern __shared__ __align__(16) unsigned char l2p_smem[];
  c64* ls = reinterpret_cast<c64*>(l2p_smem);  // [kL2pCols][n_coef]
  const long long c0 = static_cast<long long>(blockIdx.x / row_tiles) * kL2pCols;
  const int i = (blockIdx.x % row_tiles) * 128 + threadIdx.x;
  const int nc = static_cast<int>(min(static_cast<long long>(kL2pCols), n_cols - c0));
  for (int e = threadIdx.x; e < kL2pCols * n_coef; e += 128)
    ls[e] = e < nc * n_coef ? local[c0 * n_coef + e] : cmk(0.0, 0.0);
  __syncthreads();
  if (i >= n) return;
  c64 yv[kL2pCols];  // the current y, loaded up front (independent of the sums)
  long long off[kL2pCols];
#pragma unroll
  for (int c = 0; c < kL2pCols; ++c) {
    const int tr = static_cast<int>(c0) + c;  // t * nrhs + r (< 2^31: checked at launch)
    off[c] = (tr % nrhs) * N + static_cast<long long>(tr / nrhs) * n + i;
    yv[c] = c < nc ? y[off[c]] : cmk(0.0, 0.0);
  }
  c64 acc[kL2pCols];
#pragma unroll
  for (int c = 0; c < kL2pCols; ++c) acc[c] = cmk(0.0, 0.0);
  int m = 0;
  for (; m + 4 <= n_coef; m += 4) {
    c64 u[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) u[v] = __ldg(u0 + static_cast<size_t>(m + v) * n + i);
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int c = 0; c < kL2pCols; ++c) acc[c] = cfma(u[v], ls[c * n_coef + m + v], acc[c]);
  }
  for (; m < n_coef; ++m) {
    const c64 u = __ldg(u0 + static_cast<size_t>(m) * n + i);
#pragma unroll
    for (int c = 0; c < kL2pCols; ++c) acc[c] = cfma(u, ls[c * n_coef + m], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < kL2pCols; ++c) {
    if (c >= nc) break;
    y[off[c]] = cadd(yv[c], cadd(cmk(0.0, 0.0), acc[c]));
  }
}

cudaError_t launch_l2p_add(const c64* u0, const c64* local, c64* y, int n, int n_coef, int n_cells, long long N,
                           int nrhs, cudaStream_t stream) {
  if (n_coef > MAX_COEF) return cudaErrorInvalidValue;
  const int row_tiles = (n + 127) / 128;
  const long long cols = static_cast<long long>(n_cells) * nrhs;
  const long long blocks = (cols + kL2pCols - 1) / kL2pCols * row_tiles;
  if (blocks > 0x7fffffffLL || cols + kL2pCols > 0x7fffffffLL) return cudaErrorInvalidValue;
  const size_t smem = sizeof(c64) * kL2pCols * n_coef;
  if (smem > 48 * 1024) {
    static std::atomic<unsigned long long> raised{0};
    cudaError_t e = ensure_max_smem(raised, reinterpret_cast<const void*>(&l2p_add_kernel), 64 * 1024);
    if (e != cudaSuccess) return e;
  }
  l2p_add_kernel<<<static_cast<unsigned>(blocks), 128, smem, stream>>>(u0, local, y, n, n_coef, cols, N, nrhs,
                                                                      row_tiles);
  return cudaGetLastError();
}

cudaError_t launch_near_reduce_l2p(const c64* W, const int* tgt_ptr, const int* tgt_pairs, const c64* u0,
                                   const c64* local, c64* y, int n, int n_coef, int n_cells, long long N,
                                   int nrhs, bool accumulate, cudaStream_t stream) {
  if (n_coef > MAX_COEF) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(static_cast<long long>((n + RED_THREADS - 1) / RED_THREADS) * n_cells * nrhs));
  near_reduce_l2p_kernel<<<grid, RED_THREADS, 0, stream>>>(W, tgt_ptr, tgt_pairs, u0, local, y, n, n_coef, N,
                                                           nrhs, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
