// P2M of the single-level FMM as one per-cell GEMM on the FP64 tensor cores
// (DMMA): M_c = V0 p_c (src/fmm.cpp:256-259; V0: b x n), i.e. out[col] (+)=
// A in[col] for every (cell, rhs) column with one shared matrix A. The FMA
// kernel streamed V0 from L2 per cell and took 66 us on cfg3 for 21 MB of
// input (now 29 us). (The L2P is fused into the last inverse near-field DFT
// pass, csrc/m2l.cu.) Here:
//   * persistent CTAs hold A in shared memory ([m][k], pitch = 4 mod 8
//     complex: conflict-free m8n8k4 fragments), loaded once per CTA;
//   * the columns come in chunks of 8 (one DMMA n-tile), double-buffered with
//     16-byte cp.async, so the next chunk's HBM reads overlap this chunk's math;
//   * warps own A's 8-row tiles; the k range is split over warp groups (b = 25
//     -> 4 row tiles, 16 warps: 4 groups) with two accumulator sets each, and
//     the partial tiles are added in a fixed order through shared memory
//     (deterministic);
//   * Gauss 3-multiplication complex product (3 DMMAs per complex 8x8x4 tile).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {

constexpr int kCwWarps = 16;

__host__ __device__ constexpr int cw_pitch(int k) { return ((k + 3) / 4 * 4 + 4 - 1) / 8 * 8 + 4; }  // >= k, = 4 mod 8

template <int MTW>  // row tiles per warp (max)
__global__ void __launch_bounds__(kCwWarps * 32, 1)
cellwise_gemm_kernel(const c64* __restrict__ a, long long a_ms, long long a_ks, int M, int K,
                     const c64* __restrict__ in, long long in_rs, long long in_cs, c64* __restrict__ out,
                     long long out_rs, long long out_cs, int nrhs, long long ncols, int accumulate) {
  extern __shared__ __align__(16) unsigned char cw_raw[];
  const int KP = cw_pitch(K), MT = (M + 7) / 8, KS = (K + 3) / 4;  // k steps
  c64* As = reinterpret_cast<c64*>(cw_raw);  // [M][KP]
  c64* Bs = As + static_cast<size_t>(M) * KP;  // 2 x [8][KP]
  c64* Red = Bs + 2 * 8 * KP;                  // k-split partial tiles [warp][32 lanes][2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
  // A into shared memory with 16-byte cp.async (no register round trip per element)
  if (a_ks == 1) {  // A rows contiguous in global memory (V0^T): k fastest
    for (int e = tid; e < M * KP; e += blockDim.x) {
      const int m = e / KP, k = e - m * KP;
      cp_async16(As + e, a + (k < K ? m * a_ms + k : 0), k < K);
    }
  } else {  // A columns contiguous (U0, column-major): m fastest for coalesced reads
    for (int e = tid; e < M * KP; e += blockDim.x) {
      const int k = e / M, m = e - k * M;
      cp_async16(As + m * KP + k, a + (k < K ? m * a_ms + k * a_ks : 0), k < K);
    }
  }
  cp_async_commit();
  // k split: G groups of warps share the row tiles (G = 8 / MT when MT < 8)
  const int G = MT >= kCwWarps ? 1 : kCwWarps / MT;
  const int grp = MT >= kCwWarps ? 0 : warp / MT, wt = MT >= kCwWarps ? warp : warp % MT;
  const int ks0 = KS * grp / G, ks1 = KS * (grp + 1) / G;
  const bool active = MT >= kCwWarps || warp < MT * G;
  const long long chunks = (ncols + 7) / 8;

  auto load = [&](int buf, long long ch) {  // columns 8 ch .. 8 ch + 7 into Bs[buf]
    c64* dst = Bs + buf * 8 * KP;
    for (int e = tid; e < 8 * KP; e += blockDim.x) {
      const int c = e / KP, k = e - c * KP;
      const long long col = ch * 8 + c;
      const bool ok = col < ncols && k < K;
      const long long cell = ok ? col / nrhs : 0, r = ok ? col - cell * nrhs : 0;
      cp_async16(dst + e, ok ? in + r * in_rs + cell * in_cs + k : in, ok);
    }
    cp_async_commit();
  };
  long long ch = blockIdx.x;
  if (ch < chunks) load(0, ch);
  int buf = 0;
  for (; ch < chunks; ch += gridDim.x, buf ^= 1) {
    const long long nxt = ch + gridDim.x;
    if (nxt < chunks) {
      load(buf ^ 1, nxt);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk ch (and A) visible to every warp
    const c64* bs = Bs + buf * 8 * KP + fr * KP + fk;
    // the outputs this thread accumulates into, requested before the k loop
    c64 prev[MTW][2];
#pragma unroll
    for (int u = 0; u < MTW; ++u)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        prev[u][j] = cmk(0.0, 0.0);
        const int m = (wt + u * kCwWarps) * 8 + fr;
        const long long col = ch * 8 + 2 * fk + j;
        if (accumulate && active && grp == 0 && wt + u * kCwWarps < MT && m < M && col < ncols) {
          const long long cell = col / nrhs, r = col - cell * nrhs;
          prev[u][j] = out[r * out_rs + cell * out_cs + m];
        }
      }
    // two accumulator sets over alternating k steps: twice the independent DMMA
    // chains per warp (the single-set version waited on DMMA latency, ncu)
    double t1[2][MTW][2], t2[2][MTW][2], t3[2][MTW][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < MTW; ++u)
        t1[h][u][0] = t1[h][u][1] = t2[h][u][0] = t2[h][u][1] = t3[h][u][0] = t3[h][u][1] = 0.0;
    if (active) {
      int s = ks0;
      for (; s + 1 < ks1; s += 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const c64 b = bs[4 * (s + h)];
          const double bsum = b.x + b.y;
#pragma unroll
          for (int u = 0; u < MTW; ++u) {
            const int mt = wt + u * kCwWarps;
            if (mt < MT) {
              const int m = mt * 8 + fr;
              const c64 av = m < M ? As[m * KP + 4 * (s + h) + fk] : cmk(0.0, 0.0);
              dmma884(t1[h][u][0], t1[h][u][1], av.x, b.x);
              dmma884(t2[h][u][0], t2[h][u][1], av.y, b.y);
              dmma884(t3[h][u][0], t3[h][u][1], av.x + av.y, bsum);
            }
          }
        }
      }
      if (s < ks1) {
        const c64 b = bs[4 * s];
        const double bsum = b.x + b.y;
#pragma unroll
        for (int u = 0; u < MTW; ++u) {
          const int mt = wt + u * kCwWarps;
          if (mt < MT) {
            const int m = mt * 8 + fr;
            const c64 av = m < M ? As[m * KP + 4 * s + fk] : cmk(0.0, 0.0);
            dmma884(t1[0][u][0], t1[0][u][1], av.x, b.x);
            dmma884(t2[0][u][0], t2[0][u][1], av.y, b.y);
            dmma884(t3[0][u][0], t3[0][u][1], av.x + av.y, bsum);
          }
        }
      }
    }
    auto tile = [&](int u, int j) {  // this warp's partial C entry (set 0 + set 1)
      const double a1 = t1[0][u][j] + t1[1][u][j], a2 = t2[0][u][j] + t2[1][u][j], a3 = t3[0][u][j] + t3[1][u][j];
      return cmk(a1 - a2, a3 - a1 - a2);
    };
    // k-split: groups 1.. hand their tiles to group 0, which adds them in group order
    if (G > 1) {
      if (active && grp > 0) {
        c64* r = Red + (static_cast<size_t>(warp) * 32 + lane) * 2;
        for (int j = 0; j < 2; ++j) r[j] = tile(0, j);
      }
      __syncthreads();
    }
    if (active && grp == 0) {
#pragma unroll
      for (int u = 0; u < MTW; ++u) {
        const int mt = wt + u * kCwWarps;
        if (mt >= MT) continue;
        const int m = mt * 8 + fr;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          c64 v = tile(u, j);
          for (int g = 1; g < G; ++g) v = cadd(v, Red[(static_cast<size_t>(g * MT + wt) * 32 + lane) * 2 + j]);
          const long long col = ch * 8 + 2 * fk + j;
          if (m < M && col < ncols) {
            const long long cell = col / nrhs, r = col - cell * nrhs;
            out[r * out_rs + cell * out_cs + m] = accumulate ? cadd(prev[u][j], v) : v;
          }
        }
      }
    }
    __syncthreads();  // Bs[buf] and Red are rewritten next
  }
}

// The same product with no shared-memory staging of the columns and no block-wide
// barrier in the loop: the CTA's warps form G = 16 / MT groups of MT warps (one
// 8-row tile of A each); every group walks its own chunks of 8 columns over the
// whole k range, loading its B fragments straight from global memory 8 k steps
// ahead (the group's warps read the same fragments: L1 hits after the first).
// The barrier-per-chunk form above ran only ~3.5 chunks per CTA on cfg3 and was
// bound by the chunk latency (29 us for 21 MB of input).
__global__ void __launch_bounds__(kCwWarps * 32, 1)
cellwise_stream_kernel(const c64* __restrict__ a, long long a_ms, int M, int K, const c64* __restrict__ in,
                       long long in_rs, long long in_cs, c64* __restrict__ out, long long out_rs, long long out_cs,
                       int nrhs, long long ncols) {
  extern __shared__ __align__(16) unsigned char cw_raw[];
  const int KP = cw_pitch(K), MT = (M + 7) / 8, KS = (K + 3) / 4;
  c64* As = reinterpret_cast<c64*>(cw_raw);  // [M][KP], rows contiguous in global (a_ks = 1)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
  for (int e = tid; e < M * KP; e += blockDim.x) {
    const int m = e / KP, k = e - m * KP;
    cp_async16(As + e, a + (k < K ? m * a_ms + k : 0), k < K);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int G = kCwWarps / MT, grp = warp / MT, mt = warp % MT;
  if (grp >= G) return;
  const int m = mt * 8 + fr;
  const c64* arow = As + (m < M ? m : 0) * KP + fk;
  const long long chunks = (ncols + 7) / 8;
  constexpr int U = 16;  // k steps of B fragments in flight
  for (long long ch = static_cast<long long>(blockIdx.x) * G + grp; ch < chunks;
       ch += static_cast<long long>(gridDim.x) * G) {
    const long long col = ch * 8 + fr;  // this lane's B column
    const bool cok = col < ncols;
    const long long cell = cok ? col / nrhs : 0, r = cok ? col - cell * nrhs : 0;
    const c64* bcol = in + r * in_rs + cell * in_cs + fk;
    double t1[2][2] = {}, t2[2][2] = {}, t3[2][2] = {};
    for (int s0 = 0; s0 < KS; s0 += U) {
      c64 bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = 4 * (s0 + u) + fk;
        bv[u] = (cok && s0 + u < KS && k < K) ? __ldg(bcol + 4 * (s0 + u)) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (s0 + u >= KS) break;
        const int h = u & 1;
        const c64 av = m < M ? arow[4 * (s0 + u)] : cmk(0.0, 0.0);
        dmma884(t1[h][0], t1[h][1], av.x, bv[u].x);
        dmma884(t2[h][0], t2[h][1], av.y, bv[u].y);
        dmma884(t3[h][0], t3[h][1], av.x + av.y, bv[u].x + bv[u].y);
      }
    }
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long oc = ch * 8 + 2 * fk + j;
      if (oc >= ncols) continue;
      const double a1 = t1[0][j] + t1[1][j], a2 = t2[0][j] + t2[1][j], a3 = t3[0][j] + t3[1][j];
      const long long ocell = oc / nrhs, orr = oc - ocell * nrhs;
      out[orr * out_rs + ocell * out_cs + m] = cmk(a1 - a2, a3 - a1 - a2);
    }
  }
}

size_t cw_smem(int M, int K) {
  const size_t KP = cw_pitch(K);
  return sizeof(c64) * (static_cast<size_t>(M) * KP + 2 * 8 * KP + static_cast<size_t>(kCwWarps) * 32 * 2);
}

}  // namespace

bool cellwise_supported(int M, int K) {
  return M >= 1 && K >= 1 && (M + 7) / 8 <= kCwWarps && cw_smem(M, K) <= static_cast<size_t>(kMaxDynSmem) - 1024;
}

cudaError_t launch_cellwise(const c64* a, long long a_ms, long long a_ks, int M, int K, const c64* in, long long in_rs,
                            long long in_cs, c64* out, long long out_rs, long long out_cs, int nrhs, long long ncols,
                            bool accumulate, cudaStream_t stream) {
  if (ncols <= 0) return cudaSuccess;
  if (!cellwise_supported(M, K)) return cudaErrorInvalidValue;
  const size_t smem = cw_smem(M, K);
  static std::atomic<unsigned long long> raised{0};
  cudaError_t e = ensure_max_smem(raised, reinterpret_cast<const void*>(&cellwise_gemm_kernel<1>), kMaxDynSmem);
  if (e != cudaSuccess) return e;
  const long long chunks = (ncols + 7) / 8;
  // FPBEM_CELLWISE_V1=1: the staged, barrier-per-chunk form (A/B)
  static const bool v1 = [] {
    const char* v = std::getenv("FPBEM_CELLWISE_V1");
    return v && std::strcmp(v, "1") == 0;
  }();
  if (!v1 && a_ks == 1 && !accumulate) {
    static std::atomic<unsigned long long> raised2{0};
    e = ensure_max_smem(raised2, reinterpret_cast<const void*>(&cellwise_stream_kernel), kMaxDynSmem);
    if (e != cudaSuccess) return e;
    const int G = kCwWarps / ((M + 7) / 8);
    const int grid = static_cast<int>(std::min<long long>((chunks + G - 1) / G, device_sms()));
    const size_t smem_s = sizeof(c64) * static_cast<size_t>(M) * cw_pitch(K);
    cellwise_stream_kernel<<<grid, kCwWarps * 32, smem_s, stream>>>(a, a_ms, M, K, in, in_rs, in_cs, out, out_rs,
                                                                     out_cs, nrhs, ncols);
    return cudaGetLastError();
  }
  // persistent: one CTA per SM (A fills most of the shared memory)
  const int grid = static_cast<int>(std::min<long long>(chunks, device_sms()));
  cellwise_gemm_kernel<1><<<grid, kCwWarps * 32, smem, stream>>>(a, a_ms, a_ks, M, K, in, in_rs, in_cs, out, out_rs,
                                                                   out_cs, nrhs, ncols, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
