// C-ABI implementation (include/fpbem_cuda.h), part 1: the operator handle —
// create / destroy, the FMM apply (near field + P2M + lattice-DFT M2L + L2P),
// the spectrum, streams and stage timing. The device GMRES is gmres.cu, the
// device assembly / M2L bank / field evaluation device_assembly.cu, NCCL and the
// multi-GPU partition comm.cu; the shared handle is handle.cuh.
//
//   FmmOperators::matvec  src/fmm.cpp:246-271  -> apply_chunk()
//   CirculantSpectrum ctor src/structured.cpp:63-108 -> build_spectrum()
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "handle.cuh"

using namespace fpbem_cu;

namespace {
int fft_friendly(int n) {  // smallest 7-smooth length >= n (src/structured.cpp:26-33)
  for (int m = n;; ++m) {
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}
}  // namespace

namespace fpbem_cu {

// Multi-GPU work split: every near-field pair (offset, target)
// costs the same n_dof^2 MACs, so ranks take equal contiguous ranges of the
// global pair order (offset-major) — balanced whatever the offset count.
// Contiguous ranges of the (offset, target) pairs: equal shares, except that
// rank 0 (which also runs the far field) takes `far_pairs` fewer, the other
// ranks sharing the rest equally; every pair is owned exactly once.
void pair_range(long long n_pairs, int nranks, int rank, double far_pairs, long long& lo, long long& hi) {
  long long d = far_pairs > 0.0 && nranks > 1 ? std::llround(far_pairs) : 0;
  if (d == 0) {
    lo = n_pairs * rank / nranks;
    hi = n_pairs * (rank + 1) / nranks;
    return;
  }
  const long long h0 = std::max(0LL, (n_pairs + d) / nranks - d);  // rank 0's share
  if (rank == 0) {
    lo = 0;
    hi = h0;
    return;
  }
  const long long rest = n_pairs - h0;
  lo = h0 + rest * (rank - 1) / (nranks - 1);
  hi = h0 + rest * rank / (nranks - 1);
}

// per-target CSR of the pairs this rank owns, in offset order (the reduction order)
void build_target_csr(fpbem_cu_op* op) {
  std::vector<std::vector<int>> per_t(op->n_cells);
  for (long long p = op->pair_lo; p < op->pair_hi; ++p) per_t[op->pair_tgt[p]].push_back(static_cast<int>(p));
  std::vector<int> tptr(op->n_cells + 1, 0), tpairs;
  for (int t = 0; t < op->n_cells; ++t) {
    tpairs.insert(tpairs.end(), per_t[t].begin(), per_t[t].end());
    tptr[t + 1] = static_cast<int>(tpairs.size());
  }
  if (!op->tgt_ptr) op->tgt_ptr = dalloc<int>(op->n_cells + 1, "target ptr");
  if (!op->tgt_pairs) op->tgt_pairs = dalloc<int>(std::max(op->n_pairs, 1), "target pairs");
  h2d(op->tgt_ptr, tptr.data(), tptr.size() * sizeof(int), op->stream, "target ptr");
  if (!tpairs.empty()) h2d(op->tgt_pairs, tpairs.data(), tpairs.size() * sizeof(int), op->stream, "target pairs");
}

void set_partition(fpbem_cu_op* op, int rank, int nranks, double far_pairs) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(FPBEM_CU_EINVAL, "partition: bad rank / nranks");
  if (!(far_pairs >= 0.0)) fail(FPBEM_CU_EINVAL, "partition: far_pairs must be >= 0");
  op->far_pairs = far_pairs;
  op->rank = rank;
  op->nranks = nranks;
  if (op->near_fft) {  // units are the stored blocks of the near-field lattice (one n x n block stream each)
    pair_range(op->n_items, nranks, rank, far_pairs, op->mode_lo, op->mode_hi);
    op->mjobs_nrhs = -1;
    return;
  }
  pair_range(op->n_pairs, nranks, rank, far_pairs, op->pair_lo, op->pair_hi);
  op->jobs_nrhs = -1;  // rebuild the GEMM job list
  build_target_csr(op);
}

// Column tiles of one offset (or of the P2M columns): as many 64-wide tiles as
// fit, then the remainder as one 64- (49..63), 32+16- (33..48), 32- (17..32)
// or 16-wide (1..16) tile. job.z = column count | width class << 8.
void tile_columns(std::vector<int4>& jobs, int s, int cols, int pair_base, bool narrow, int flags = 0) {
  int c0 = 0;
  auto push = [&](int w, int cls) {
    jobs.push_back(make_int4(s, c0, w | (cls << 8) | flags, pair_base));
    c0 += w;
  };
  while (cols - c0 >= 64) push(64, 0);
  const int r = cols - c0;
  if (r == 0) return;
  if (!narrow || r > 48) {
    push(r, 0);
  } else if (r > 32) {
    push(32, 1);
    push(r - 32, 2);
  } else if (r > 16) {
    push(r, 1);
  } else {
    push(r, 2);
  }
}

void build_jobs(fpbem_cu_op* op, int nrhs) {
  if (op->jobs_nrhs == nrhs) return;
  const char* nv = std::getenv("FPBEM_NARROW_TILES");
  const bool narrow = !(nv && std::strcmp(nv, "0") == 0);
  std::vector<int4> jobs;
  for (int s = 0; s < op->n_near; ++s) {  // this rank's share of every offset's pairs
    const long long a = std::max<long long>(op->pair_start[s], op->pair_lo);
    const long long b = std::min<long long>(op->pair_start[s + 1], op->pair_hi);
    if (a < b) tile_columns(jobs, s, static_cast<int>(b - a) * nrhs, static_cast<int>(a), narrow);
  }
  // offset order: consecutive tiles share S_o in L2 (longest-first ordering measured neutral)
  if (static_cast<int>(jobs.size()) > op->jobs_cap) {
    if (op->jobs) cudaFree(op->jobs);
    op->jobs = dalloc<int4>(jobs.size(), "jobs");
    op->jobs_cap = static_cast<int>(jobs.size());
  }
  if (!jobs.empty()) h2d(op->jobs, jobs.data(), jobs.size() * sizeof(int4), op->stream, "jobs upload");
  op->n_jobs = static_cast<int>(jobs.size());
  op->jobs_nrhs = nrhs;
}

// DMMA jobs of the lattice path: one column tile set (the nrhs right-hand sides)
// per mode of this rank's range; block slot = mode, unit = mode
void build_mode_jobs(fpbem_cu_op* op, int nrhs) {
  if (op->mjobs_nrhs == nrhs) return;
  std::vector<int4> jobs;
  // FPBEM_ORBIT_JOBS=0: one job per image mode even when the orbit fits one column tile (A/B)
  static const bool orbit_env = [] {
    const char* v = std::getenv("FPBEM_ORBIT_JOBS");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  for (long long t = op->mode_lo; t < op->mode_hi; ++t) {
    int nimg = 0;
    for (int i = 0; i < 8; ++i) nimg += op->items_q[t * 8 + i] >= 0;
    if (orbit_env) {
      // the orbit's (image, rhs) columns in tiles of 64 (job bit 15): the block is
      // streamed once per tile instead of once per image (8 images x 8 rhs: once)
      tile_columns(jobs, static_cast<int>(t), nimg * nrhs, 0, true, 1 << 15);
      continue;
    }
    for (int i = 0; i < 8; ++i) {  // one column set per image mode; g != 0: through P_g (job bits 12-14)
      const int q = op->items_q[t * 8 + i];
      if (q >= 0) tile_columns(jobs, static_cast<int>(t), nrhs, q, true, op->items_g[t * 8 + i] << 12);
    }
  }
  if (static_cast<int>(jobs.size()) > op->mjobs_cap) {
    if (op->mjobs) cudaFree(op->mjobs);
    op->mjobs = dalloc<int4>(jobs.size(), "mode jobs");
    op->mjobs_cap = static_cast<int>(jobs.size());
  }
  if (!jobs.empty()) h2d(op->mjobs, jobs.data(), jobs.size() * sizeof(int4), op->stream, "mode jobs upload");
  op->n_mjobs = static_cast<int>(jobs.size());
  op->mjobs_nrhs = nrhs;
}

void twiddles(fpbem_cu_op* op, int L, c64** out);
void ev_record(fpbem_cu_op* op, int i, cudaStream_t st);

// Block spectrum of the near field (the CirculantSpectrum construction,
// src/structured.cpp:63-108, applied to the Toeplitz blocks): S_o at slot
// (o mod Ln), forward DFT over every axis. Ln_d = M_d + max|o_d| is the
// smallest length whose circular convolution reproduces the truncated
// Toeplitz product (sources t - o in [-R, M-1+R] never alias into [0, M)).
void build_near_spectrum(fpbem_cu_op* op, int n_toeplitz) {
  const size_t nn = static_cast<size_t>(op->n) * op->n;
  const size_t total = static_cast<size_t>(op->qn) * nn;
  const long long Lx = op->Ln[0], Ly = op->Ln[1], Lz = op->Ln[2];
  using DevPtr = std::unique_ptr<void, decltype(&cudaFree)>;
  c64* a = dalloc<c64>(total, "near spectrum");
  DevPtr keep_a(a, &cudaFree);
  c64* b = dalloc<c64>(total, "near spectrum scratch");
  DevPtr keep_b(b, &cudaFree);
  int* offs = dalloc<int>(static_cast<size_t>(n_toeplitz) * 3, "near offsets");
  DevPtr keep_offs(offs, &cudaFree);
  h2d(offs, op->near_offsets.data(), static_cast<size_t>(n_toeplitz) * 3 * sizeof(int), op->stream, "near offsets");
  for (int k = 0; k < 3; ++k) twiddles(op, op->Ln[k], &op->twn[k]);
  check(cudaMemsetAsync(a, 0, total * sizeof(c64), op->stream), "near spectrum clear");
  check(launch_scatter_bank(op->S, offs, n_toeplitz, static_cast<int>(nn), op->Ln[0], op->Ln[1], op->Ln[2], a,
                            op->stream),
        "near scatter");
  c64* cur = a;
  c64* nxt = b;
  if (Lx > 1) {
    check(launch_dft_axis(cur, nxt, op->twn[0], Ly * Lz, op->Ln[0], op->Ln[0], nn, op->Ln[0], false, 1.0, op->stream),
          "near spectrum dft x");
    std::swap(cur, nxt);
  }
  if (Ly > 1) {
    check(launch_dft_axis(cur, nxt, op->twn[1], Lz, op->Ln[1], op->Ln[1], Lx * nn, op->Ln[1], false, 1.0, op->stream),
          "near spectrum dft y");
    std::swap(cur, nxt);
  }
  if (Lz > 1) {
    check(launch_dft_axis(cur, nxt, op->twn[2], 1, op->Ln[2], op->Ln[2], Lx * Ly * nn, op->Ln[2], false, 1.0,
                          op->stream),
          "near spectrum dft z");
    std::swap(cur, nxt);
  }
  // work items: one per orbit of modes under the verified symmetries (one per mode without)
  const size_t n_items = static_cast<size_t>(op->n_items);
  op->items = dalloc<int>(n_items * 16, "near items");
  h2d(op->items, op->items_q.data(), n_items * 8 * sizeof(int), op->stream, "near items");
  h2d(op->items + n_items * 8, op->items_g.data(), n_items * 8 * sizeof(int), op->stream, "near items");
  if (op->near_nimg > 1) {  // keep only the blocks of the orbits' representatives
    c64* compact = dalloc<c64>(n_items * nn, "near spectrum (orbits)");
    DevPtr keep_c(compact, &cudaFree);
    for (size_t t = 0; t < n_items; ++t)
      check(cudaMemcpyAsync(compact + t * nn, cur + static_cast<size_t>(op->items_q[t * 8]) * nn, nn * sizeof(c64),
                            cudaMemcpyDeviceToDevice, op->stream),
            "near spectrum compaction");
    check(cudaStreamSynchronize(op->stream), "near spectrum compaction");
    op->shat = static_cast<c64*>(keep_c.release());
    return;  // a and b freed here
  }
  check(cudaStreamSynchronize(op->stream), "near spectrum build");
  if (cur == a)
    keep_a.release();
  else
    keep_b.release();
  op->shat = cur;
}

// Cell symmetries: every axis-sign map g the caller gives
// with its element permutation P_g is kept when the offset set is closed under
// A_g and S_{A_g o}[P_g i, P_g j] == S_o[i, j] on the device to 1e-12 of
// max |S|; the kept set is reduced to a group. Sets near_sym_mask / _dev.
void check_symmetries(fpbem_cu_op* op, const fpbem_cu_fmm_desc* d) {
  op->near_sym_mask = 1;
  op->near_sym_dev = -1.0;
  if (d->n_sym <= 0 || !d->sym_axes || !d->sym_perms || d->n_near == 0) return;
  using DevPtr = std::unique_ptr<void, decltype(&cudaFree)>;
  if (!op->perm) op->perm = dalloc<int>(static_cast<size_t>(7) * op->n, "cell symmetries");
  int* dm = dalloc<int>(d->n_near, "symmetry slots");
  DevPtr keep_m(dm, &cudaFree);
  unsigned long long* dv = dalloc<unsigned long long>(2, "symmetry check");
  DevPtr keep_dv(dv, &cudaFree);
  double worst = 0.0;
  int mask = 1;
  for (int u = 0; u < d->n_sym; ++u) {
    const int g = d->sym_axes[u];
    if (g < 1 || g > 7) fail(FPBEM_CU_EINVAL, "create: sym_axes entries must be in 1..7");
    const int* pg = d->sym_perms + static_cast<size_t>(u) * op->n;
    std::vector<char> seen(op->n, 0);
    for (int i = 0; i < op->n; ++i) {
      if (pg[i] < 0 || pg[i] >= op->n || seen[pg[i]]) fail(FPBEM_CU_EINVAL, "create: sym_perms row is not a permutation");
      seen[pg[i]] = 1;
    }
    std::vector<int> mirror(d->n_near, -1);  // slot of A_g o
    bool closed = true;
    for (int s = 0; s < d->n_near && closed; ++s) {
      int o[3];
      for (int k = 0; k < 3; ++k) o[k] = (g >> k & 1) ? -op->near_offsets[3 * s + k] : op->near_offsets[3 * s + k];
      for (int t = 0; t < d->n_near && mirror[s] < 0; ++t)
        if (op->near_offsets[3 * t] == o[0] && op->near_offsets[3 * t + 1] == o[1] && op->near_offsets[3 * t + 2] == o[2])
          mirror[s] = t;
      closed = mirror[s] >= 0;
    }
    if (!closed) continue;
    int* prow = op->perm + static_cast<size_t>(g - 1) * op->n;
    h2d(prow, pg, op->n * sizeof(int), op->stream, "cell symmetry");
    h2d(dm, mirror.data(), mirror.size() * sizeof(int), op->stream, "symmetry slots");
    check(cudaMemsetAsync(dv, 0, 2 * sizeof(unsigned long long), op->stream), "symmetry check");
    check(launch_near_symmetry(op->S, op->n, d->n_near, dm, prow, dv, op->stream), "symmetry check");
    unsigned long long hv[2];
    check(cudaMemcpyAsync(hv, dv, sizeof(hv), cudaMemcpyDeviceToHost, op->stream), "symmetry check");
    check(cudaStreamSynchronize(op->stream), "symmetry check");
    double dev, amax;
    std::memcpy(&dev, &hv[0], sizeof(double));
    std::memcpy(&amax, &hv[1], sizeof(double));
    const double rel = amax > 0.0 ? dev / amax : (dev > 0.0 ? 1.0 : 0.0);
    worst = std::max(worst, rel);
    if (amax > 0.0 && dev <= 1e-12 * amax) mask |= 1 << g;
  }
  for (bool changed = true; changed;) {  // a group: drop g whose products leave the set
    changed = false;
    for (int g1 = 1; g1 < 8; ++g1)
      for (int g2 = 1; g2 < 8; ++g2)
        if ((mask >> g1 & 1) && (mask >> g2 & 1) && !(mask >> (g1 ^ g2) & 1)) {
          mask &= ~(1 << std::max(g1, g2));
          changed = true;
        }
  }
  op->near_sym_mask = mask;
  op->near_sym_dev = worst;
}

// Orbits of the Ln modes under the verified symmetries: items_q / items_g
// (8 slots per item, representative = smallest mode first), n_items, near_nimg.
void build_items(fpbem_cu_op* op, const int Ln[3]) {
  const long long qn = static_cast<long long>(Ln[0]) * Ln[1] * Ln[2];
  op->items_q.clear();
  op->items_g.clear();
  op->near_nimg = 1;
  std::vector<char> seen(qn, 0);
  for (long long q = 0; q < qn; ++q) {
    if (seen[q]) continue;
    const long long c[3] = {q % Ln[0], (q / Ln[0]) % Ln[1], q / (static_cast<long long>(Ln[0]) * Ln[1])};
    int slot = 0;
    int qs[8], gs[8];
    for (int g = 0; g < 8; ++g) {
      if (!(op->near_sym_mask >> g & 1)) continue;
      long long m[3];
      for (int k = 0; k < 3; ++k) m[k] = (g >> k & 1) ? (Ln[k] - c[k]) % Ln[k] : c[k];
      const long long qi = (m[2] * Ln[1] + m[1]) * Ln[0] + m[0];
      if (seen[qi]) continue;  // this mode already has an image (or is q itself)
      seen[qi] = 1;
      qs[slot] = static_cast<int>(qi);
      gs[slot] = g;
      ++slot;
    }
    for (int i = 0; i < 8; ++i) {
      op->items_q.push_back(i < slot ? qs[i] : -1);
      op->items_g.push_back(i < slot ? gs[i] : 0);
    }
    op->near_nimg = std::max(op->near_nimg, slot);
  }
  op->n_items = static_cast<long long>(op->items_q.size() / 8);
  while (op->near_nimg & (op->near_nimg - 1)) ++op->near_nimg;  // 1, 2, 4 or 8 (kernel instances)
}

// Lattice-path near field: y = (1/qn) IDFT(Shat . DFT(x)) truncated to the M
// cells per axis, for this rank's modes (zero elsewhere, so the ranks' partial
// products sum to the product). Forward passes read only the M nonzero cells
// per axis, inverse passes write only the M kept cells; the last one writes y.
// Lattice near field y = S x. With `fuse_loc` (the far field's locals, complete
// once `join` fires on the aux stream) the L2P y += U0 L is fused into the last
// inverse pass when that pass is an x-axis DMMA DFT; returns whether it was.
// the per-mode block products of the lattice near field: x_hat -> y_hat over
// this handle's stored blocks (DMMA ring, FMA GEMV or the block GEMM by shape)
void near_mode_stage(fpbem_cu_op* op, const c64* xh, c64* yh, int nrhs, cudaStream_t s) {
  const long long n = op->n;
  if (op->mode_lo > 0 || op->mode_hi < op->n_items)
    check(cudaMemsetAsync(yh, 0, static_cast<size_t>(nrhs * op->qn * n) * sizeof(c64), s), "near spectrum clear");
  ev_record(op, 7, s);
  // FPBEM_NEAR_MMA=0 keeps the FMA GEMV where the tensor-core mode product applies (A/B)
  static const bool mma_env = [] {
    const char* v = std::getenv("FPBEM_NEAR_MMA");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  int nw_, kc_, ring_;
  size_t smem_;
  if (mma_env && mode_mma_shape(op->n, nrhs * op->near_nimg, &nw_, &kc_, &ring_, &smem_)) {
    check(launch_mode_mma(op->shat, op->items, op->n_items, op->perm, xh, yh, op->n, op->mode_lo, op->mode_hi,
                          op->qn, nrhs, op->near_nimg, s),
          "near mode mma");
  } else if (nrhs * op->near_nimg <= kModeGemvMaxAcc) {
    check(launch_mode_gemv(op->shat, op->items, op->n_items, op->perm, xh, yh, op->n, op->mode_lo, op->mode_hi,
                           op->qn, nrhs, op->near_nimg, s),
          "near mode gemv");
  } else {
    build_mode_jobs(op, nrhs);
    check(launch_block_gemm(op->shat, n * n, op->n, op->n, xh, yh, op->n, nullptr, op->mjobs, op->n_mjobs, op->n,
                            op->n, op->qn * n, nrhs, s, op->qn * n, op->perm, op->items, op->n_items),
          "near mode gemm");
  }
  ev_record(op, 8, s);
  op->launches++;
}

bool near_fft_apply(fpbem_cu_op* op, const c64* x, c64* y, int nrhs, cudaStream_t s, const c64* fuse_loc = nullptr,
                    cudaEvent_t join = nullptr) {
  Nvtx range("near field (lattice convolution)");
  const long long n = op->n, r = nrhs;
  const int Mx = op->counts[0], My = op->counts[1], Mz = op->counts[2];
  const int Lx = op->Ln[0], Ly = op->Ln[1], Lz = op->Ln[2];
  c64* bufs[2] = {op->nfa, op->nfb};
  int which = 0;
  const c64* cur = x;
  auto fwd = [&](int axis, long long n_a, int m, int l, long long inner) {
    c64* out = bufs[which];
    which ^= 1;
    check(launch_dft_axis(cur, out, op->twn[axis], n_a, m, l, inner, l, false, 1.0, s), "near dft");
    op->launches++;
    cur = out;
  };
  // x and y together per (plane, field) for 2-D lattices (the M2L's plane
  // kernel; measured faster there, slower on the 3-D lattices of cfg3 / cfg5:
  // tools/ab_near_xy.sh); FPBEM_NEAR_XY=0 keeps the axis passes
  static const bool xy_env = [] {
    const char* v = std::getenv("FPBEM_NEAR_XY");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const bool xy = xy_env && Lx > 1 && Ly > 1 && Lz == 1 && n <= 0x7fffffffLL &&
                  xy_plane_smem(Mx, My, Lx, Ly, false) <= 200 * 1024 && xy_plane_smem(Mx, My, Lx, Ly, true) <= 200 * 1024;
  if (xy) {
    c64* out = bufs[which];
    which ^= 1;
    check(launch_xy_plane(cur, out, op->twn[0], op->twn[1], Mx, My, Lx, Ly, static_cast<int>(r * Mz),
                          static_cast<int>(n), false, 1.0, s),
          "near xy dft");
    op->launches++;
    cur = out;
  } else {
    if (Lx > 1) fwd(0, r * My * Mz, Mx, Lx, n);
    if (Ly > 1) fwd(1, r * Mz, My, Ly, Lx * n);
  }
  if (Lz > 1) fwd(2, r, Mz, Lz, static_cast<long long>(Ly) * Lx * n);
  c64* yh = bufs[which];
  which ^= 1;
  near_mode_stage(op, cur, yh, nrhs, s);
  cur = yh;
  int left = (Lx > 1) + (Ly > 1) + (Lz > 1);
  const double scale = 1.0 / static_cast<double>(op->qn);
  bool fused = false;
  auto inv = [&](int axis, long long n_a, int l, int m, long long inner) {
    const bool last = --left == 0;
    c64* out = last ? y : bufs[which];
    which ^= 1;
    if (last && axis == 0 && fuse_loc && dft_l2p_supported(l, m, op->b)) {
      check(cudaStreamWaitEvent(s, join, 0), "join");  // the locals of the far field
      check(launch_dft_axis_l2p(cur, out, op->twn[axis], n_a, l, m, inner, l, scale, op->u0, fuse_loc, op->b, nrhs,
                                s),
            "near inverse dft + l2p");
      fused = true;
    } else {
      check(launch_dft_axis(cur, out, op->twn[axis], n_a, l, m, inner, l, true, last ? scale : 1.0, s),
            "near inverse dft");
    }
    op->launches++;
    cur = out;
  };
  if (Lz > 1) inv(2, r, Lz, Mz, static_cast<long long>(Ly) * Lx * n);
  if (xy) {  // the last inverse pass: writes y with the 1/q scale
    check(launch_xy_plane(cur, y, op->twn[0], op->twn[1], Mx, My, Lx, Ly, static_cast<int>(r * Mz),
                          static_cast<int>(n), true, scale, s),
          "near xy inverse dft");
    op->launches++;
  } else {
    if (Ly > 1) inv(1, r * Mz, Ly, My, Lx * n);
    if (Lx > 1) inv(0, r * My * Mz, Lx, Mx, n);
  }
  return fused;
}

void twiddles(fpbem_cu_op* op, int L, c64** out) {
  std::vector<c64> t(L);
  for (int j = 0; j < L; ++j) {
    long double a = -2.0L * 3.141592653589793238462643383279502884L * j / L;
    t[j] = cmk(static_cast<double>(std::cos(a)), static_cast<double>(std::sin(a)));
  }
  *out = dalloc<c64>(L, "twiddles");
  h2d(*out, t.data(), L * sizeof(c64), op->stream, "twiddle upload");
}

// lattice DFT of the embedded K column on the device (src/structured.cpp:63-108):
// scatter the n_far bank blocks to slot (o mod L), DFT over every axis
void build_spectrum(fpbem_cu_op* op, int n_far, const int* far_offsets, const fpbem_c64* far_blocks,
                    bool blocks_on_device, const fpbem_c64* prebuilt, c64** out) {
  const int b2 = op->b * op->b;
  const size_t total = static_cast<size_t>(op->q_total) * b2;
  const long long Lx = op->L[0], Ly = op->L[1], Lz = op->L[2];
  using DevPtr = std::unique_ptr<void, decltype(&cudaFree)>;  // temporaries freed on every exit path
  c64* work = dalloc<c64>(total, "spectrum");
  DevPtr keep_work(work, &cudaFree);
  DevPtr keep_tmp(nullptr, &cudaFree), keep_offs(nullptr, &cudaFree), keep_staged(nullptr, &cudaFree);
  c64* cur = work;
  c64* tmp = nullptr;
  if (prebuilt) {
    h2d(work, prebuilt, total * sizeof(c64), op->stream, "spectrum upload");
  } else {
    tmp = dalloc<c64>(total, "spectrum scratch");
    keep_tmp.reset(tmp);
    const c64* blocks = reinterpret_cast<const c64*>(far_blocks);  // device bank (fpbem_cu_m2l_bank)
    if (!blocks_on_device) {
      c64* staged = dalloc<c64>(static_cast<size_t>(n_far) * b2, "far bank");
      keep_staged.reset(staged);
      if (n_far > 0)
        h2d(staged, far_blocks, static_cast<size_t>(n_far) * b2 * sizeof(c64), op->stream, "far bank upload");
      blocks = staged;
    }
    int* offs = dalloc<int>(static_cast<size_t>(n_far) * 3, "far offsets");
    keep_offs.reset(offs);
    if (n_far > 0)
      h2d(offs, far_offsets, static_cast<size_t>(n_far) * 3 * sizeof(int), op->stream, "far offsets upload");
    check(cudaMemsetAsync(work, 0, total * sizeof(c64), op->stream), "spectrum clear");
    check(launch_scatter_bank(blocks, offs, n_far, b2, op->L[0], op->L[1], op->L[2], work, op->stream),
          "scatter bank");
    c64* nxt = tmp;
    if (Lx > 1) {
      check(launch_dft_axis(cur, nxt, op->tw[0], Ly * Lz, op->L[0], op->L[0], b2, op->L[0], false, 1.0, op->stream),
            "spectrum dft x");
      std::swap(cur, nxt);
    }
    if (Ly > 1) {
      check(launch_dft_axis(cur, nxt, op->tw[1], Lz, op->L[1], op->L[1], Lx * b2, op->L[1], false, 1.0, op->stream),
            "spectrum dft y");
      std::swap(cur, nxt);
    }
    if (Lz > 1) {
      check(launch_dft_axis(cur, nxt, op->tw[2], 1, op->L[2], op->L[2], Lx * Ly * b2, op->L[2], false, 1.0,
                            op->stream),
            "spectrum dft z");
      std::swap(cur, nxt);
    }
  }
  check(cudaStreamSynchronize(op->stream), "spectrum build");
  // the result stays in whichever buffer the last pass wrote
  if (cur == work)
    keep_work.release();
  else
    keep_tmp.release();
  *out = cur;
}

void ev_record(fpbem_cu_op* op, int i, cudaStream_t st) {
  if (op->timing) cudaEventRecord(op->ev[i], st);
}

// Pruned separable lattice DFT, per-mode product, pruned inverse:
// moments (op->mom) -> locals (op->loc), CirculantSpectrum::matvec restated
// (src/structured.cpp:122-166), everything enqueued on `s`.
struct M2lPass {
  int kind;  // 0 dft, 1 mode product, 2 fused z-dft + mode product + inverse z-dft,
             // 3 / 4 forward / inverse x+y plane DFTs (one kernel each),
             // 5 the flat Λ stream in place on the z-extended field
  long long n_a;
  int n_in, n_out;
  long long inner;
  int L;
  int axis;
  bool back;
};

// the M2L's pass list for nrhs right-hand sides (CirculantSpectrum::matvec as
// pruned separable DFT passes, src/structured.cpp:122-166)
std::vector<M2lPass> m2l_plan(fpbem_cu_op* op, int nrhs) {
  const long long E = static_cast<long long>(nrhs) * op->b;
  const long long Mx = op->counts[0], My = op->counts[1], Mz = op->counts[2];
  const long long Lx = op->L[0], Ly = op->L[1], Lz = op->L[2];
  using Pass = M2lPass;
  std::vector<Pass> passes;
  long long cx = Mx, cy = My;  // current x / y extents
  // z forward + mode product + z inverse fused into one kernel when the
  // column's fields fit in shared memory (FPBEM_M2L_FUSE=0 disables)
  static const char* fz = std::getenv("FPBEM_M2L_FUSE");
  // the z stage as z-DFT axis passes around one flat Λ stream over all modes (kind 5) wherever the
  // stream kernel applies; FPBEM_M2L_Z=fused keeps the per-column fused kernel (A/B, and the form
  // the slab plan uses). Read per plan, not cached: the parity tests switch it within one process
  const char* zenv = std::getenv("FPBEM_M2L_Z");
  const bool z_stream_env = !(zenv && std::strcmp(zenv, "fused") == 0);
  const bool z_stream = z_stream_env && Lz > 1 && mode_stream_ring(static_cast<int>(E), op->b) >= 2;
  const bool fuse_z = !z_stream && Lz > 1 && !(fz && std::strcmp(fz, "0") == 0) &&
                      m2l_zfused_ring(static_cast<int>(Mz), static_cast<int>(Lz), static_cast<int>(E), op->b) > 0;
  // x and y together in shared memory per z-plane when the plane fits (FPBEM_M2L_XY=0: per-axis passes)
  static const int xy_env = [] {  // 0: per-axis passes; 2: plane kernels wherever they fit; else the rule below
    const char* v = std::getenv("FPBEM_M2L_XY");
    return v ? std::atoi(v) : 1;
  }();
  // where it measured faster than the per-axis passes: enough (plane, field)
  // CTAs to fill the GPU without splitting (cfg3), or small planes with both axes periodic (cfg2)
  const bool xy_wins = Mz * E >= 2LL * 148 || (Lx > 1 && Ly > 1 && Lx * Ly <= 1024);
  const bool fuse_xy = xy_env != 0 && (xy_wins || xy_env == 2) && (Lx > 1 || Ly > 1) &&
                       xy_plane_smem(static_cast<int>(Mx), static_cast<int>(My), static_cast<int>(Lx),
                                     static_cast<int>(Ly), true) <= 200 * 1024 &&
                       xy_plane_smem(static_cast<int>(Mx), static_cast<int>(My), static_cast<int>(Lx),
                                     static_cast<int>(Ly), false) <= 200 * 1024;
  if (fuse_xy) {
    passes.push_back({3, 0, 0, 0, 0, 0, -1, false});
    cx = Lx;
    cy = Ly;
  } else {
    if (Lx > 1) {
      passes.push_back({0, My * Mz, static_cast<int>(Mx), static_cast<int>(Lx), E, static_cast<int>(Lx), 0, false});
      cx = Lx;
    }
    if (Ly > 1) {
      passes.push_back({0, Mz, static_cast<int>(My), static_cast<int>(Ly), cx * E, static_cast<int>(Ly), 1, false});
      cy = Ly;
    }
  }
  if (fuse_z) {
    passes.push_back({2, 0, 0, 0, 0, static_cast<int>(Lz), 2, false});
  } else {
    if (Lz > 1)
      passes.push_back({0, 1, static_cast<int>(Mz), static_cast<int>(Lz), cy * cx * E, static_cast<int>(Lz), 2, false});
    passes.push_back({z_stream ? 5 : 1, 0, 0, 0, 0, 0, -1, false});
    if (Lz > 1)
      passes.push_back({0, 1, static_cast<int>(Lz), static_cast<int>(Mz), Ly * Lx * E, static_cast<int>(Lz), 2, true});
  }
  if (fuse_xy) {
    passes.push_back({4, 0, 0, 0, 0, 0, -1, true});
  } else {
    if (Ly > 1)
      passes.push_back({0, Mz, static_cast<int>(Ly), static_cast<int>(My), Lx * E, static_cast<int>(Ly), 1, true});
    if (Lx > 1)
      passes.push_back({0, My * Mz, static_cast<int>(Lx), static_cast<int>(Mx), E, static_cast<int>(Lx), 0, true});
  }
  return passes;
}

// FPBEM_M2L_QUAD=0: the flat Λ stream without the z-reflection parity (A/B; read per call)
bool zquad_on() {
  const char* v = std::getenv("FPBEM_M2L_QUAD");
  return !(v && std::strcmp(v, "0") == 0);
}

// M2L moments -> locals. xy_done: the first pass (the forward x+y plane DFTs,
// kind 3) already ran into op->fa (the pipelined host apply does it slab by slab)
void m2l_apply(fpbem_cu_op* op, int nrhs, cudaStream_t s, const c64* moments, const c64* lambda, c64* locals,
               bool xy_done = false) {
  const long long E = static_cast<long long>(nrhs) * op->b;
  const long long Mx = op->counts[0], My = op->counts[1], Mz = op->counts[2];
  const long long Lx = op->L[0], Ly = op->L[1], Lz = op->L[2];
  using Pass = M2lPass;
  const std::vector<Pass> passes = m2l_plan(op, nrhs);
  if (xy_done && (passes.empty() || passes[0].kind != 3)) fail(FPBEM_CU_EINVAL, "m2l: no x+y plane pass to skip");
  int last_dft = -1;  // the pass that applies the 1/q scale
  for (int i = 0; i < static_cast<int>(passes.size()); ++i)
    if ((passes[i].kind == 0 && passes[i].back) || passes[i].kind == 2 || passes[i].kind == 4) last_dft = i;
  const c64* cur = xy_done ? op->fa : moments;
  c64* bufs[2] = {op->fa, op->fb};
  int which = xy_done ? 1 : 0;
  for (int i = xy_done ? 1 : 0; i < static_cast<int>(passes.size()); ++i) {
    const Pass& p = passes[i];
    const bool final = i + 1 == static_cast<int>(passes.size());
    c64* out = final ? locals : bufs[which];
    if (p.kind == 3 || p.kind == 4) {
      const double scale = (i == last_dft) ? 1.0 / static_cast<double>(op->q_total) : 1.0;
      check(launch_xy_plane(cur, out, op->tw[0], op->tw[1], static_cast<int>(Mx), static_cast<int>(My),
                            static_cast<int>(Lx), static_cast<int>(Ly), static_cast<int>(Mz), static_cast<int>(E),
                            p.kind == 4, scale, s),
            "lattice xy dft");
    } else if (p.kind == 5) {
      // in place on the z-extended field the forward z pass just wrote (one of op->fa / op->fb)
      const bool paired = lambda == op->lambda && op->lam_paired;
      check(launch_mode_stream(const_cast<c64*>(cur), lambda, static_cast<int>(Lz), Ly * Lx, static_cast<int>(E),
                               op->b, paired ? op->z_items_pair : op->z_items_single,
                               paired ? op->n_z_items_pair : op->n_z_items_single, paired && op->lam_zsym && zquad_on(),
                               s),
            "mode stream");
      op->launches++;
      continue;
    } else if (p.kind == 1) {
      check(launch_mode_product(lambda, cur, out, op->q_total, op->b, nrhs, s), "mode product");
    } else if (p.kind == 2) {
      const double scale = (i == last_dft) ? 1.0 / static_cast<double>(op->q_total) : 1.0;
      // the main spectrum's mirror parity lets one Λ stream serve a column and its mirror
      const bool paired = lambda == op->lambda && op->lam_paired;
      check(launch_m2l_zfused(cur, out, lambda, op->tw[2], static_cast<int>(Mz), static_cast<int>(Lz), Ly * Lx,
                              static_cast<int>(E), op->b, scale, paired ? op->z_items_pair : op->z_items_single,
                              paired ? op->n_z_items_pair : op->n_z_items_single, s),
            "m2l z-fused");
    } else {
      const double scale = (i == last_dft) ? 1.0 / static_cast<double>(op->q_total) : 1.0;
      check(launch_dft_axis(cur, out, op->tw[p.axis], p.n_a, p.n_in, p.n_out, p.inner, p.L, p.back, scale, s),
            "lattice dft");
    }
    op->launches++;
    cur = out;
    which ^= 1;
  }
}

// P2M / L2P as per-cell DMMA GEMMs (csrc/cellwise.cu); FPBEM_CELLWISE=0 keeps
// the FMA kernels (A/B)
bool cellwise_on() {
  static const bool on = [] {
    const char* v = std::getenv("FPBEM_CELLWISE");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  return on;
}

// Far field of one product: P2M (events 2-3) and M2L into op->loc (events 3-4);
// the Hankel image pair adds the K_hat term (src/fmm.cpp:256-263)
// P2M as the per-cell DMMA GEMM (V0 staged in shared memory per CTA) when there are
// enough cells to fill the GPU (cfg1's 8 cells: 16 us against the FMA kernel's 8);
// every product of a handle makes the same choice (same arithmetic, same bits)
bool p2m_cellwise(const fpbem_cu_op* op, int nrhs) {
  return cellwise_on() && cellwise_supported(op->b, op->n) &&
         static_cast<long long>(op->n_cells) * nrhs >= 2LL * device_sms();
}

void far_field(fpbem_cu_op* op, const c64* x, int nrhs, cudaStream_t a) {
  Nvtx range("far field (P2M + M2L)");
  ev_record(op, 2, a);
  if (p2m_cellwise(op, nrhs))  // M_c = V0 p_c: V0[m][k] = v0t[m n + k]
    check(launch_cellwise(op->v0t, op->n, 1, op->b, op->n, x, op->N, op->n, op->mom, op->b,
                          static_cast<long long>(nrhs) * op->b, nrhs, static_cast<long long>(op->n_cells) * nrhs,
                          false, a),
          "p2m");
  else
    check(launch_p2m(op->v0t, x, op->mom, op->n, op->b, op->N, nrhs, op->n_cells, a), "p2m");
  op->launches++;
  ev_record(op, 3, a);
  m2l_apply(op, nrhs, a, op->mom, op->lambda, op->loc);
  if (op->mirrored_level >= 0) {  // local += hankel_matvec(K_hat spectrum, mirror_permute(moments)) (src/fmm.cpp:262-263)
    const long long E = static_cast<long long>(nrhs) * op->b;
    check(launch_mirror_permute(op->mom, op->mom_perm, op->counts, op->mirrored_level, E, a), "mirror permute");
    m2l_apply(op, nrhs, a, op->mom_perm, op->lambda_hat, op->loc_hat);
    check(launch_add(op->loc, op->loc_hat, static_cast<long long>(op->n_cells) * E, a), "local image add");
    op->launches += 2;
  }
  ev_record(op, 4, a);
}

// Cost of the far field in near-field pair equivalents, measured on this
// device: t(P2M + M2L) / t(near GEMM over all pairs) x n_pairs, single RHS,
// all on the handle's stream (best of 3 after a warm-up). Rank 0 carries the
// far field under the pair partition, so it gets this many fewer pairs.
double calibrate_far_pairs(fpbem_cu_op* op) {
  if (op->n_pairs == 0 && !op->near_fft) return 0.0;
  const int rank = op->rank, nranks = op->nranks;
  const double far_pairs = op->far_pairs;
  set_partition(op, 0, 1, 0.0);
  cudaStream_t s = op->stream;
  c64* x = dalloc<c64>(static_cast<size_t>(op->N), "calibration input");
  std::unique_ptr<c64, decltype(&cudaFree)> keep_x(x, &cudaFree);
  check(cudaMemsetAsync(x, 0, static_cast<size_t>(op->N) * sizeof(c64), s), "calibration input");
  cudaEvent_t e[3];
  for (auto& ev : e) check(cudaEventCreate(&ev), "calibration events");
  std::unique_ptr<cudaEvent_t, void (*)(cudaEvent_t*)> keep_e(e, [](cudaEvent_t* v) {
    for (int i = 0; i < 3; ++i) cudaEventDestroy(v[i]);
  });
  c64* yc = nullptr;
  if (op->near_fft) yc = dalloc<c64>(static_cast<size_t>(op->N), "calibration output");
  std::unique_ptr<c64, decltype(&cudaFree)> keep_y(yc, &cudaFree);
  if (!op->near_fft) build_jobs(op, 1);
  float best_near = 1e30f, best_far = 1e30f;
  for (int it = 0; it < 4; ++it) {
    check(cudaEventRecord(e[0], s), "calibration");
    if (op->near_fft)
      near_fft_apply(op, x, yc, 1, s);
    else
      check(launch_block_gemm(op->S, static_cast<long long>(op->n) * op->n, op->n, op->n, x, op->W, op->n,
                              op->pair_src, op->jobs, op->n_jobs, op->n, op->n, op->N, 1, s),
            "calibration gemm");
    check(cudaEventRecord(e[1], s), "calibration");
    far_field(op, x, 1, s);
    check(cudaEventRecord(e[2], s), "calibration");
    check(cudaEventSynchronize(e[2]), "calibration");
    float t_near, t_far;
    cudaEventElapsedTime(&t_near, e[0], e[1]);
    cudaEventElapsedTime(&t_far, e[1], e[2]);
    if (it > 0) {
      best_near = std::min(best_near, t_near);
      best_far = std::min(best_far, t_far);
    }
  }
  set_partition(op, rank, nranks, far_pairs);
  const double units = op->near_fft ? static_cast<double>(op->n_items) : static_cast<double>(op->n_pairs);
  return best_near > 0.0f ? static_cast<double>(best_far) / best_near * units : 0.0;
}

// One FMM product for nrhs <= max_rhs right-hand sides, device pointers.
// Order of the sums follows src/fmm.cpp:253-267: y = S p, then y += U0 L.
// With an offset partition (nranks > 1) this rank computes the product of
// its own near-field offsets; rank 0 also adds the far field (P2M, M2L,
// L2P); with a communicator the partial products are all-reduced.
void apply_chunk(fpbem_cu_op* op, const c64* x, c64* y, int nrhs, bool reduce) {
  Nvtx range("fpbem apply (FmmOperators::matvec)");
  cudaStream_t s = op->stream;
  // FPBEM_SERIAL=1 runs P2M + M2L on the main stream (exact per-stage timing)
  static const bool serial = [] {
    const char* v = std::getenv("FPBEM_SERIAL");
    return v && std::strcmp(v, "1") == 0;
  }();
  cudaStream_t a = (serial || op->serial_timing) ? op->stream : op->aux;
  const bool far_here = op->rank == 0;
  if (!op->near_fft) build_jobs(op, nrhs);
  // fork: P2M + M2L on the aux stream while the near field runs on the main one
  check(cudaEventRecord(op->fork, s), "fork");
  check(cudaStreamWaitEvent(a, op->fork, 0), "fork");
  ev_record(op, 0, s);
  bool l2p_done = false;
  // the L2P fused into the last inverse near pass (FPBEM_FUSE_L2P=0 keeps it separate);
  // not under serial stage timing, where the far field runs on this stream
  static const bool fuse_env = [] {
    const char* v = std::getenv("FPBEM_FUSE_L2P");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const bool fuse = op->near_fft && far_here && fuse_env && a != s;
  if (fuse) {  // far field first on the aux stream, joined inside the near field before its last pass
    far_field(op, x, nrhs, a);
    check(cudaEventRecord(op->join, a), "join");
    l2p_done = near_fft_apply(op, x, y, nrhs, s, op->loc, op->join);  // y = S p (+ U0 L)
    ev_record(op, 1, s);
  } else if (op->near_fft) {
    near_fft_apply(op, x, y, nrhs, s);  // y = S p
  } else {
    check(launch_block_gemm(op->S, static_cast<long long>(op->n) * op->n, op->n, op->n, x, op->W, op->n,
                            op->pair_src, op->jobs, op->n_jobs, op->n, op->n, op->N, nrhs, s),
          "near gemm");
    op->launches += op->n_jobs > 0;
  }
  if (!fuse) {
    ev_record(op, 1, s);
    if (far_here) far_field(op, x, nrhs, a);
    check(cudaEventRecord(op->join, a), "join");
  }
  s = op->stream;
  check(cudaStreamWaitEvent(s, op->join, 0), "join");
  ev_record(op, 5, s);
  if (l2p_done) {
    // y already holds S p + U0 L
  } else if (!op->near_fft) {
    check(launch_near_reduce_l2p(op->W, op->tgt_ptr, op->tgt_pairs, op->u0, far_here ? op->loc : nullptr, y, op->n,
                                 op->b, op->n_cells, op->N, nrhs, false, s),
          "near reduce + l2p");
    op->launches++;
  } else if (far_here) {  // y += U0 L (src/fmm.cpp:265-267): the reduction with no pairs, accumulating
    check(launch_l2p_add(op->u0, op->loc, y, op->n, op->b, op->n_cells, op->N, nrhs, s), "l2p");
    op->launches++;
  }
  if (op->comm && reduce)  // sum the ranks' partial products, in place, on the same stream
    comm_allreduce(op->comm, reinterpret_cast<double*>(y), static_cast<size_t>(2) * op->N * nrhs, s);
  ev_record(op, 6, s);
  if (op->timing) {
    check(cudaEventSynchronize(op->ev[6]), "timing sync");
    float ms;
    cudaEventElapsedTime(&ms, op->ev[0], op->ev[1]);
    op->stage_ms[0] += ms;
    cudaEventElapsedTime(&ms, op->ev[5], op->ev[6]);
    op->stage_ms[1] += ms;
    cudaEventElapsedTime(&ms, op->ev[2], op->ev[3]);
    op->stage_ms[2] += ms;
    cudaEventElapsedTime(&ms, op->ev[3], op->ev[4]);
    op->stage_ms[3] += ms;
    cudaEventElapsedTime(&ms, op->ev[0], op->ev[6]);
    op->stage_ms[4] += ms;
    if (op->near_fft) {
      cudaEventElapsedTime(&ms, op->ev[7], op->ev[8]);
      op->stage_ms[5] += ms;
    }
    op->applies++;
  }
}

// Host-pointer product of one right-hand side with the copies overlapped
// (the C-ABI's synchronous FPBEM_CU_PTR_HOST apply, src/fmm.cpp:246-271 as an
// ApplyFn). x arrives in slabs of z-planes on a copy stream while the near
// field's x and y DFT passes run on the slabs already there; the far field
// starts once x is complete; after the z passes and the block products, the
// inverse y and x (+ L2P) passes run slab by slab and each slab of y goes back
// on a second copy stream while the next is computed. Same kernels, same
// arithmetic as apply_chunk. Applies to 3-D lattices on the lattice near
// field (cfg3, cfg5) with the fused L2P; returns false (nothing done) otherwise.
bool apply_host_pipelined(fpbem_cu_op* op, const c64* xh, c64* yh) {
  static const bool env = [] {
    const char* v = std::getenv("FPBEM_PIPE_H2D");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const int Mx = op->counts[0], My = op->counts[1], Mz = op->counts[2];
  const int Lx = op->Ln[0], Ly = op->Ln[1], Lz = op->Ln[2];
  if (!env || !op->near_fft || op->nranks > 1 || op->comm || op->mirrored_level >= 0 || op->timing ||
      Mz < 4 || Lx < 2 || Ly < 2 || Lz < 2 || !dft_l2p_supported(Lx, Mx, op->b) ||
      op->mode_lo > 0 || op->mode_hi < op->n_items)
    return false;
  const long long n = op->n;
  static const int chunks_env = [] {  // FPBEM_PIPE_CHUNKS: z-plane slabs per product (A/B), at most 8
    const char* v = std::getenv("FPBEM_PIPE_CHUNKS");
    const int c = v ? std::atoi(v) : 4;
    return c < 1 ? 1 : (c > 8 ? 8 : c);
  }();
  const int chunks = std::min(chunks_env, Mz);
  cudaStream_t s = op->stream, a = op->aux;
  if (!op->cin) {
    check(cudaStreamCreateWithFlags(&op->cin, cudaStreamNonBlocking), "copy-in stream");
    check(cudaStreamCreateWithFlags(&op->cout, cudaStreamNonBlocking), "copy-out stream");
    for (int i = 0; i < 8; ++i) {
      check(cudaEventCreateWithFlags(&op->pev_in[i], cudaEventDisableTiming), "pipeline events");
      check(cudaEventCreateWithFlags(&op->pev_out[i], cudaEventDisableTiming), "pipeline events");
    }
  }
  auto z0_of = [&](int c) { return static_cast<long long>(Mz) * c / chunks; };
  const long long xplane = static_cast<long long>(My) * Mx * n;  // one z-plane of x / y
  // FPBEM_PIPE_TRACE=1: the product's timeline on stderr (timed events; diagnostic)
  static const bool trace = [] {
    const char* v = std::getenv("FPBEM_PIPE_TRACE");
    return v && std::atoi(v) != 0;
  }();
  static cudaEvent_t tev[8];
  static bool tev_ok = false;
  if (trace && !tev_ok) {
    for (auto& e : tev) check(cudaEventCreate(&e), "trace events");
    tev_ok = true;
  }
  auto mark = [&](int i, cudaStream_t st) {
    if (trace) check(cudaEventRecord(tev[i], st), "trace");
  };
  mark(0, s);
  // the copy-in stream starts after whatever the handle's stream has queued (staging reuse)
  check(cudaEventRecord(op->fork, s), "pipeline fork");
  check(cudaStreamWaitEvent(op->cin, op->fork, 0), "pipeline fork");
  for (int c = 0; c < chunks; ++c) {
    const long long z0 = z0_of(c), z1 = z0_of(c + 1);
    check(cudaMemcpyAsync(op->xin + z0 * xplane, xh + z0 * xplane, static_cast<size_t>((z1 - z0) * xplane) * sizeof(c64),
                          cudaMemcpyHostToDevice, op->cin),
          "x upload");
    check(cudaEventRecord(op->pev_in[c], op->cin), "pipeline event");
  }
  mark(1, op->cin);  // x uploaded
  // far field (aux stream): P2M and the forward x+y plane DFTs of the M2L slab
  // by slab as x arrives, the rest once x is complete; joined before the first L2P
  const std::vector<M2lPass> plan = m2l_plan(op, 1);
  const bool far_xy = !plan.empty() && plan[0].kind == 3;
  const int fLx = op->L[0], fLy = op->L[1];
  for (int c = 0; c < chunks; ++c) {
    const long long z0 = z0_of(c), z1 = z0_of(c + 1);
    const long long c0 = z0 * My * Mx, nc = (z1 - z0) * My * Mx;  // the slab's cells
    check(cudaStreamWaitEvent(a, op->pev_in[c], 0), "pipeline far");
    if (p2m_cellwise(op, 1))  // M_c = V0 p_c (src/fmm.cpp:256-259), as far_field decides
      check(launch_cellwise(op->v0t, op->n, 1, op->b, op->n, op->xin + c0 * n, op->N, op->n, op->mom + c0 * op->b,
                            op->b, op->b, 1, nc, false, a),
            "p2m");
    else
      check(launch_p2m(op->v0t, op->xin + c0 * n, op->mom + c0 * op->b, op->n, op->b, op->N, 1, static_cast<int>(nc),
                       a),
            "p2m");
    op->launches++;
    if (far_xy) {
      check(launch_xy_plane(op->mom + c0 * op->b, op->fa + z0 * fLy * fLx * op->b, op->tw[0], op->tw[1], Mx, My, fLx,
                            fLy, static_cast<int>(z1 - z0), op->b, false, 1.0, a),
            "lattice xy dft");
      op->launches++;
    }
  }
  m2l_apply(op, 1, a, op->mom, op->lambda, op->loc, far_xy);
  mark(2, a);  // far field done
  check(cudaEventRecord(op->join, a), "pipeline join");
  // near field: x and y passes slab by slab (buffers as near_fft_apply: x -> nfa -> nfb)
  for (int c = 0; c < chunks; ++c) {
    const long long z0 = z0_of(c), z1 = z0_of(c + 1), m = z1 - z0;
    check(cudaStreamWaitEvent(s, op->pev_in[c], 0), "pipeline in");
    check(launch_dft_axis(op->xin + z0 * xplane, op->nfa + z0 * My * Lx * n, op->twn[0], m * My, Mx, Lx, n, Lx, false,
                          1.0, s),
          "near dft x");
    check(launch_dft_axis(op->nfa + z0 * My * Lx * n, op->nfb + z0 * static_cast<long long>(Ly) * Lx * n, op->twn[1],
                          m, My, Ly, static_cast<long long>(Lx) * n, Ly, false, 1.0, s),
          "near dft y");
    op->launches += 2;
  }
  const long long zstride = static_cast<long long>(Ly) * Lx * n;
  mark(3, s);  // near x, y passes done
  check(launch_dft_axis(op->nfb, op->nfa, op->twn[2], 1, Mz, Lz, zstride, Lz, false, 1.0, s), "near dft z");
  near_mode_stage(op, op->nfa, op->nfb, 1, s);
  check(launch_dft_axis(op->nfb, op->nfa, op->twn[2], 1, Lz, Mz, zstride, Lz, true, 1.0, s), "near inverse dft z");
  mark(4, s);  // near inverse z done
  op->launches += 2;
  const double scale = 1.0 / static_cast<double>(op->qn);
  check(cudaStreamWaitEvent(s, op->join, 0), "pipeline join");  // the locals of the far field
  for (int c = 0; c < chunks; ++c) {
    const long long z0 = z0_of(c), z1 = z0_of(c + 1), m = z1 - z0;
    check(launch_dft_axis(op->nfa + z0 * zstride, op->nfb + z0 * My * Lx * n, op->twn[1], m, Ly, My,
                          static_cast<long long>(Lx) * n, Ly, true, 1.0, s),
          "near inverse dft y");
    check(launch_dft_axis_l2p(op->nfb + z0 * My * Lx * n, op->yout + z0 * xplane, op->twn[0], m * My, Lx, Mx, n, Lx,
                              scale, op->u0, op->loc + z0 * My * Mx * op->b, op->b, 1, s),
          "near inverse dft x + l2p");
    op->launches += 2;
    check(cudaEventRecord(op->pev_out[c], s), "pipeline event");
    if (c == 0) mark(5, s);  // first slab of y ready
    if (c == chunks - 1) mark(6, s);  // last slab of y ready
    check(cudaStreamWaitEvent(op->cout, op->pev_out[c], 0), "pipeline out");
    check(cudaMemcpyAsync(yh + z0 * xplane, op->yout + z0 * xplane, static_cast<size_t>(m * xplane) * sizeof(c64),
                          cudaMemcpyDeviceToHost, op->cout),
          "y download");
  }
  mark(7, op->cout);  // y downloaded
  check(cudaStreamSynchronize(op->cout), "apply sync");
  if (trace) {
    float t[8] = {0};
    for (int i = 1; i < 8; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[i]);
    std::fprintf(stderr,
                 "[fpbem pipe] x up %.3f | far done %.3f | near xy %.3f | near z-inv %.3f | y slab0 %.3f | y last %.3f | "
                 "y down %.3f ms\n",
                 t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
  }
  return true;
}

void apply_device(fpbem_cu_op* op, const c64* x, c64* y, int nrhs, bool reduce) {
  for (int r0 = 0; r0 < nrhs; r0 += op->max_rhs) {
    const int c = std::min(op->max_rhs, nrhs - r0);
    apply_chunk(op, x + static_cast<long long>(r0) * op->N, y + static_cast<long long>(r0) * op->N, c, reduce);
  }
}

// Direct Toeplitz GEMM or lattice convolution for the near field. Cost model
// (DESIGN.md §3.1b), at the largest batch the handle serves: the direct path is
// FP64-tensor bound, 8 n^2 flops per (pair, rhs) at ~36 TFLOP/s; the lattice
// path streams the block spectrum once (16 n^2 bytes per mode, ~6 TB/s) or, for
// many right-hand sides, is bound by its 8 n^2 flops per (mode, rhs), plus the
// pruned DFT passes of x and y. Lattice when it is >= 20 % cheaper and its
// spectrum fits in a third of the free device memory. FPBEM_NEAR=direct|lattice
// overrides the descriptor (A/B runs).
void choose_near_path(fpbem_cu_op* op, const fpbem_cu_fmm_desc* d) {
  int path = d->near_path;
  if (const char* e = std::getenv("FPBEM_NEAR")) {
    if (std::strcmp(e, "direct") == 0) path = FPBEM_CU_NEAR_DIRECT;
    if (std::strcmp(e, "lattice") == 0) path = FPBEM_CU_NEAR_LATTICE;
  }
  if (path < FPBEM_CU_NEAR_AUTO || path > FPBEM_CU_NEAR_LATTICE) fail(FPBEM_CU_EINVAL, "create: bad near_path");
  const bool possible = op->n_hat == 0 && op->n_cells > 1 && d->n_near > 0;
  if (path == FPBEM_CU_NEAR_LATTICE && !possible)
    fail(FPBEM_CU_EINVAL, "create: lattice near field needs >= 2 cells, near blocks and no half-space image pair");
  int R[3] = {0, 0, 0};
  for (int s = 0; s < d->n_near; ++s)
    for (int k = 0; k < 3; ++k) R[k] = std::max(R[k], std::abs(op->near_offsets[3 * s + k]));
  int Ln[3];
  long long qn = 1;
  for (int k = 0; k < 3; ++k) {
    Ln[k] = op->counts[k] == 1 ? 1 : op->counts[k] + R[k];
    qn *= Ln[k];
  }
  const double nn = static_cast<double>(op->n) * op->n;
  build_items(op, Ln);  // stored blocks: one per orbit of modes under the verified symmetries
  const double spec_bytes = 16.0 * nn * static_cast<double>(op->n_items);
  bool use = path == FPBEM_CU_NEAR_LATTICE;
  if (path == FPBEM_CU_NEAR_AUTO && possible) {
    const double r = op->max_rhs;
    const double t_direct = 8.0 * nn * op->n_pairs * r / 36e12;
    int axes = 0;
    for (int k = 0; k < 3; ++k) axes += Ln[k] > 1;
    const double t_pass = axes * 2.0 * 32.0 * r * op->n * static_cast<double>(qn + op->n_cells) / 4e12;
    const double t_lat = std::max(spec_bytes / 6e12, 8.0 * nn * static_cast<double>(qn) * r / 30e12) + t_pass;
    // (build transient: two full spectra)
    size_t free_b = 0, total_b = 0;
    check(cudaMemGetInfo(&free_b, &total_b), "mem info");
    use = t_lat < 0.8 * t_direct && 2.5 * 16.0 * nn * qn < static_cast<double>(free_b) / 1.5;
  }
  if (!use) return;
  op->near_fft = true;
  for (int k = 0; k < 3; ++k) op->Ln[k] = Ln[k];
  op->qn = qn;
}

void ensure_pinned(fpbem_cu_op* op, size_t bytes) {
  if (op->pinned_bytes >= bytes) return;
  if (op->pinned) cudaFreeHost(op->pinned);
  op->pinned = nullptr;
  check(cudaMallocHost(&op->pinned, bytes), "pinned host buffer");
  op->pinned_bytes = bytes;
}

}  // namespace fpbem_cu

extern "C" {

const char* fpbem_cu_last_error(void) { return g_err.c_str(); }
const char* fpbem_cu_version(void) { return "fpbem_cuda 0.1 sm_100a"; }

int fpbem_cu_fmm_create(const fpbem_cu_fmm_desc* d, int device, fpbem_cu_op** out) {
  return guard([&] {
    if (!d || !out) fail(FPBEM_CU_EINVAL, "create: null argument");
    *out = nullptr;
    for (int k = 0; k < 3; ++k)
      if (d->counts[k] < 1) fail(FPBEM_CU_EDIM, "create: counts must be >= 1");
    if (d->n_dof < 1 || d->n_coef < 1 || d->n_coef > 256) fail(FPBEM_CU_EDIM, "create: bad n_dof / n_coef (n_t <= 15)");
    if (d->mirrored_level < -1 || d->mirrored_level > 2) fail(FPBEM_CU_EINVAL, "create: mirrored_level in [-1, 2]");
    if (d->mirrored_level >= 0 && ((d->n_hat > 0 && (!d->hat_indices || !d->hat_blocks)) ||
                                   (!d->lambda_hat && d->n_far_hat > 0 && (!d->far_hat_indices || !d->far_hat_blocks))))
      fail(FPBEM_CU_EINVAL, "create: half-space image pair missing");
    if (!d->u0 || !d->v0) fail(FPBEM_CU_EINVAL, "create: u0 / v0 required");
    if (d->n_near > 0 && (!d->near_offsets || !d->near_blocks)) fail(FPBEM_CU_EINVAL, "create: near blocks missing");
    if (!d->lambda && d->n_far > 0 && (!d->far_offsets || !d->far_blocks))
      fail(FPBEM_CU_EINVAL, "create: far bank missing");
    check(cudaSetDevice(device), "set device");
    auto* op = new fpbem_cu_op();
    std::unique_ptr<fpbem_cu_op, void (*)(fpbem_cu_op*)> guard_op(op, fpbem_cu_fmm_destroy);
    op->device = device;
    check(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking), "stream");
    op->own_stream = true;
    {  // aux stream (P2M + M2L) at the highest priority: its few CTAs are
       // scheduled ahead of the near-field GEMM's as SM slots free up
      int lo = 0, hi = 0;
      check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
      check(cudaStreamCreateWithPriority(&op->aux, cudaStreamNonBlocking, hi), "aux stream");
    }
    check(cudaEventCreateWithFlags(&op->fork, cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&op->join, cudaEventDisableTiming), "event");
    for (int k = 0; k < 3; ++k) op->counts[k] = d->counts[k];
    op->n = d->n_dof;
    op->b = d->n_coef;
    op->n_cells = d->counts[0] * d->counts[1] * d->counts[2];
    op->N = static_cast<long long>(op->n_cells) * op->n;
    op->max_rhs = std::max(1, d->max_rhs);

    // near field: pairs per offset (offset order), per-target CSR in offset order
    op->n_near = d->n_near;
    op->near_offsets.assign(d->near_offsets, d->near_offsets + 3 * d->n_near);
    const int* m = d->counts;
    std::vector<int> psrc;
    op->pair_start.assign(1, 0);
    for (int s = 0; s < d->n_near; ++s) {
      const int ox = op->near_offsets[3 * s], oy = op->near_offsets[3 * s + 1], oz = op->near_offsets[3 * s + 2];
      if (std::abs(ox) >= m[0] || std::abs(oy) >= m[1] || std::abs(oz) >= m[2])
        fail(FPBEM_CU_EDIM, "create: near offset outside [1-M, M-1]");
      for (int tz = 0; tz < m[2]; ++tz)
        for (int ty = 0; ty < m[1]; ++ty)
          for (int tx = 0; tx < m[0]; ++tx) {
            const int sx = tx - ox, sy = ty - oy, sz = tz - oz;
            if (sx < 0 || sx >= m[0] || sy < 0 || sy >= m[1] || sz < 0 || sz >= m[2]) continue;
            op->pair_tgt.push_back(tx + m[0] * (ty + m[1] * tz));
            psrc.push_back(sx + m[0] * (sy + m[1] * sz));
          }
      op->pair_start.push_back(static_cast<int>(psrc.size()));
    }
    // S_hat slots follow: Hankel pairs, src[a] = idx[a] - t[a], src[d] = t[d] - idx[d]
    // (BlockHankelMatrix::matvec, src/assembly.cpp:152-178)
    op->mirrored_level = d->mirrored_level;
    op->n_hat = d->mirrored_level >= 0 ? d->n_hat : 0;
    for (int h = 0; h < op->n_hat; ++h) {
      const int* idx = d->hat_indices + 3 * h;
      for (int tz = 0; tz < m[2]; ++tz)
        for (int ty = 0; ty < m[1]; ++ty)
          for (int tx = 0; tx < m[0]; ++tx) {
            const int t[3] = {tx, ty, tz};
            int src[3];
            bool ok = true;
            for (int k = 0; k < 3 && ok; ++k) {
              src[k] = k == op->mirrored_level ? idx[k] - t[k] : t[k] - idx[k];
              ok = src[k] >= 0 && src[k] < m[k];
            }
            if (!ok) continue;
            op->pair_tgt.push_back(tx + m[0] * (ty + m[1] * tz));
            psrc.push_back(src[0] + m[0] * (src[1] + m[1] * src[2]));
          }
      op->pair_start.push_back(static_cast<int>(psrc.size()));
    }
    op->n_pairs = static_cast<int>(psrc.size());
    const int n_slots = d->n_near + op->n_hat;
    op->n_near = n_slots;  // slot count seen by the GEMM / reduction / partition
    op->pair_lo = 0;
    op->pair_hi = op->n_pairs;
    const size_t nn = static_cast<size_t>(op->n) * op->n;
    op->S = dalloc<c64>(nn * n_slots, "near blocks");
    auto put = [&](c64* dst, const fpbem_c64* src, size_t count, const char* what) {
      if (count == 0) return;
      if (d->blocks_on_device) {
        check(cudaMemcpyAsync(dst, src, count * sizeof(c64), cudaMemcpyDeviceToDevice, op->stream), what);
        check(cudaStreamSynchronize(op->stream), what);
      } else {
        h2d(dst, src, count * sizeof(c64), op->stream, what);
      }
    };
    put(op->S, d->near_blocks, nn * d->n_near, "S upload");
    put(op->S + nn * d->n_near, d->hat_blocks, nn * op->n_hat, "S_hat upload");
    op->pair_src = dalloc<int>(psrc.size(), "pair sources");
    if (!psrc.empty()) h2d(op->pair_src, psrc.data(), psrc.size() * sizeof(int), op->stream, "pairs");
    build_target_csr(op);

    // expansions
    const size_t nb = static_cast<size_t>(op->n) * op->b;
    op->u0 = dalloc<c64>(nb, "u0");
    op->v0 = dalloc<c64>(nb, "v0");
    h2d(op->u0, d->u0, nb * sizeof(c64), op->stream, "u0 upload");
    h2d(op->v0, d->v0, nb * sizeof(c64), op->stream, "v0 upload");
    {
      std::vector<fpbem_c64> t(nb);  // V0 is b x n column-major: v0[c + b j] -> v0t[c n + j]
      for (int j = 0; j < op->n; ++j)
        for (int c = 0; c < op->b; ++c) t[static_cast<size_t>(c) * op->n + j] = d->v0[static_cast<size_t>(j) * op->b + c];
      op->v0t = dalloc<c64>(nb, "v0t");
      h2d(op->v0t, t.data(), nb * sizeof(c64), op->stream, "v0t upload");
    }

    // spectrum sizes: caller's, else the reference's 7-smooth padding
    for (int k = 0; k < 3; ++k) {
      int l = d->fft_sizes[k];
      if (l <= 0) l = m[k] == 1 ? 1 : fft_friendly(2 * m[k] - 1);
      if (m[k] > 1 && l < 2 * m[k] - 1) fail(FPBEM_CU_EDIM, "create: fft size < 2M-1");
      if (m[k] == 1 && l != 1) fail(FPBEM_CU_EDIM, "create: fft size must be 1 on a single-cell axis");
      op->L[k] = l;
    }
    op->q_total = static_cast<long long>(op->L[0]) * op->L[1] * op->L[2];
    for (int k = 0; k < 3; ++k) twiddles(op, op->L[k], &op->tw[k]);
    build_spectrum(op, d->n_far, d->far_offsets, d->far_blocks, d->far_on_device != 0, d->lambda, &op->lambda);
    if (op->L[2] > 1) {  // work items of the fused z kernel
      const int Lx = op->L[0], Ly = op->L[1];
      std::vector<int2> pairs, singles;
      for (int qy = 0; qy < Ly; ++qy)
        for (int qx = 0; qx < Lx; ++qx) {
          const int c = qy * Lx + qx, cm = ((Ly - qy) % Ly) * Lx + (Lx - qx) % Lx;
          singles.push_back(make_int2(c, -1));
          if (c < cm) pairs.push_back(make_int2(c, cm));
          if (c == cm) pairs.push_back(make_int2(c, -1));
        }
      op->z_items_pair = dalloc<int2>(pairs.size(), "z items");
      op->z_items_single = dalloc<int2>(singles.size(), "z items");
      h2d(op->z_items_pair, pairs.data(), pairs.size() * sizeof(int2), op->stream, "z items");
      h2d(op->z_items_single, singles.data(), singles.size() * sizeof(int2), op->stream, "z items");
      op->n_z_items_pair = static_cast<int>(pairs.size());
      op->n_z_items_single = static_cast<int>(singles.size());
      // parities of the spectrum actually built (or handed over): Λ(-q) = D Λ(q) D, and the
      // reflection Λ(qx, qy, -qz) = Dz Λ(q) Dz
      unsigned long long* dv = dalloc<unsigned long long>(4, "parity check");
      std::unique_ptr<unsigned long long, decltype(&cudaFree)> keep_dv(dv, &cudaFree);
      check(cudaMemsetAsync(dv, 0, 4 * sizeof(unsigned long long), op->stream), "parity check");
      check(launch_lambda_parity(op->lambda, op->L, op->b, false, dv, op->stream), "parity check");
      check(launch_lambda_parity(op->lambda, op->L, op->b, true, dv + 2, op->stream), "parity check");
      unsigned long long hv[4];
      check(cudaMemcpyAsync(hv, dv, sizeof(hv), cudaMemcpyDeviceToHost, op->stream), "parity check");
      check(cudaStreamSynchronize(op->stream), "parity check");
      double dev, amax, devz;
      std::memcpy(&dev, &hv[0], sizeof(double));
      std::memcpy(&amax, &hv[1], sizeof(double));
      std::memcpy(&devz, &hv[2], sizeof(double));
      op->lam_paired = amax > 0.0 && dev <= 1e-12 * amax;
      op->lam_zsym = op->lam_paired && devz <= 1e-12 * amax;
    }
    if (op->mirrored_level >= 0) {
      // spectrum of K_hat P: Toeplitz offsets o = idx with o[a] = idx[a] - (M_a - 1)
      // (hankel_spectrum, src/structured.cpp:185-198)
      const int a = op->mirrored_level;
      std::vector<int> offs(d->far_hat_indices, d->far_hat_indices + 3 * d->n_far_hat);
      for (int s = 0; s < d->n_far_hat; ++s) offs[3 * s + a] -= m[a] - 1;
      build_spectrum(op, d->n_far_hat, offs.data(), d->far_hat_blocks, d->far_on_device != 0, d->lambda_hat,
                     &op->lambda_hat);
    }

    if (d->n_near > 0 && op->n_hat == 0) check_symmetries(op, d);
    choose_near_path(op, d);
    if (op->near_fft) {
      build_near_spectrum(op, d->n_near);
      const size_t f = static_cast<size_t>(op->max_rhs) * op->qn * op->n;
      op->nfa = dalloc<c64>(f, "near x spectrum");
      op->nfb = dalloc<c64>(f, "near y spectrum");
      op->mode_lo = 0;
      op->mode_hi = op->n_items;
    }

    // apply buffers
    const long long E = static_cast<long long>(op->max_rhs) * op->b;
    op->W = dalloc<c64>(op->near_fft ? 1 : static_cast<size_t>(op->n_pairs) * op->max_rhs * op->n, "near workspace");
    op->mom = dalloc<c64>(static_cast<size_t>(op->n_cells) * E, "moments");
    op->loc = dalloc<c64>(static_cast<size_t>(op->n_cells) * E, "locals");
    op->fa = dalloc<c64>(static_cast<size_t>(op->q_total) * E, "m2l field");
    op->fb = dalloc<c64>(static_cast<size_t>(op->q_total) * E, "m2l image");
    if (op->mirrored_level >= 0) {
      op->mom_perm = dalloc<c64>(static_cast<size_t>(op->n_cells) * E, "permuted moments");
      op->loc_hat = dalloc<c64>(static_cast<size_t>(op->n_cells) * E, "image locals");
    }
    for (auto& e : op->ev) check(cudaEventCreate(&e), "event");
    check(cudaStreamSynchronize(op->stream), "create sync");
    *out = guard_op.release();
  });
}

void fpbem_cu_fmm_destroy(fpbem_cu_op* op) {
  if (!op) return;
  cudaSetDevice(op->device);
  if (op->stream) cudaStreamSynchronize(op->stream);
  slab_destroy(op);
  for (void* p : {static_cast<void*>(op->S), static_cast<void*>(op->pair_src), static_cast<void*>(op->tgt_ptr),
                  static_cast<void*>(op->tgt_pairs), static_cast<void*>(op->jobs), static_cast<void*>(op->u0),
                  static_cast<void*>(op->v0), static_cast<void*>(op->v0t), static_cast<void*>(op->z_items_pair),
                  static_cast<void*>(op->z_items_single), static_cast<void*>(op->lambda), static_cast<void*>(op->lambda_hat),
                  static_cast<void*>(op->mom_perm), static_cast<void*>(op->loc_hat), static_cast<void*>(op->tw[0]),
                  static_cast<void*>(op->tw[1]), static_cast<void*>(op->tw[2]), static_cast<void*>(op->W),
                  static_cast<void*>(op->mom), static_cast<void*>(op->loc), static_cast<void*>(op->fa),
                  static_cast<void*>(op->fb), static_cast<void*>(op->xin), static_cast<void*>(op->yout),
                  static_cast<void*>(op->basis), static_cast<void*>(op->gx), static_cast<void*>(op->gb),
                  static_cast<void*>(op->gt), static_cast<void*>(op->gsol), static_cast<void*>(op->scal_c), static_cast<void*>(op->rs.partial_d),
                  static_cast<void*>(op->rs.partial_c), static_cast<void*>(op->rs.counter),
                  static_cast<void*>(op->shat), static_cast<void*>(op->twn[0]), static_cast<void*>(op->twn[1]),
                  static_cast<void*>(op->twn[2]), static_cast<void*>(op->nfa), static_cast<void*>(op->nfb),
                  static_cast<void*>(op->mjobs), static_cast<void*>(op->perm),
                  static_cast<void*>(op->items), op->bws, op->dws})
    if (p) cudaFree(p);
  if (op->pinned) cudaFreeHost(op->pinned);
  for (auto& e : op->ev)
    if (e) cudaEventDestroy(e);
  for (auto* evs : {op->pev_in, op->pev_out})
    for (int i = 0; i < 8; ++i)
      if (evs[i]) cudaEventDestroy(evs[i]);
  for (cudaStream_t cs : {op->cin, op->cout})
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
  if (op->aux) {
    cudaStreamSynchronize(op->aux);
    cudaStreamDestroy(op->aux);
  }
  if (op->fork) cudaEventDestroy(op->fork);
  if (op->join) cudaEventDestroy(op->join);
  if (op->own_stream && op->stream) cudaStreamDestroy(op->stream);
  delete op;
}

int fpbem_cu_fmm_apply(fpbem_cu_op* op, const fpbem_c64* x, fpbem_c64* y, int nrhs, int ptr_kind) {
  return guard([&] {
    if (!op || !x || !y) fail(FPBEM_CU_EINVAL, "apply: null argument");
    if (nrhs < 1) fail(FPBEM_CU_EDIM, "fmm matvec: dimension mismatch");
    check(cudaSetDevice(op->device), "set device");
    if (ptr_kind == FPBEM_CU_PTR_DEVICE) {
      apply_device(op, reinterpret_cast<const c64*>(x), reinterpret_cast<c64*>(y), nrhs);
      check(cudaGetLastError(), "apply");
      return;
    }
    if (ptr_kind != FPBEM_CU_PTR_HOST) fail(FPBEM_CU_EINVAL, "apply: bad ptr_kind");
    const size_t bytes = static_cast<size_t>(op->N) * op->max_rhs * sizeof(c64);
    if (!op->xin) {
      op->xin = dalloc<c64>(static_cast<size_t>(op->N) * op->max_rhs, "x staging");
      op->yout = dalloc<c64>(static_cast<size_t>(op->N) * op->max_rhs, "y staging");
    }
    if (nrhs == 1 && apply_host_pipelined(op, reinterpret_cast<const c64*>(x), reinterpret_cast<c64*>(y))) return;
    for (int r0 = 0; r0 < nrhs; r0 += op->max_rhs) {
      const int c = std::min(op->max_rhs, nrhs - r0);
      const size_t cb = static_cast<size_t>(op->N) * c * sizeof(c64);
      (void)bytes;
      check(cudaMemcpyAsync(op->xin, x + static_cast<size_t>(r0) * op->N, cb, cudaMemcpyHostToDevice, op->stream),
            "x upload");
      apply_chunk(op, op->xin, op->yout, c, true);
      check(cudaMemcpyAsync(y + static_cast<size_t>(r0) * op->N, op->yout, cb, cudaMemcpyDeviceToHost, op->stream),
            "y download");
    }
    check(cudaStreamSynchronize(op->stream), "apply sync");
  });
}

int fpbem_cu_fmm_bytes(const fpbem_cu_op* op, size_t* bytes) {
  if (!op || !bytes) {
    g_err = "bytes: null argument";
    return FPBEM_CU_EINVAL;
  }
  const size_t c = sizeof(c64);
  // S (+ S_hat, counted in n_near slots) + spectrum (+ image spectrum) + U0 + V0 (src/fmm.cpp:273-279)
  const size_t spectra = op->lambda_hat ? 2 : 1;
  *bytes = c * (static_cast<size_t>(op->n_near) * op->n * op->n +
                spectra * static_cast<size_t>(op->q_total) * op->b * op->b + 2 * static_cast<size_t>(op->n) * op->b);
  return FPBEM_CU_OK;
}

int fpbem_cu_fmm_near_path(const fpbem_cu_op* op, int* path, int* sizes, size_t* spectrum_bytes, int* modes_per_block,
                           int* symmetry_mask, double* symmetry_dev) {
  if (!op || !path || !sizes || !spectrum_bytes || !modes_per_block || !symmetry_mask || !symmetry_dev) {
    g_err = "near_path: null argument";
    return FPBEM_CU_EINVAL;
  }
  *path = op->near_fft ? FPBEM_CU_NEAR_LATTICE : FPBEM_CU_NEAR_DIRECT;
  for (int k = 0; k < 3; ++k) sizes[k] = op->near_fft ? op->Ln[k] : 1;
  *spectrum_bytes = op->near_fft ? static_cast<size_t>(op->n_items) * op->n * op->n * sizeof(c64) : 0;
  *modes_per_block = op->near_fft ? op->near_nimg : 1;
  *symmetry_mask = op->near_sym_mask;
  *symmetry_dev = op->near_sym_dev;
  return FPBEM_CU_OK;
}

int fpbem_cu_spectrum(const fpbem_cu_op* op, int* sizes, fpbem_c64* lambda_out) {
  return guard([&] {
    if (!op || !sizes) fail(FPBEM_CU_EINVAL, "spectrum: null argument");
    for (int k = 0; k < 3; ++k) sizes[k] = op->L[k];
    if (lambda_out) {
      check(cudaSetDevice(op->device), "set device");
      check(cudaStreamSynchronize(op->stream), "sync");
      check(cudaMemcpyAsync(lambda_out, op->lambda, static_cast<size_t>(op->q_total) * op->b * op->b * sizeof(c64),
                            cudaMemcpyDeviceToHost, op->stream),
            "spectrum download");
      check(cudaStreamSynchronize(op->stream), "spectrum download");
    }
  });
}

int fpbem_cu_far_info(const fpbem_cu_op* op, int* sizes, int* paired) {
  if (!op || !sizes || !paired) return FPBEM_CU_EINVAL;
  for (int k = 0; k < 3; ++k) sizes[k] = op->L[k];
  *paired = op->lam_zsym ? 2 : (op->lam_paired ? 1 : 0);  // 2: also the z-reflection parity
  return FPBEM_CU_OK;
}

int fpbem_cu_set_stream(fpbem_cu_op* op, void* stream) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_stream: null op");
    check(cudaSetDevice(op->device), "set device");
    check(cudaStreamSynchronize(op->stream), "sync");
    if (op->own_stream) cudaStreamDestroy(op->stream);
    if (stream) {
      op->stream = static_cast<cudaStream_t>(stream);
      op->own_stream = false;
    } else {
      check(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking), "stream");
      op->own_stream = true;
    }
  });
}

int fpbem_cu_get_stream(const fpbem_cu_op* op, void** stream) {
  if (!op || !stream) return FPBEM_CU_EINVAL;
  *stream = static_cast<void*>(op->stream);
  return FPBEM_CU_OK;
}

int fpbem_cu_enable_stage_timing(fpbem_cu_op* op, int enable) {
  if (!op) return FPBEM_CU_EINVAL;
  op->timing = enable != 0;
  op->serial_timing = enable == 2;
  return FPBEM_CU_OK;
}

int fpbem_cu_stage_times(fpbem_cu_op* op, double* ms_out) {
  if (!op || !ms_out) return FPBEM_CU_EINVAL;
  for (int i = 0; i < 5; ++i) ms_out[i] = op->stage_ms[i];
  ms_out[5] = static_cast<double>(op->applies);
  ms_out[6] = op->stage_ms[5];
  for (double& v : op->stage_ms) v = 0.0;
  op->applies = 0;
  return FPBEM_CU_OK;
}

long long fpbem_cu_kernel_launches(const fpbem_cu_op* op) { return op ? op->launches : 0; }

}  // extern "C"
