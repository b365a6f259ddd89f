// C-ABI implementation (include/fpbem_cuda.h): operator handle, the fused
// FMM apply (near field + P2M + lattice-DFT M2L + L2P) and the device-
// resident restarted GMRES.
//
//   FmmOperators::matvec  src/fmm.cpp:246-271  -> apply_chunk()
//   solver::gmres         src/solver.cpp:21-123 -> gmres_one()
//   CirculantSpectrum ctor src/structured.cpp:63-108 -> build_spectrum()
#include <dlfcn.h>

#include <algorithm>
#include <functional>
#include <memory>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fpbem_cuda.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace fpbem_cu;

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? FPBEM_CU_ENOMEM : FPBEM_CU_ECUDA;
    fail(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename T>
T* dalloc(size_t count, const char* what) {
  void* p = nullptr;
  if (count == 0) count = 1;
  check(cudaMalloc(&p, count * sizeof(T)), what);
  return static_cast<T*>(p);
}

// host->device copy ordered on `stream` (never the legacy default stream,
// which does not synchronise with the handle's non-blocking stream)
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t stream, const char* what) {
  if (bytes == 0) return;
  check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream), what);
  check(cudaStreamSynchronize(stream), what);
}

int fft_friendly(int n) {  // smallest 7-smooth length >= n (src/structured.cpp:26-33)
  for (int m = n;; ++m) {
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}

}  // namespace

// --------------------------------------------------------------------------
// NCCL, loaded at runtime so the library has no hard NCCL dependency.

struct fpbem_cu_comm {
  void* lib = nullptr;
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0, device = 0;
  int (*allreduce)(const void*, void*, size_t, int, int, void*, void*) = nullptr;
  int (*destroy)(void*) = nullptr;
};

namespace {
void* load_nccl() {
  static void* lib = nullptr;
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  return lib;
}
}  // namespace

struct fpbem_cu_op {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t aux = nullptr;  // P2M + M2L run here, concurrently with the near-field GEMM
  cudaEvent_t fork = nullptr, join = nullptr;
  int counts[3] = {1, 1, 1};
  int n = 0, b = 0, n_cells = 0;
  long long N = 0;
  int max_rhs = 1;

  // near field
  int n_near = 0;
  std::vector<int> near_offsets;
  c64* S = nullptr;
  int n_pairs = 0;
  std::vector<int> pair_start;  // per offset slot, n_near + 1
  int* pair_src = nullptr;
  int* tgt_ptr = nullptr;
  int* tgt_pairs = nullptr;
  int4* jobs = nullptr;  // near-field GEMM jobs followed by the P2M jobs
  int jobs_nrhs = -1, n_jobs = 0, jobs_cap = 0;
  double far_pairs = 0.0;  // rank 0's deficit under the pair partition (calibrate_far_pairs)
  long long pair_lo = 0, pair_hi = 0;  // global pair range this rank computes (all without a partition)
  std::vector<int> pair_tgt;    // host copy: target cell of every pair
  int rank = 0, nranks = 1;     // near-field offset partition

  // expansions and spectrum
  c64* u0 = nullptr;
  c64* v0 = nullptr;
  c64* v0t = nullptr;  // V0^T (b rows of n), for the P2M kernel
  int L[3] = {1, 1, 1};
  long long q_total = 1;
  c64* lambda = nullptr;
  c64* tw[3] = {nullptr, nullptr, nullptr};
  // half-space image pair: S_hat blocks live in S after the n_near Toeplitz
  // slots (Hankel-indexed pairs); lambda_hat is the spectrum of K_hat P
  int mirrored_level = -1;
  int n_hat = 0;
  c64* lambda_hat = nullptr;
  c64* mom_perm = nullptr;
  c64* loc_hat = nullptr;

  // per-apply buffers (sized for max_rhs)
  c64* W = nullptr;
  c64* mom = nullptr;
  c64* loc = nullptr;
  c64* fa = nullptr;
  c64* fb = nullptr;
  c64* xin = nullptr;   // host-pointer staging
  c64* yout = nullptr;

  // GMRES
  c64* basis = nullptr;
  int basis_cols = 0;
  c64* gx = nullptr;
  c64* gb = nullptr;
  c64* gt = nullptr;
  c64* gsol = nullptr;
  c64* scal_c = nullptr;    // h[0..m], hc[0..m], y[0..m]
  double* scal_d = nullptr;  // [0] pre^2 [1] post^2 [2] misc [3] rnorm^2
  int* flag = nullptr;
  int scal_cap = 0;
  RedScratch rs{};
  void* pinned = nullptr;
  size_t pinned_bytes = 0;

  // timing
  bool timing = false;
  cudaEvent_t ev[8] = {};
  double stage_ms[5] = {0, 0, 0, 0, 0};
  long long applies = 0;
  long long launches = 0;

  fpbem_cu_comm* comm = nullptr;
};

namespace {

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
  pair_range(op->n_pairs, nranks, rank, far_pairs, op->pair_lo, op->pair_hi);
  op->far_pairs = far_pairs;
  op->rank = rank;
  op->nranks = nranks;
  op->jobs_nrhs = -1;  // rebuild the GEMM job list
  build_target_csr(op);
}

// Column tiles of one offset (or of the P2M columns): as many 64-wide tiles as
// fit, then the remainder as one 64- (49..63), 32+16- (33..48), 32- (17..32)
// or 16-wide (1..16) tile. job.z = column count | width class << 8.
void tile_columns(std::vector<int4>& jobs, int s, int cols, int pair_base, bool narrow) {
  int c0 = 0;
  auto push = [&](int w, int cls) {
    jobs.push_back(make_int4(s, c0, w | (cls << 8), pair_base));
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
void m2l_apply(fpbem_cu_op* op, int nrhs, cudaStream_t s, const c64* moments, const c64* lambda, c64* locals) {
  const long long E = static_cast<long long>(nrhs) * op->b;
  const long long Mx = op->counts[0], My = op->counts[1], Mz = op->counts[2];
  const long long Lx = op->L[0], Ly = op->L[1], Lz = op->L[2];
  struct Pass {
    int kind;  // 0 dft, 1 mode product, 2 fused z-dft + mode product + inverse z-dft,
               // 3 / 4 forward / inverse x+y plane DFTs (one kernel each)
    long long n_a;
    int n_in, n_out;
    long long inner;
    int L;
    int axis;
    bool back;
  };
  std::vector<Pass> passes;
  long long cx = Mx, cy = My;  // current x / y extents
  // z forward + mode product + z inverse fused into one kernel when the
  // column's fields fit in shared memory (FPBEM_M2L_FUSE=0 disables)
  static const char* fz = std::getenv("FPBEM_M2L_FUSE");
  const bool fuse_z = Lz > 1 && !(fz && std::strcmp(fz, "0") == 0) &&
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
    passes.push_back({1, 0, 0, 0, 0, 0, -1, false});
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
  int last_dft = -1;  // the pass that applies the 1/q scale
  for (int i = 0; i < static_cast<int>(passes.size()); ++i)
    if ((passes[i].kind == 0 && passes[i].back) || passes[i].kind == 2 || passes[i].kind == 4) last_dft = i;
  const c64* cur = moments;
  c64* bufs[2] = {op->fa, op->fb};
  int which = 0;
  for (int i = 0; i < static_cast<int>(passes.size()); ++i) {
    const Pass& p = passes[i];
    const bool final = i + 1 == static_cast<int>(passes.size());
    c64* out = final ? locals : bufs[which];
    if (p.kind == 3 || p.kind == 4) {
      const double scale = (i == last_dft) ? 1.0 / static_cast<double>(op->q_total) : 1.0;
      check(launch_xy_plane(cur, out, op->tw[0], op->tw[1], static_cast<int>(Mx), static_cast<int>(My),
                            static_cast<int>(Lx), static_cast<int>(Ly), static_cast<int>(Mz), static_cast<int>(E),
                            p.kind == 4, scale, s),
            "lattice xy dft");
    } else if (p.kind == 1) {
      check(launch_mode_product(lambda, cur, out, op->q_total, op->b, nrhs, s), "mode product");
    } else if (p.kind == 2) {
      const double scale = (i == last_dft) ? 1.0 / static_cast<double>(op->q_total) : 1.0;
      check(launch_m2l_zfused(cur, out, lambda, op->tw[2], static_cast<int>(Mz), static_cast<int>(Lz), Ly * Lx,
                              static_cast<int>(E), op->b, scale, s),
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

// Far field of one product: P2M (events 2-3) and M2L into op->loc (events 3-4);
// the Hankel image pair adds the K_hat term (src/fmm.cpp:256-263)
void far_field(fpbem_cu_op* op, const c64* x, int nrhs, cudaStream_t a) {
  ev_record(op, 2, a);
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
  if (op->n_pairs == 0) return 0.0;
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
  build_jobs(op, 1);
  float best_near = 1e30f, best_far = 1e30f;
  for (int it = 0; it < 4; ++it) {
    check(cudaEventRecord(e[0], s), "calibration");
    check(launch_block_gemm(op->S, static_cast<long long>(op->n) * op->n, op->n, op->n, x, op->W, op->n, op->pair_src,
                            op->jobs, op->n_jobs, op->n, op->n, op->N, 1, s),
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
  return best_near > 0.0f ? static_cast<double>(best_far) / best_near * static_cast<double>(op->n_pairs) : 0.0;
}

// One FMM product for nrhs <= max_rhs right-hand sides, device pointers.
// Order of the sums follows src/fmm.cpp:253-267: y = S p, then y += U0 L.
// With an offset partition (nranks > 1) this rank computes the product of
// its own near-field offsets; rank 0 also adds the far field (P2M, M2L,
// L2P); with a communicator the partial products are all-reduced.
void apply_chunk(fpbem_cu_op* op, const c64* x, c64* y, int nrhs) {
  cudaStream_t s = op->stream;
  // FPBEM_SERIAL=1 runs P2M + M2L on the main stream (exact per-stage timing)
  static const bool serial = [] {
    const char* v = std::getenv("FPBEM_SERIAL");
    return v && std::strcmp(v, "1") == 0;
  }();
  cudaStream_t a = serial ? op->stream : op->aux;
  const bool far_here = op->rank == 0;
  build_jobs(op, nrhs);
  // fork: P2M + M2L on the aux stream while the near-field GEMM runs on the main one
  check(cudaEventRecord(op->fork, s), "fork");
  check(cudaStreamWaitEvent(a, op->fork, 0), "fork");
  ev_record(op, 0, s);
  check(launch_block_gemm(op->S, static_cast<long long>(op->n) * op->n, op->n, op->n, x, op->W, op->n, op->pair_src,
                          op->jobs, op->n_jobs, op->n, op->n, op->N, nrhs, s),
        "near gemm");
  op->launches += op->n_jobs > 0;
  ev_record(op, 1, s);
  if (far_here) far_field(op, x, nrhs, a);
  check(cudaEventRecord(op->join, a), "join");
  s = op->stream;
  check(cudaStreamWaitEvent(s, op->join, 0), "join");
  ev_record(op, 5, s);
  check(launch_near_reduce_l2p(op->W, op->tgt_ptr, op->tgt_pairs, op->u0, far_here ? op->loc : nullptr, y, op->n,
                               op->b, op->n_cells, op->N, nrhs, false, s),
        "near reduce + l2p");
  op->launches++;
  if (op->comm) {  // sum the ranks' partial products, in place, on the same stream
    const int rc = op->comm->allreduce(y, y, static_cast<size_t>(2) * op->N * nrhs, /*ncclFloat64*/ 8,
                                       /*ncclSum*/ 0, op->comm->comm, s);
    if (rc != 0) fail(FPBEM_CU_ENCCL, "ncclAllReduce failed: " + std::to_string(rc));
  }
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
    op->applies++;
  }
}

void apply_device(fpbem_cu_op* op, const c64* x, c64* y, int nrhs) {
  for (int r0 = 0; r0 < nrhs; r0 += op->max_rhs) {
    const int c = std::min(op->max_rhs, nrhs - r0);
    apply_chunk(op, x + static_cast<long long>(r0) * op->N, y + static_cast<long long>(r0) * op->N, c);
  }
}

void ensure_pinned(fpbem_cu_op* op, size_t bytes) {
  if (op->pinned_bytes >= bytes) return;
  if (op->pinned) cudaFreeHost(op->pinned);
  op->pinned = nullptr;
  check(cudaMallocHost(&op->pinned, bytes), "pinned host buffer");
  op->pinned_bytes = bytes;
}

void ensure_gmres(fpbem_cu_op* op, int restart) {
  const int cols = restart + 1;
  if (op->basis_cols < cols) {
    if (op->basis) cudaFree(op->basis);
    op->basis = dalloc<c64>(static_cast<size_t>(cols) * op->N, "gmres basis");
    op->basis_cols = cols;
  }
  if (!op->gx) {
    op->gx = dalloc<c64>(op->N, "gmres x");
    op->gb = dalloc<c64>(op->N, "gmres b");
    op->gt = dalloc<c64>(op->N, "gmres tmp");
    op->gsol = dalloc<c64>(op->N, "gmres solution");
    op->rs.partial_d = dalloc<double>(2 * kRedBlocks, "reduction partials");
    op->rs.partial_c = dalloc<c64>(2 * kRedBlocks, "reduction partials");
    op->rs.counter = dalloc<unsigned>(1, "reduction counter");
    check(cudaMemsetAsync(op->rs.counter, 0, sizeof(unsigned), op->stream), "counter init");
    check(cudaStreamSynchronize(op->stream), "counter init");
  }
  if (op->scal_cap < cols) {
    // one contiguous block so a single read-back per Arnoldi step returns the
    // non-finite flag, both norms and the projections: 128-byte header
    // (doubles 0..7, int flag at byte 64), then h[cols], hc[cols], y[cols]
    if (op->scal_c) cudaFree(op->scal_c);
    op->scal_c = dalloc<c64>(8 + 3 * static_cast<size_t>(cols), "gmres scalars");
    op->scal_cap = cols;
    op->scal_d = reinterpret_cast<double*>(op->scal_c);
    op->flag = reinterpret_cast<int*>(op->scal_d + 8);
  }
  ensure_pinned(op, sizeof(c64) * (8 + 3 * static_cast<size_t>(cols)) + 64);
}

struct GmresOut {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
};

// Faithful device-resident restatement of src/solver.cpp:21-123 for one rhs.
using ApplyDev = std::function<void(const c64*, c64*)>;

GmresOut gmres_one(fpbem_cu_op* op, const ApplyDev& apply, const c64* b_dev, c64* x_dev, double tol, int restart,
                   int max_iter) {
  using cd = std::complex<double>;
  cudaStream_t s = op->stream;
  const long long n = op->N;
  GmresOut rep;
  ensure_gmres(op, std::max(1, restart));
  c64* V = op->basis;
  auto col = [&](int j) { return V + static_cast<long long>(j) * n; };
  c64* h = op->scal_c + 8;                    // pass-1 projections (after the 128-byte header)
  c64* hc = h + op->scal_cap;                  // pass-2 corrections
  c64* ydev = hc + op->scal_cap;
  double* sd = op->scal_d;
  char* pin = static_cast<char*>(op->pinned);
  auto fetch = [&](const void* src, size_t bytes) {
    check(cudaMemcpyAsync(pin, src, bytes, cudaMemcpyDeviceToHost, s), "gmres readback");
    check(cudaStreamSynchronize(s), "gmres sync");
  };
  auto fetch_d = [&](int idx) {
    fetch(sd + idx, sizeof(double));
    double v;
    std::memcpy(&v, pin, sizeof(double));
    return v;
  };

  check(cudaMemsetAsync(x_dev, 0, n * sizeof(c64), s), "x0");
  check(cudaMemsetAsync(op->flag, 0, sizeof(int), s), "flag");
  check(launch_sqnorm(b_dev, n, op->rs, sd + 3, nullptr, s), "bnorm");
  op->launches++;
  const double bnorm = std::sqrt(fetch_d(3));
  if (bnorm == 0.0) {
    rep.converged = true;
    return rep;
  }
  const int m = std::max(1, restart);
  std::vector<cd> H(static_cast<size_t>(m + 1) * m, cd(0, 0));
  auto Hm = [&](int i, int j) -> cd& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
  std::vector<cd> g(m + 1);
  std::vector<double> gc(m);
  std::vector<cd> gs(m);
  const c64* r = b_dev;  // r = b_eff on the first cycle
  double rnorm = bnorm;

  while (rep.iterations < max_iter) {
    check(launch_div(r, col(0), n, rnorm, s), "v0");
    op->launches++;
    std::fill(g.begin(), g.end(), cd(0, 0));
    g[0] = rnorm;
    int j = 0;
    for (; j < m && rep.iterations < max_iter; ++j) {
      c64* w = col(j + 1);
      apply(col(j), w);
      const bool fused = mgs_fused_supported(n);
      if (fused) {  // pre-norm + all j+1 MGS steps + post-norm in one cooperative launch
        check(launch_mgs_fused(w, V, n, j, n, h, sd, op->flag, op->rs, true, s), "mgs fused");
        op->launches++;
      } else {
        check(launch_sqnorm(w, n, op->rs, sd + 0, op->flag, s), "pre norm");
        // MGS: h_0 = <v_0,w>; (w -= h_i v_i, h_{i+1} = <v_{i+1}, w>)...; w -= h_j v_j, ||w||^2
        check(launch_dotc(col(0), w, n, op->rs, h + 0, s), "mgs dot");
        for (int i = 0; i < j; ++i)
          check(launch_axpy_dotc(w, col(i), h + i, col(i + 1), n, op->rs, h + i + 1, s), "mgs step");
        check(launch_axpy_sqnorm(w, col(j), h + j, n, op->rs, sd + 1, s), "mgs last");
        op->launches += j + 3;
      }
      // one read-back: flag, ||w||^2 before and after MGS, h_0..h_j
      fetch(sd, 128 + sizeof(c64) * (j + 1));
      {
        int fl;
        std::memcpy(&fl, pin + 64, sizeof(int));
        if (fl) {
          check(cudaMemsetAsync(op->flag, 0, sizeof(int), s), "flag reset");
          fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value");
        }
      }
      double pre2, post2;
      std::memcpy(&pre2, pin, sizeof(double));
      std::memcpy(&post2, pin + sizeof(double), sizeof(double));
      for (int i = 0; i <= j; ++i) {
        c64 v;
        std::memcpy(&v, pin + 128 + i * sizeof(c64), sizeof(c64));
        Hm(i, j) = cd(v.x, v.y);
      }
      double wnorm2 = post2;
      if (std::sqrt(post2) < 0.5 * std::sqrt(pre2)) {  // reorthogonalisation (:63-69)
        if (fused) {
          check(launch_mgs_fused(w, V, n, j, n, hc, sd + 4, op->flag, op->rs, false, s), "reorth fused");
          check(cudaMemcpyAsync(sd + 2, sd + 5, sizeof(double), cudaMemcpyDeviceToDevice, s), "reorth norm");
          op->launches++;
        } else {
          check(launch_dotc(col(0), w, n, op->rs, hc + 0, s), "reorth dot");
          for (int i = 0; i < j; ++i)
            check(launch_axpy_dotc(w, col(i), hc + i, col(i + 1), n, op->rs, hc + i + 1, s), "reorth step");
          check(launch_axpy_sqnorm(w, col(j), hc + j, n, op->rs, sd + 2, s), "reorth last");
          op->launches += j + 2;
        }
        fetch(hc, sizeof(c64) * (j + 1));
        for (int i = 0; i <= j; ++i) {
          c64 v;
          std::memcpy(&v, pin + i * sizeof(c64), sizeof(c64));
          Hm(i, j) += cd(v.x, v.y);
        }
        wnorm2 = fetch_d(2);
      }
      const double hlast = std::sqrt(wnorm2);
      Hm(j + 1, j) = hlast;
      if (hlast > 0.0) {
        check(launch_div(w, w, n, hlast, s), "normalise");
        op->launches++;
      }
      for (int i = 0; i < j; ++i) {  // accumulated rotations (:75-79)
        cd t = gc[i] * Hm(i, j) + gs[i] * Hm(i + 1, j);
        Hm(i + 1, j) = -std::conj(gs[i]) * Hm(i, j) + gc[i] * Hm(i + 1, j);
        Hm(i, j) = t;
      }
      const cd a = Hm(j, j);  // new rotation (:80-94)
      const double bb = std::abs(Hm(j + 1, j));
      const double denom = std::hypot(std::abs(a), bb);
      if (denom == 0.0) {
        gc[j] = 1.0;
        gs[j] = cd(0, 0);
      } else if (std::abs(a) == 0.0) {
        gc[j] = 0.0;
        gs[j] = cd(1, 0);
      } else {
        gc[j] = std::abs(a) / denom;
        gs[j] = (a / std::abs(a)) * std::conj(Hm(j + 1, j)) / denom;
      }
      Hm(j, j) = gc[j] * a + gs[j] * Hm(j + 1, j);
      Hm(j + 1, j) = cd(0, 0);
      const cd gj = g[j];
      g[j] = gc[j] * gj;
      g[j + 1] = -std::conj(gs[j]) * gj;
      ++rep.iterations;
      const double est = std::abs(g[j + 1]) / bnorm;
      rep.history.push_back(est);
      if (est <= tol || hlast == 0.0) {
        ++j;
        break;
      }
    }
    // y = triu(H_jj)^{-1} g ; x += V y (:109-110)
    std::vector<cd> y(j);
    for (int i = j - 1; i >= 0; --i) {
      cd acc = g[i];
      for (int k = i + 1; k < j; ++k) acc -= Hm(i, k) * y[k];
      y[i] = acc / Hm(i, i);
    }
    if (j > 0) {
      std::vector<c64> yh(j);
      for (int i = 0; i < j; ++i) yh[i] = cmk(y[i].real(), y[i].imag());
      std::memcpy(pin, yh.data(), j * sizeof(c64));
      check(cudaMemcpyAsync(ydev, pin, j * sizeof(c64), cudaMemcpyHostToDevice, s), "y upload");
      check(launch_update_x(x_dev, V, n, ydev, j, n, s), "x update");
      op->launches++;
    }
    // true residual r = b - A x (:111-112)
    apply(x_dev, op->gt);
    check(launch_sqnorm(op->gt, n, op->rs, sd + 2, op->flag, s), "residual finite check");
    check(launch_residual(b_dev, op->gt, op->gx, n, op->rs, sd + 3, s), "residual");
    op->launches += 2;
    fetch(sd, 128);  // flag + ||r||^2 in one read-back
    {
      int fl;
      std::memcpy(&fl, pin + 64, sizeof(int));
      if (fl) {
        check(cudaMemsetAsync(op->flag, 0, sizeof(int), s), "flag reset");
        fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value");
      }
      double r2;
      std::memcpy(&r2, pin + 3 * sizeof(double), sizeof(double));
      rnorm = std::sqrt(r2);
    }
    r = op->gx;
    if (rnorm / bnorm <= tol) {
      rep.converged = true;
      break;
    }
  }
  if (!rep.history.empty()) rep.converged = rep.converged || rnorm / bnorm <= tol;
  return rep;
}

// ---------------------------------------------------------------------------
// Lockstep batched GMRES: G right-hand sides advance one Arnoldi step together
// (one batched matvec, batched MGS with per-RHS reductions); every RHS follows
// exactly the control flow of src/solver.cpp:21-123 on its own scalars (host),
// leaves its cycle's inner loop on its own estimate, and leaves the batch when
// converged or out of iterations. Basis layout: column j of RHS r at
// V + (j * G + r) * N, so column j of all RHS is one contiguous batch.
struct BatchOut {
  std::vector<int> iterations;
  std::vector<char> converged;
  std::vector<std::vector<double>> history;
};

BatchOut gmres_batched(fpbem_cu_op* op, const c64* Bd, c64* Xd, int G, double tol, int restart, int max_iter) {
  using cd = std::complex<double>;
  cudaStream_t s = op->stream;
  const long long n = op->N;
  const int m = std::max(1, restart);
  BatchOut out;
  out.iterations.assign(G, 0);
  out.converged.assign(G, 0);
  out.history.assign(G, {});

  std::vector<void*> owned;  // device buffers scoped to the call
  struct Free {
    std::vector<void*>& v;
    ~Free() {
      for (void* p : v) cudaFree(p);
    }
  } free_all{owned};
  auto alloc = [&](size_t bytes, const char* what) {
    void* p = nullptr;
    check(cudaMalloc(&p, bytes), what);
    owned.push_back(p);
    return p;
  };
  const size_t vecb = static_cast<size_t>(n) * sizeof(c64);
  c64* V = static_cast<c64*>(alloc(vecb * G * (m + 1), "batched basis"));
  c64* R = static_cast<c64*>(alloc(vecb * G, "batched residual"));
  c64* T = static_cast<c64*>(alloc(vecb * G, "batched A x"));
  c64* P = static_cast<c64*>(alloc(vecb * G, "batched pack in"));
  c64* Q = static_cast<c64*>(alloc(vecb * G, "batched pack out"));
  // scalars: [flags G int (8 B slots)][pre2 G][post2 G][post2b G][rn2 G][bn2 G][d G]
  //          [h (m+1)G c64][hc (m+1)G][y mG][jr G int][mask G int][idx G int]
  const size_t g8 = 8 * static_cast<size_t>((G + 1) & ~1);  // even count: c64 sections stay 16-byte aligned
  const size_t o_flag = 0, o_pre = g8, o_post = o_pre + g8, o_post2 = o_post + g8, o_rn = o_post2 + g8,
               o_bn = o_rn + g8, o_d = o_bn + g8, o_h = o_d + g8, o_hc = o_h + 2 * g8 * (m + 1),
               o_y = o_hc + 2 * g8 * (m + 1), o_jr = o_y + 2 * g8 * m, o_mask = o_jr + g8 / 2,
               o_idx = o_mask + g8 / 2, total = o_idx + g8 / 2;
  char* sc = static_cast<char*>(alloc(total, "batched scalars"));
  int* d_flag = reinterpret_cast<int*>(sc + o_flag);
  double* d_pre = reinterpret_cast<double*>(sc + o_pre);
  double* d_post = reinterpret_cast<double*>(sc + o_post);
  double* d_post2 = reinterpret_cast<double*>(sc + o_post2);
  double* d_rn = reinterpret_cast<double*>(sc + o_rn);
  double* d_bn = reinterpret_cast<double*>(sc + o_bn);
  double* d_d = reinterpret_cast<double*>(sc + o_d);
  c64* d_h = reinterpret_cast<c64*>(sc + o_h);
  c64* d_hc = reinterpret_cast<c64*>(sc + o_hc);
  c64* d_y = reinterpret_cast<c64*>(sc + o_y);
  int* d_jr = reinterpret_cast<int*>(sc + o_jr);
  int* d_mask = reinterpret_cast<int*>(sc + o_mask);
  int* d_idx = reinterpret_cast<int*>(sc + o_idx);
  BatchScratch bs;
  bs.partial_d = static_cast<double*>(alloc(sizeof(double) * kBatchBlocks * G, "batch partials"));
  bs.partial_c = static_cast<c64*>(alloc(sizeof(c64) * kBatchBlocks * G, "batch partials"));
  bs.counter = static_cast<unsigned*>(alloc(sizeof(unsigned) * G, "batch counters"));
  check(cudaMemsetAsync(bs.counter, 0, sizeof(unsigned) * G, s), "counters");
  check(cudaMemsetAsync(d_flag, 0, g8, s), "flags");
  ensure_pinned(op, total + 64);
  char* pin = static_cast<char*>(op->pinned);
  auto fetch = [&](size_t off, size_t bytes) {
    check(cudaMemcpyAsync(pin + off, sc + off, bytes, cudaMemcpyDeviceToHost, s), "batched readback");
    check(cudaStreamSynchronize(s), "batched sync");
  };
  auto put = [&](size_t off, const void* src, size_t bytes) {
    // pinned staging is reused: the previous upload must have been consumed
    check(cudaStreamSynchronize(s), "batched sync");
    std::memcpy(pin + off, src, bytes);
    check(cudaMemcpyAsync(sc + off, pin + off, bytes, cudaMemcpyHostToDevice, s), "batched upload");
  };
  auto get_d = [&](size_t off, int r) {
    double v;
    std::memcpy(&v, pin + off + 8 * static_cast<size_t>(r), 8);
    return v;
  };
  auto get_c = [&](size_t off, size_t idx) {
    c64 v;
    std::memcpy(&v, pin + off + 16 * idx, 16);
    return cd(v.x, v.y);
  };
  auto set_mask = [&](const std::vector<int>& on) {
    std::vector<int> mk(G, 0);
    for (int r : on) mk[r] = 1;
    put(o_mask, mk.data(), 4 * static_cast<size_t>(G));
  };
  auto flags_of = [&](const std::vector<int>& rs) {
    for (int r : rs) {
      int fl;
      std::memcpy(&fl, pin + o_flag + 4 * static_cast<size_t>(r), 4);
      if (fl) fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value");
    }
  };
  // y = A x for the listed RHS (packed unless the list is 0..G-1)
  auto apply_set = [&](const c64* src_base, c64* dst_base, const std::vector<int>& rs) {
    const int cnt = static_cast<int>(rs.size());
    bool all = cnt == G;
    for (int q = 0; all && q < cnt; ++q) all = rs[q] == q;
    if (all) {
      apply_device(op, src_base, dst_base, G);
      return;
    }
    put(o_idx, rs.data(), 4 * static_cast<size_t>(cnt));
    check(launch_b_pack(src_base, P, d_idx, cnt, n, true, s), "pack");
    apply_device(op, P, Q, cnt);
    check(launch_b_pack(Q, dst_base, d_idx, cnt, n, false, s), "unpack");
    op->launches += 2;
  };

  check(cudaMemsetAsync(Xd, 0, vecb * G, s), "x0");
  std::vector<int> all(G);
  for (int r = 0; r < G; ++r) all[r] = r;
  set_mask(all);
  check(launch_b_sqnorm(Bd, n, n, G, d_mask, bs, d_bn, nullptr, s), "bnorm");
  fetch(o_bn, g8);
  std::vector<double> bnorm(G), rnorm(G);
  std::vector<char> done(G, 0);
  for (int r = 0; r < G; ++r) {
    bnorm[r] = std::sqrt(get_d(o_bn, r));
    rnorm[r] = bnorm[r];
    if (bnorm[r] == 0.0) {
      out.converged[r] = 1;
      done[r] = 1;
    }
  }
  const size_t hsz = static_cast<size_t>(m + 1) * m;
  std::vector<std::vector<cd>> H(G, std::vector<cd>(hsz)), g(G, std::vector<cd>(m + 1));
  std::vector<std::vector<double>> gc(G, std::vector<double>(m));
  std::vector<std::vector<cd>> gs(G, std::vector<cd>(m));
  std::vector<int> jr(G, 0);
  std::vector<char> inner(G, 0);
  const c64* rsrc = Bd;

  while (true) {
    std::vector<int> act;
    for (int r = 0; r < G; ++r)
      if (!done[r] && out.iterations[r] < max_iter) act.push_back(r);
    if (act.empty()) break;
    set_mask(act);
    put(o_d, rnorm.data(), g8);
    check(launch_b_div(rsrc, V, n, n, G, d_mask, d_d, s), "v0");  // v0 = r / ||r||
    for (int r : act) {
      std::fill(g[r].begin(), g[r].end(), cd(0, 0));
      g[r][0] = rnorm[r];
      std::fill(H[r].begin(), H[r].end(), cd(0, 0));
      jr[r] = 0;
      inner[r] = 1;
    }
    for (int j = 0; j < m; ++j) {
      std::vector<int> it;
      for (int r : act)
        if (inner[r] && out.iterations[r] < max_iter) it.push_back(r);
      if (it.empty()) break;
      c64* Vj = V + static_cast<long long>(j) * G * n;
      c64* W = V + static_cast<long long>(j + 1) * G * n;
      apply_set(Vj, W, it);
      set_mask(it);
      check(launch_b_sqnorm(W, n, n, G, d_mask, bs, d_pre, d_flag, s), "pre norm");
      check(launch_b_dotc(V, W, n, n, G, d_mask, bs, d_h, s), "mgs dot");
      for (int i = 0; i < j; ++i)
        check(launch_b_axpy_dotc(W, V + static_cast<long long>(i) * G * n, d_h + static_cast<long long>(i) * G,
                                 V + static_cast<long long>(i + 1) * G * n, n, n, G, d_mask, bs,
                                 d_h + static_cast<long long>(i + 1) * G, s),
              "mgs step");
      check(launch_b_axpy_sqnorm(W, Vj, d_h + static_cast<long long>(j) * G, n, n, G, d_mask, bs, d_post, s),
            "mgs last");
      op->launches += j + 3;
      fetch(0, o_h + 16 * static_cast<size_t>(j + 1) * G);  // flags, norms and h_0..h_j of every RHS
      flags_of(it);
      std::vector<int> reo;
      std::vector<double> wn2(G, 0.0);
      for (int r : it) {
        for (int i = 0; i <= j; ++i)
          H[r][static_cast<size_t>(j) * (m + 1) + i] = get_c(o_h, static_cast<size_t>(i) * G + r);
        wn2[r] = get_d(o_post, r);
        if (std::sqrt(wn2[r]) < 0.5 * std::sqrt(get_d(o_pre, r))) reo.push_back(r);  // (:63-69)
      }
      if (!reo.empty()) {
        set_mask(reo);
        check(launch_b_dotc(V, W, n, n, G, d_mask, bs, d_hc, s), "reorth dot");
        for (int i = 0; i < j; ++i)
          check(launch_b_axpy_dotc(W, V + static_cast<long long>(i) * G * n, d_hc + static_cast<long long>(i) * G,
                                   V + static_cast<long long>(i + 1) * G * n, n, n, G, d_mask, bs,
                                   d_hc + static_cast<long long>(i + 1) * G, s),
                "reorth step");
        check(launch_b_axpy_sqnorm(W, Vj, d_hc + static_cast<long long>(j) * G, n, n, G, d_mask, bs, d_post2, s),
              "reorth last");
        op->launches += j + 2;
        fetch(o_post2, g8);
        fetch(o_hc, 16 * static_cast<size_t>(j + 1) * G);
        for (int r : reo) {
          for (int i = 0; i <= j; ++i)
            H[r][static_cast<size_t>(j) * (m + 1) + i] += get_c(o_hc, static_cast<size_t>(i) * G + r);
          wn2[r] = get_d(o_post2, r);
        }
      }
      std::vector<double> hl(G, 1.0);
      std::vector<int> norm_set;
      for (int r : it) {
        hl[r] = std::sqrt(wn2[r]);
        if (hl[r] > 0.0) norm_set.push_back(r);
      }
      if (!norm_set.empty()) {
        set_mask(norm_set);
        put(o_d, hl.data(), g8);
        check(launch_b_div(W, W, n, n, G, d_mask, d_d, s), "normalise");
        op->launches++;
      }
      for (int r : it) {  // rotations, Givens, estimate (:74-105), per RHS
        auto Hm = [&](int a, int b) -> cd& { return H[r][static_cast<size_t>(b) * (m + 1) + a]; };
        const double hlast = hl[r];
        Hm(j + 1, j) = hlast;
        for (int i = 0; i < j; ++i) {
          cd t = gc[r][i] * Hm(i, j) + gs[r][i] * Hm(i + 1, j);
          Hm(i + 1, j) = -std::conj(gs[r][i]) * Hm(i, j) + gc[r][i] * Hm(i + 1, j);
          Hm(i, j) = t;
        }
        const cd a = Hm(j, j);
        const double bb = std::abs(Hm(j + 1, j));
        const double denom = std::hypot(std::abs(a), bb);
        if (denom == 0.0) {
          gc[r][j] = 1.0;
          gs[r][j] = cd(0, 0);
        } else if (std::abs(a) == 0.0) {
          gc[r][j] = 0.0;
          gs[r][j] = cd(1, 0);
        } else {
          gc[r][j] = std::abs(a) / denom;
          gs[r][j] = (a / std::abs(a)) * std::conj(Hm(j + 1, j)) / denom;
        }
        Hm(j, j) = gc[r][j] * a + gs[r][j] * Hm(j + 1, j);
        Hm(j + 1, j) = cd(0, 0);
        const cd gj = g[r][j];
        g[r][j] = gc[r][j] * gj;
        g[r][j + 1] = -std::conj(gs[r][j]) * gj;
        ++out.iterations[r];
        const double est = std::abs(g[r][j + 1]) / bnorm[r];
        out.history[r].push_back(est);
        jr[r] = j + 1;
        if (est <= tol || hlast == 0.0) inner[r] = 0;
      }
    }
    // x_r += V_r y_r for every RHS of the cycle, then the true residuals (:109-116)
    std::vector<c64> yh(static_cast<size_t>(m) * G, cmk(0.0, 0.0));
    for (int r : act) {
      auto Hm = [&](int a, int b) -> cd& { return H[r][static_cast<size_t>(b) * (m + 1) + a]; };
      const int jj = jr[r];
      std::vector<cd> y(jj);
      for (int i = jj - 1; i >= 0; --i) {
        cd acc = g[r][i];
        for (int k = i + 1; k < jj; ++k) acc -= Hm(i, k) * y[k];
        y[i] = acc / Hm(i, i);
      }
      for (int i = 0; i < jj; ++i) yh[static_cast<size_t>(r) * m + i] = cmk(y[i].real(), y[i].imag());
    }
    put(o_y, yh.data(), 16 * yh.size());
    put(o_jr, jr.data(), 4 * static_cast<size_t>(G));
    set_mask(act);
    check(launch_b_update_x(Xd, V, G, n, d_y, m, d_jr, n, d_mask, s), "x update");
    apply_set(Xd, T, act);
    set_mask(act);
    check(launch_b_residual(Bd, T, R, n, n, G, d_mask, bs, d_rn, d_flag, s), "residual");
    op->launches += 2;
    fetch(0, o_pre);
    flags_of(act);
    fetch(o_rn, g8);
    for (int r : act) {
      rnorm[r] = std::sqrt(get_d(o_rn, r));
      if (rnorm[r] / bnorm[r] <= tol) {
        out.converged[r] = 1;
        done[r] = 1;
      }
    }
    rsrc = R;
  }
  for (int r = 0; r < G; ++r)
    if (!out.history[r].empty()) out.converged[r] = out.converged[r] || rnorm[r] / bnorm[r] <= tol;
  check(cudaStreamSynchronize(s), "batched gmres");
  return out;
}

}  // namespace

namespace {
int guard(const std::function<void()>& fn) {
  try {
    fn();
    return FPBEM_CU_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FPBEM_CU_EINVAL;
  }
}
}  // namespace

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
    if (op->mirrored_level >= 0) {
      // spectrum of K_hat P: Toeplitz offsets o = idx with o[a] = idx[a] - (M_a - 1)
      // (hankel_spectrum, src/structured.cpp:185-198)
      const int a = op->mirrored_level;
      std::vector<int> offs(d->far_hat_indices, d->far_hat_indices + 3 * d->n_far_hat);
      for (int s = 0; s < d->n_far_hat; ++s) offs[3 * s + a] -= m[a] - 1;
      build_spectrum(op, d->n_far_hat, offs.data(), d->far_hat_blocks, d->far_on_device != 0, d->lambda_hat,
                     &op->lambda_hat);
    }

    // apply buffers
    const long long E = static_cast<long long>(op->max_rhs) * op->b;
    op->W = dalloc<c64>(static_cast<size_t>(op->n_pairs) * op->max_rhs * op->n, "near workspace");
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
  for (void* p : {static_cast<void*>(op->S), static_cast<void*>(op->pair_src), static_cast<void*>(op->tgt_ptr),
                  static_cast<void*>(op->tgt_pairs), static_cast<void*>(op->jobs), static_cast<void*>(op->u0),
                  static_cast<void*>(op->v0), static_cast<void*>(op->v0t), static_cast<void*>(op->lambda), static_cast<void*>(op->lambda_hat),
                  static_cast<void*>(op->mom_perm), static_cast<void*>(op->loc_hat), static_cast<void*>(op->tw[0]),
                  static_cast<void*>(op->tw[1]), static_cast<void*>(op->tw[2]), static_cast<void*>(op->W),
                  static_cast<void*>(op->mom), static_cast<void*>(op->loc), static_cast<void*>(op->fa),
                  static_cast<void*>(op->fb), static_cast<void*>(op->xin), static_cast<void*>(op->yout),
                  static_cast<void*>(op->basis), static_cast<void*>(op->gx), static_cast<void*>(op->gb),
                  static_cast<void*>(op->gt), static_cast<void*>(op->gsol), static_cast<void*>(op->scal_c), static_cast<void*>(op->rs.partial_d),
                  static_cast<void*>(op->rs.partial_c), static_cast<void*>(op->rs.counter)})
    if (p) cudaFree(p);
  if (op->pinned) cudaFreeHost(op->pinned);
  for (auto& e : op->ev)
    if (e) cudaEventDestroy(e);
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
    for (int r0 = 0; r0 < nrhs; r0 += op->max_rhs) {
      const int c = std::min(op->max_rhs, nrhs - r0);
      const size_t cb = static_cast<size_t>(op->N) * c * sizeof(c64);
      (void)bytes;
      check(cudaMemcpyAsync(op->xin, x + static_cast<size_t>(r0) * op->N, cb, cudaMemcpyHostToDevice, op->stream),
            "x upload");
      apply_chunk(op, op->xin, op->yout, c);
      check(cudaMemcpyAsync(y + static_cast<size_t>(r0) * op->N, op->yout, cb, cudaMemcpyDeviceToHost, op->stream),
            "y download");
    }
    check(cudaStreamSynchronize(op->stream), "apply sync");
  });
}

int fpbem_cu_gmres(fpbem_cu_op* op, const fpbem_c64* b, fpbem_c64* x, int nrhs, double tol, int restart,
                   int max_iter, int ptr_kind, int* iterations, int* converged, double* history, int history_cap,
                   int* history_len) {
  return guard([&] {
    if (!op || !b || !x || !iterations || !converged) fail(FPBEM_CU_EINVAL, "gmres: null argument");
    if (nrhs < 1) fail(FPBEM_CU_EDIM, "gmres: nrhs >= 1 required");
    check(cudaSetDevice(op->device), "set device");
    ensure_gmres(op, std::max(1, restart));
    const char* lock = std::getenv("FPBEM_GMRES_BATCHED");
    const bool batched = nrhs > 1 && !(lock && std::strcmp(lock, "0") == 0);
    if (batched) {  // lockstep batch over all right-hand sides
      const size_t bytes = static_cast<size_t>(op->N) * nrhs * sizeof(c64);
      const c64* bd;
      c64* xd;
      c64* tmp_b = nullptr;
      c64* tmp_x = nullptr;
      if (ptr_kind == FPBEM_CU_PTR_DEVICE) {
        bd = reinterpret_cast<const c64*>(b);
        xd = reinterpret_cast<c64*>(x);
      } else {
        tmp_b = dalloc<c64>(static_cast<size_t>(op->N) * nrhs, "batched b");
        tmp_x = dalloc<c64>(static_cast<size_t>(op->N) * nrhs, "batched x");
        h2d(tmp_b, b, bytes, op->stream, "b upload");
        bd = tmp_b;
        xd = tmp_x;
      }
      std::unique_ptr<c64, decltype(&cudaFree)> kb(tmp_b, &cudaFree), kx(tmp_x, &cudaFree);
      BatchOut o = gmres_batched(op, bd, xd, nrhs, tol, restart, max_iter);
      for (int r = 0; r < nrhs; ++r) {
        iterations[r] = o.iterations[r];
        converged[r] = o.converged[r];
        if (history_len) history_len[r] = static_cast<int>(o.history[r].size());
        if (history)
          for (int i = 0; i < std::min(history_cap, static_cast<int>(o.history[r].size())); ++i)
            history[static_cast<size_t>(r) * history_cap + i] = o.history[r][i];
      }
      if (ptr_kind != FPBEM_CU_PTR_DEVICE)
        check(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, op->stream), "x download");
      check(cudaStreamSynchronize(op->stream), "gmres sync");
      return;
    }
    for (int r = 0; r < nrhs; ++r) {
      const size_t off = static_cast<size_t>(r) * op->N;
      const c64* bd;
      c64* xd;
      if (ptr_kind == FPBEM_CU_PTR_DEVICE) {
        bd = reinterpret_cast<const c64*>(b) + off;
        xd = reinterpret_cast<c64*>(x) + off;
      } else {
        check(cudaMemcpyAsync(op->gb, b + off, op->N * sizeof(c64), cudaMemcpyHostToDevice, op->stream), "b upload");
        bd = op->gb;
        xd = op->gsol;
      }
      GmresOut o = gmres_one(
          op, [op](const c64* in, c64* out) { apply_device(op, in, out, 1); }, bd, xd, tol, restart, max_iter);
      iterations[r] = o.iterations;
      converged[r] = o.converged ? 1 : 0;
      if (history_len) history_len[r] = static_cast<int>(o.history.size());
      if (history)
        for (int i = 0; i < std::min(history_cap, static_cast<int>(o.history.size())); ++i)
          history[static_cast<size_t>(r) * history_cap + i] = o.history[i];
      if (ptr_kind != FPBEM_CU_PTR_DEVICE) {
        check(cudaMemcpyAsync(x + off, xd, op->N * sizeof(c64), cudaMemcpyDeviceToHost, op->stream), "x download");
        check(cudaStreamSynchronize(op->stream), "gmres sync");
      }
    }
    check(cudaStreamSynchronize(op->stream), "gmres sync");
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

int fpbem_cu_enable_stage_timing(fpbem_cu_op* op, int enable) {
  if (!op) return FPBEM_CU_EINVAL;
  op->timing = enable != 0;
  return FPBEM_CU_OK;
}

int fpbem_cu_stage_times(fpbem_cu_op* op, double* ms_out) {
  if (!op || !ms_out) return FPBEM_CU_EINVAL;
  for (int i = 0; i < 5; ++i) ms_out[i] = op->stage_ms[i];
  ms_out[5] = static_cast<double>(op->applies);
  for (double& v : op->stage_ms) v = 0.0;
  op->applies = 0;
  return FPBEM_CU_OK;
}

long long fpbem_cu_kernel_launches(const fpbem_cu_op* op) { return op ? op->launches : 0; }

int fpbem_cu_gmres_fn(int device, long long n, fpbem_cu_apply_fn apply, void* actx, fpbem_cu_apply_fn precond,
                      void* pctx, const fpbem_c64* b, fpbem_c64* x, double tol, int restart, int max_iter,
                      int ptr_kind, int* iterations, int* converged, double* history, int history_cap,
                      int* history_len) {
  fpbem_cu_op* op = nullptr;
  int rc = guard([&] {
    if (!apply || !b || !x || !iterations || !converged || n < 1) fail(FPBEM_CU_EINVAL, "gmres_fn: bad argument");
    check(cudaSetDevice(device), "set device");
    op = new fpbem_cu_op();
    op->device = device;
    op->N = n;
    check(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking), "stream");
    op->own_stream = true;
    ensure_gmres(op, std::max(1, restart));
    c64* pre_tmp = precond ? dalloc<c64>(n, "precond scratch") : nullptr;
    std::unique_ptr<c64, decltype(&cudaFree)> keep(pre_tmp, &cudaFree);
    auto call = [&](fpbem_cu_apply_fn fn, void* ctx, const c64* in, c64* out) {
      if (fn(ctx, reinterpret_cast<const fpbem_c64*>(in), reinterpret_cast<fpbem_c64*>(out), op->stream) != 0)
        fail(FPBEM_CU_EINVAL, "gmres: operator callback failed");
    };
    ApplyDev eff = [&](const c64* in, c64* out) {
      if (precond) {
        call(apply, actx, in, pre_tmp);
        check(launch_sqnorm(pre_tmp, n, op->rs, op->scal_d + 4, op->flag, op->stream), "finite check");
        call(precond, pctx, pre_tmp, out);
      } else {
        call(apply, actx, in, out);
      }
    };
    const c64* bd;
    c64* xd;
    if (ptr_kind == FPBEM_CU_PTR_DEVICE) {
      bd = reinterpret_cast<const c64*>(b);
      xd = reinterpret_cast<c64*>(x);
    } else {
      check(cudaMemcpyAsync(op->gb, b, n * sizeof(c64), cudaMemcpyHostToDevice, op->stream), "b upload");
      bd = op->gb;
      xd = op->gsol;
    }
    if (precond) {  // b_eff = M^{-1} b, checked (src/solver.cpp:30)
      call(precond, pctx, bd, op->gt);
      check(cudaMemsetAsync(op->flag, 0, sizeof(int), op->stream), "flag");
      check(launch_sqnorm(op->gt, n, op->rs, op->scal_d + 4, op->flag, op->stream), "finite check");
      int f = 0;
      check(cudaMemcpyAsync(op->pinned, op->flag, sizeof(int), cudaMemcpyDeviceToHost, op->stream), "flag");
      check(cudaStreamSynchronize(op->stream), "sync");
      std::memcpy(&f, op->pinned, sizeof(int));
      if (f) fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value");
      check(cudaMemcpyAsync(op->gb, op->gt, n * sizeof(c64), cudaMemcpyDeviceToDevice, op->stream), "b_eff");
      bd = op->gb;
    }
    GmresOut o = gmres_one(op, eff, bd, xd, tol, restart, max_iter);
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    if (history_len) *history_len = static_cast<int>(o.history.size());
    if (history)
      for (int i = 0; i < std::min(history_cap, static_cast<int>(o.history.size())); ++i) history[i] = o.history[i];
    if (ptr_kind != FPBEM_CU_PTR_DEVICE)
      check(cudaMemcpyAsync(x, xd, n * sizeof(c64), cudaMemcpyDeviceToHost, op->stream), "x download");
    check(cudaStreamSynchronize(op->stream), "gmres sync");
  });
  fpbem_cu_fmm_destroy(op);
  return rc;
}

namespace {

// Gauss-Legendre nodes/weights by Newton on P_n (the host rule, kernels.cpp:162-194)
void gauss_rule(int n, double* x, double* w) {
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(3.14159265358979323846 * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 0; j < n; ++j) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j + 1.0) * z * p1 - j * p2) / (j + 1);
      }
      dp = n * (z * p0 - p1) / (z * z - 1.0);
      const double dz = p0 / dp;
      z -= dz;
      if (std::abs(dz) < 1e-15) break;
    }
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

struct CellDev {
  double* corners = nullptr;
  int* nv = nullptr;
  double* cen = nullptr;
  double* nrm = nullptr;
  double* diam = nullptr;
  c64* beta = nullptr;
  ~CellDev() {
    for (void* p : {static_cast<void*>(corners), static_cast<void*>(nv), static_cast<void*>(cen),
                    static_cast<void*>(nrm), static_cast<void*>(diam), static_cast<void*>(beta)})
      if (p) cudaFree(p);
  }
};

void upload_cell(const fpbem_cu_cell* c, CellDev& d, cudaStream_t s) {
  if (!c || c->n < 1 || !c->corners || !c->nv || !c->centroid || !c->normal || !c->diameter)
    fail(FPBEM_CU_EINVAL, "assemble: bad cell");
  const size_t n = static_cast<size_t>(c->n);
  d.corners = dalloc<double>(12 * n, "cell corners");
  d.nv = dalloc<int>(n, "cell nv");
  d.cen = dalloc<double>(3 * n, "cell centroids");
  d.nrm = dalloc<double>(3 * n, "cell normals");
  d.diam = dalloc<double>(n, "cell diameters");
  h2d(d.corners, c->corners, 12 * n * sizeof(double), s, "cell upload");
  h2d(d.nv, c->nv, n * sizeof(int), s, "cell upload");
  h2d(d.cen, c->centroid, 3 * n * sizeof(double), s, "cell upload");
  h2d(d.nrm, c->normal, 3 * n * sizeof(double), s, "cell upload");
  h2d(d.diam, c->diameter, n * sizeof(double), s, "cell upload");
  if (c->beta) {
    d.beta = dalloc<c64>(n, "cell beta");
    h2d(d.beta, c->beta, n * sizeof(c64), s, "cell upload");
  }
  double x6[6], w6[6], x8[8], w8[8];
  gauss_rule(6, x6, w6);
  gauss_rule(8, x8, w8);
  check(assembly_set_rules(x6, w6, x8, w8), "quadrature rules");
}

// run the slots (two passes: plain, then accumulated images) into out
void run_assembly(const fpbem_cu_cell* cell, double k, fpbem_c64 alpha, int hs_axis, double hs_offset,
                  const std::vector<AssemblySlot>& plain, const std::vector<AssemblySlot>& images, int device,
                  fpbem_c64* out, int ptr_kind) {
  check(cudaSetDevice(device), "set device");
  cudaStream_t s;
  check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> keep_s(s, [](cudaStream_t st) { cudaStreamDestroy(st); });
  CellDev dc;
  upload_cell(cell, dc, s);
  const size_t n = static_cast<size_t>(cell->n);
  const size_t total = plain.size() * n * n;
  c64* dst = reinterpret_cast<c64*>(out);
  c64* tmp = nullptr;
  if (ptr_kind != FPBEM_CU_PTR_DEVICE) dst = tmp = dalloc<c64>(total, "assembly output");
  std::unique_ptr<c64, decltype(&cudaFree)> keep_tmp(tmp, &cudaFree);
  AssemblySlot* ds = dalloc<AssemblySlot>(plain.size() + images.size(), "assembly slots");
  std::unique_ptr<AssemblySlot, decltype(&cudaFree)> keep_ds(ds, &cudaFree);
  h2d(ds, plain.data(), plain.size() * sizeof(AssemblySlot), s, "slots");
  if (!images.empty()) h2d(ds + plain.size(), images.data(), images.size() * sizeof(AssemblySlot), s, "slots");
  const c64 al = cmk(alpha.re, alpha.im);
  // z-chunks of at most 65535 slots per launch (grid.z limit)
  for (size_t s0 = 0; s0 < plain.size(); s0 += 65535) {
    const int cnt = static_cast<int>(std::min<size_t>(65535, plain.size() - s0));
    check(launch_assemble(dc.corners, dc.nv, dc.cen, dc.nrm, dc.diam, dc.beta, cell->n, ds + s0, cnt, k, al, hs_axis,
                          hs_offset, dst + s0 * n * n, false, s),
          "assemble");
  }
  for (size_t s0 = 0; s0 < images.size(); s0 += 65535) {
    const int cnt = static_cast<int>(std::min<size_t>(65535, images.size() - s0));
    check(launch_assemble(dc.corners, dc.nv, dc.cen, dc.nrm, dc.diam, dc.beta, cell->n, ds + plain.size() + s0, cnt, k,
                          al, hs_axis, hs_offset, dst + s0 * n * n, true, s),
          "assemble images");
  }
  if (ptr_kind != FPBEM_CU_PTR_DEVICE)
    check(cudaMemcpyAsync(out, dst, total * sizeof(c64), cudaMemcpyDeviceToHost, s), "assembly download");
  check(cudaStreamSynchronize(s), "assembly");
}

AssemblySlot make_slot(const double t[3], const double src[3], c64 scale, int mirror, int self) {
  AssemblySlot sl;
  for (int d = 0; d < 3; ++d) {
    sl.tshift[d] = t[d];
    sl.sshift[d] = src[d];
  }
  sl.scale = scale;
  sl.mirror = mirror;
  sl.self = self;
  return sl;
}

}  // namespace

int fpbem_cu_assemble_near(const fpbem_cu_cell* cell, double k, fpbem_c64 alpha, const double pitch[3], int n_off,
                           const int* offsets, int fold, int hs_axis, double hs_offset, fpbem_c64 hs_reflection,
                           int device, fpbem_c64* out, int ptr_kind) {
  return guard([&] {
    if (!pitch || (n_off > 0 && (!offsets || !out))) fail(FPBEM_CU_EINVAL, "assemble_near: null argument");
    std::vector<AssemblySlot> plain, images;
    const double zero[3] = {0, 0, 0};
    const bool with_image = fold && (hs_reflection.re != 0.0 || hs_reflection.im != 0.0);
    for (int s = 0; s < n_off; ++s) {
      const int* o = offsets + 3 * s;
      const double t[3] = {o[0] * pitch[0], o[1] * pitch[1], o[2] * pitch[2]};
      const int self = o[0] == 0 && o[1] == 0 && o[2] == 0;
      plain.push_back(make_slot(t, zero, cmk(1.0, 0.0), 0, self));
      if (with_image) images.push_back(make_slot(t, zero, cmk(hs_reflection.re, hs_reflection.im), 1, 0));
    }
    run_assembly(cell, k, alpha, hs_axis, hs_offset, plain, images, device, out, ptr_kind);
  });
}

int fpbem_cu_assemble_hat(const fpbem_cu_cell* cell, double k, fpbem_c64 alpha, const double pitch[3],
                          const int counts[3], int n_hat, const int* hat_indices, int hs_axis, double hs_offset,
                          fpbem_c64 hs_reflection, int device, fpbem_c64* out, int ptr_kind) {
  return guard([&] {
    if (!pitch || !counts || (n_hat > 0 && (!hat_indices || !out))) fail(FPBEM_CU_EINVAL, "assemble_hat: null");
    if (hs_axis < 0 || hs_axis > 2) fail(FPBEM_CU_EINVAL, "assemble_hat: bad axis");
    std::vector<AssemblySlot> plain, images;
    for (int h = 0; h < n_hat; ++h) {
      const int* idx = hat_indices + 3 * h;
      int tgt[3] = {idx[0], idx[1], idx[2]}, src[3] = {0, 0, 0};
      tgt[hs_axis] = std::min(idx[hs_axis], counts[hs_axis] - 1);
      src[hs_axis] = idx[hs_axis] - tgt[hs_axis];
      const double t[3] = {tgt[0] * pitch[0], tgt[1] * pitch[1], tgt[2] * pitch[2]};
      const double sv[3] = {src[0] * pitch[0], src[1] * pitch[1], src[2] * pitch[2]};
      plain.push_back(make_slot(t, sv, cmk(hs_reflection.re, hs_reflection.im), 1, 0));
    }
    run_assembly(cell, k, alpha, hs_axis, hs_offset, plain, images, device, out, ptr_kind);
  });
}

int fpbem_cu_evaluate_field(const fpbem_cu_cell* cell, double k, const double pitch[3], const int counts[3],
                            const fpbem_c64* solution, int n_points, const double* points,
                            const fpbem_c64* p_incident, int hs_axis, double hs_offset, fpbem_c64 hs_reflection,
                            int device, fpbem_c64* out, int ptr_kind) {
  return guard([&] {
    if (!cell || !pitch || !counts || (n_points > 0 && (!points || !out || !solution)))
      fail(FPBEM_CU_EINVAL, "evaluate_field: null argument");
    if (n_points < 0 || counts[0] < 1 || counts[1] < 1 || counts[2] < 1)
      fail(FPBEM_CU_EDIM, "evaluate_field: bad counts or point count");
    const bool with_image = hs_reflection.re != 0.0 || hs_reflection.im != 0.0;
    if (with_image && (hs_axis < 0 || hs_axis > 2)) fail(FPBEM_CU_EINVAL, "evaluate_field: bad half-space axis");
    if (n_points == 0) return;
    check(cudaSetDevice(device), "set device");
    cudaStream_t s;
    check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> keep_s(s, [](cudaStream_t st) { cudaStreamDestroy(st); });
    CellDev dc;
    upload_cell(cell, dc, s);
    const long long n_total = static_cast<long long>(cell->n) * counts[0] * counts[1] * counts[2];
    const bool dev = ptr_kind == FPBEM_CU_PTR_DEVICE;
    double* dp = dalloc<double>(3 * static_cast<size_t>(n_points), "field points");
    std::unique_ptr<double, decltype(&cudaFree)> keep_p(dp, &cudaFree);
    h2d(dp, points, 3 * static_cast<size_t>(n_points) * sizeof(double), s, "field points");
    const c64* sol = reinterpret_cast<const c64*>(solution);
    std::unique_ptr<c64, decltype(&cudaFree)> keep_sol(nullptr, &cudaFree);
    if (!dev) {
      keep_sol.reset(dalloc<c64>(static_cast<size_t>(n_total), "field solution"));
      h2d(keep_sol.get(), solution, static_cast<size_t>(n_total) * sizeof(c64), s, "field solution");
      sol = keep_sol.get();
    }
    const c64* pinc = reinterpret_cast<const c64*>(p_incident);
    std::unique_ptr<c64, decltype(&cudaFree)> keep_pinc(nullptr, &cudaFree);
    if (!dev && p_incident) {
      keep_pinc.reset(dalloc<c64>(static_cast<size_t>(n_points), "incident values"));
      h2d(keep_pinc.get(), p_incident, static_cast<size_t>(n_points) * sizeof(c64), s, "incident values");
      pinc = keep_pinc.get();
    }
    c64* partial = dalloc<c64>(static_cast<size_t>(field_chunks(n_total)) * n_points, "field partial sums");
    std::unique_ptr<c64, decltype(&cudaFree)> keep_part(partial, &cudaFree);
    c64* dst = reinterpret_cast<c64*>(out);
    c64* out_tmp = nullptr;
    if (!dev) dst = out_tmp = dalloc<c64>(static_cast<size_t>(n_points), "field output");
    std::unique_ptr<c64, decltype(&cudaFree)> keep_out(out_tmp, &cudaFree);
    check(launch_field(dc.corners, dc.nv, dc.cen, dc.nrm, dc.diam, dc.beta, cell->n, counts, pitch, sol, dp, n_points,
                       pinc, k, with_image, hs_axis, hs_offset, cmk(hs_reflection.re, hs_reflection.im), partial, dst,
                       s),
          "field evaluation");
    if (!dev) check(cudaMemcpyAsync(out, dst, static_cast<size_t>(n_points) * sizeof(c64), cudaMemcpyDeviceToHost, s),
                    "field download");
    check(cudaStreamSynchronize(s), "field evaluation");
  });
}

int fpbem_cu_m2l_bank(int n_t, double k, int n_blk, const double* delta, const double* image_delta,
                      int parity_axis, fpbem_c64 reflection, int device, fpbem_c64* out, int ptr_kind) {
  return guard([&] {
    if (n_t < 0 || n_t > far_bank_max_nt()) fail(FPBEM_CU_EINVAL, "m2l_bank: n_t out of range");
    if (n_blk < 0 || (n_blk > 0 && (!out || (!delta && !image_delta))))
      fail(FPBEM_CU_EINVAL, "m2l_bank: null argument");
    if (image_delta && (parity_axis < 0 || parity_axis > 2)) fail(FPBEM_CU_EINVAL, "m2l_bank: bad parity axis");
    if (!std::isfinite(k) || k <= 0.0) fail(FPBEM_CU_EINVAL, "m2l_bank: wavenumber must be positive");
    for (const double* v : {delta, image_delta}) {
      if (!v) continue;
      for (int s = 0; s < n_blk; ++s) {
        const double r2 = v[3 * s] * v[3 * s] + v[3 * s + 1] * v[3 * s + 1] + v[3 * s + 2] * v[3 * s + 2];
        if (!(r2 > 0.0) || !std::isfinite(r2))  // solid_singular: evaluation at the singularity
          fail(FPBEM_CU_EINVAL, "m2l_bank: zero or non-finite translation vector");
      }
    }
    if (n_blk == 0) return;
    check(cudaSetDevice(device), "set device");
    cudaStream_t s;
    check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> keep_s(s, [](cudaStream_t st) { cudaStreamDestroy(st); });
    const size_t b = static_cast<size_t>(n_t + 1) * (n_t + 1), total = static_cast<size_t>(n_blk) * b * b;
    std::unique_ptr<double, decltype(&cudaFree)> keep_d(nullptr, &cudaFree), keep_i(nullptr, &cudaFree);
    if (delta) {
      keep_d.reset(dalloc<double>(3 * static_cast<size_t>(n_blk), "bank deltas"));
      h2d(keep_d.get(), delta, 3 * static_cast<size_t>(n_blk) * sizeof(double), s, "bank deltas");
    }
    if (image_delta) {
      keep_i.reset(dalloc<double>(3 * static_cast<size_t>(n_blk), "bank image deltas"));
      h2d(keep_i.get(), image_delta, 3 * static_cast<size_t>(n_blk) * sizeof(double), s, "bank image deltas");
    }
    const double* dd = keep_d.get();
    const double* di = keep_i.get();
    c64* dst = reinterpret_cast<c64*>(out);
    c64* tmp = nullptr;
    if (ptr_kind != FPBEM_CU_PTR_DEVICE) dst = tmp = dalloc<c64>(total, "bank output");
    std::unique_ptr<c64, decltype(&cudaFree)> keep_tmp(tmp, &cudaFree);
    check(launch_far_bank(device, n_t, k, n_blk, dd, di, parity_axis, cmk(reflection.re, reflection.im), dst, s),
          "m2l bank");
    if (ptr_kind != FPBEM_CU_PTR_DEVICE)
      check(cudaMemcpyAsync(out, dst, total * sizeof(c64), cudaMemcpyDeviceToHost, s), "bank download");
    check(cudaStreamSynchronize(s), "m2l bank");
  });
}

int fpbem_cu_comm_unique_id(unsigned char id_out[128]) {
  return guard([&] {
    void* lib = load_nccl();
    if (!lib) fail(FPBEM_CU_ENCCL, "libnccl.so.2 not loadable");
    auto get_id = reinterpret_cast<int (*)(void*)>(dlsym(lib, "ncclGetUniqueId"));
    if (!get_id) fail(FPBEM_CU_ENCCL, "ncclGetUniqueId missing");
    if (get_id(id_out) != 0) fail(FPBEM_CU_ENCCL, "ncclGetUniqueId failed");
  });
}

int fpbem_cu_comm_init(const unsigned char id[128], int nranks, int rank, int device, fpbem_cu_comm** out) {
  return guard([&] {
    void* lib = load_nccl();
    if (!lib) fail(FPBEM_CU_ENCCL, "libnccl.so.2 not loadable");
    struct IdBlob {
      unsigned char b[128];
    } blob;
    std::memcpy(blob.b, id, 128);
    auto init = reinterpret_cast<int (*)(void**, int, IdBlob, int)>(dlsym(lib, "ncclCommInitRank"));
    auto* c = new fpbem_cu_comm();
    c->lib = lib;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->allreduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, void*)>(
        dlsym(lib, "ncclAllReduce"));
    c->destroy = reinterpret_cast<int (*)(void*)>(dlsym(lib, "ncclCommDestroy"));
    if (!init || !c->allreduce || !c->destroy) {
      delete c;
      fail(FPBEM_CU_ENCCL, "NCCL symbols missing");
    }
    check(cudaSetDevice(device), "set device");
    if (init(&c->comm, nranks, blob, rank) != 0) {
      delete c;
      fail(FPBEM_CU_ENCCL, "ncclCommInitRank failed");
    }
    *out = c;
  });
}

void fpbem_cu_comm_destroy(fpbem_cu_comm* comm) {
  if (!comm) return;
  if (comm->comm && comm->destroy) comm->destroy(comm->comm);
  delete comm;
}

int fpbem_cu_fmm_set_comm(fpbem_cu_op* op, fpbem_cu_comm* comm) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_comm: null op");
    check(cudaSetDevice(op->device), "set device");
    if (!comm) {
      op->comm = nullptr;
      set_partition(op, 0, 1, 0.0);
      return;
    }
    // rank 0's far-field cost in pair equivalents, averaged over the ranks so
    // that every rank derives the same partition
    double f = comm->nranks > 1 ? calibrate_far_pairs(op) : 0.0;
    if (comm->nranks > 1) {
      double* df = dalloc<double>(1, "far pairs");
      std::unique_ptr<double, decltype(&cudaFree)> keep_df(df, &cudaFree);
      h2d(df, &f, sizeof(double), op->stream, "far pairs");
      const int rc = comm->allreduce(df, df, 1, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm->comm, op->stream);
      if (rc != 0) fail(FPBEM_CU_ENCCL, "ncclAllReduce failed: " + std::to_string(rc));
      check(cudaMemcpyAsync(&f, df, sizeof(double), cudaMemcpyDeviceToHost, op->stream), "far pairs");
      check(cudaStreamSynchronize(op->stream), "far pairs");
      f /= comm->nranks;
    }
    set_partition(op, comm->rank, comm->nranks, f);
    op->comm = comm;
  });
}

int fpbem_cu_fmm_set_partition(fpbem_cu_op* op, int rank, int nranks, double far_pairs) {
  return guard([&] {
    if (!op) fail(FPBEM_CU_EINVAL, "set_partition: null op");
    check(cudaSetDevice(op->device), "set device");
    set_partition(op, rank, nranks, far_pairs);
  });
}

int fpbem_cu_fmm_partition(const fpbem_cu_op* op, long long* lo, long long* hi, double* far_pairs) {
  return guard([&] {
    if (!op || !lo || !hi || !far_pairs) fail(FPBEM_CU_EINVAL, "partition: null argument");
    *lo = op->pair_lo;
    *hi = op->pair_hi;
    *far_pairs = op->far_pairs;
  });
}

int fpbem_cu_fmm_far_pairs(fpbem_cu_op* op, double* far_pairs) {
  return guard([&] {
    if (!op || !far_pairs) fail(FPBEM_CU_EINVAL, "far_pairs: null argument");
    check(cudaSetDevice(op->device), "set device");
    *far_pairs = calibrate_far_pairs(op);
  });
}

int fpbem_cu_partition_pairs(long long n_pairs, int nranks, int rank, double far_pairs, long long* lo,
                             long long* hi) {
  return guard([&] {
    if (n_pairs < 0 || nranks < 1 || rank < 0 || rank >= nranks || !lo || !hi || !(far_pairs >= 0.0))
      fail(FPBEM_CU_EINVAL, "partition: bad args");
    pair_range(n_pairs, nranks, rank, far_pairs, *lo, *hi);
  });
}

}  // extern "C"
