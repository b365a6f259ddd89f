// Internal to libfpbem_cuda.so (not installed): the operator handle shared by
// the C-ABI translation units — fpbem_cuda.cu (operator create / apply /
// spectrum), gmres.cu (device GMRES), device_assembly.cu (near-field blocks,
// M2L bank, field evaluation) and comm.cu (NCCL, multi-GPU partition).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: no-ops unless a profiler injects itself

#include <functional>
#include <string>
#include <vector>

#include "../../include/fpbem_cuda.h"
#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

inline thread_local std::string g_err;  // fpbem_cu_last_error

// host-side stage range on the NVTX timeline (nsys / ncu --nvtx), scoped
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

struct Fail {
  int code;
};

[[noreturn]] inline void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

inline void check(cudaError_t e, const char* what) {
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
inline void h2d(void* dst, const void* src, size_t bytes, cudaStream_t stream, const char* what) {
  if (bytes == 0) return;
  check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream), what);
  check(cudaStreamSynchronize(stream), what);
}

// C-ABI body: error code for the caller, message in g_err
inline int guard(const std::function<void()>& fn) {
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

}  // namespace fpbem_cu

using namespace fpbem_cu;  // internal header: the handle below is written in the kernel types

// --------------------------------------------------------------------------
// Communicator: NCCL (loaded at runtime, so the library has no hard NCCL
// dependency) or a caller-supplied host all-reduce (e.g. a gloo group),
// staged through pinned host memory. comm.cu implements the collectives.

struct fpbem_cu_comm {
  void* lib = nullptr;
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0, device = 0;
  int (*allreduce)(const void*, void*, size_t, int, int, void*, void*) = nullptr;
  int (*reduce_scatter)(const void*, void*, size_t, int, int, void*, void*) = nullptr;
  int (*allgather)(const void*, void*, size_t, int, void*, void*) = nullptr;
  int (*destroy)(void*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, void*) = nullptr;  // ncclSend(buf, count, type, peer, comm, stream)
  int (*recv)(void*, size_t, int, int, void*, void*) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  // host callback form (cb != nullptr)
  fpbem_cu_allreduce_fn cb = nullptr;
  void* cb_ctx = nullptr;
  double* stage = nullptr;  // pinned
  size_t stage_count = 0;
  // simulated form (fpbem_cu_comm_simulated): rank `rank` of `nranks` alone on
  // this device; collectives move only this rank's own blocks and count the
  // bytes the real exchange would send (per-rank timing on one GPU)
  bool sim = false;
  unsigned long long sim_bytes = 0;
  long long sim_calls = 0;
};

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

  // near field as a lattice convolution: the Toeplitz blocks
  // embedded in an Ln lattice (Ln = M + max|o| per axis) and DFT'd once, so the
  // product is pruned DFT -> per-mode block product -> pruned inverse DFT
  bool near_fft = false;
  int Ln[3] = {1, 1, 1};
  long long qn = 0;
  c64* shat = nullptr;  // qn blocks n x n column-major, q = (qz*Lny + qy)*Lnx + qx
  c64* twn[3] = {nullptr, nullptr, nullptr};
  c64* nfa = nullptr;   // spectra of x / y, [rhs][q][n], sized for max_rhs
  c64* nfb = nullptr;
  int4* mjobs = nullptr;    // DMMA jobs over this rank's items (many right-hand sides)
  int mjobs_nrhs = -1, n_mjobs = 0, mjobs_cap = 0;
  // stored blocks = work items = orbits of Fourier modes under the cell's
  // verified axis-sign symmetries g (S_{A_g o} = P_g S_o P_g, so
  // Shat(A_g q) = P_g Shat(q) P_g): one block per orbit serves
  // up to 8 modes, the images through P_g; without symmetries every mode is an item
  int near_sym_mask = 1;        // bit g: axis-sign map g verified (bit 0 = identity)
  double near_sym_dev = -1.0;   // max over the given g of max|S_{A_g o}[P_g i, P_g j] - S_o[i, j]| / max|S|
  int* perm = nullptr;          // device: P_g for g = 1..7 (row g - 1, n entries)
  int near_nimg = 1;            // images per item (largest orbit): 1, 2, 4 or 8
  int* items = nullptr;         // device: [n_items][8] modes (-1 unused), then [n_items][8] g (0 = identity)
  std::vector<int> items_q, items_g;
  long long n_items = 0;
  long long mode_lo = 0, mode_hi = 0;  // this rank's items

  // expansions and spectrum
  c64* u0 = nullptr;
  c64* v0 = nullptr;
  c64* v0t = nullptr;  // V0^T (b rows of n), for the P2M kernel
  // work items of the fused z kernel: column pairs (c, mirror) when Λ has the
  // parity Λ(-q) = D Λ(q) D (checked on the device at create), single columns
  // otherwise (and always for the image spectrum)
  int2* z_items_pair = nullptr;
  int2* z_items_single = nullptr;
  int n_z_items_pair = 0, n_z_items_single = 0;
  bool lam_paired = false;
  bool lam_zsym = false;  // also Λ(qx, qy, -qz) = Dz Λ(q) Dz (the flat stream reads a quarter of Λ)
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
  // pipelined host-pointer product (apply_host_pipelined): copy-in / copy-out
  // streams and per-chunk events
  cudaStream_t cin = nullptr, cout = nullptr;
  // lockstep GMRES workspace (basis + work vectors), kept between solves
  void* bws = nullptr;
  size_t bws_bytes = 0;
  void* dws = nullptr;  // distributed GMRES arena
  size_t dws_bytes = 0;
  cudaEvent_t pev_in[8] = {}, pev_out[8] = {};

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
  bool serial_timing = false;  // stage timing with the far field on the main stream (exact stage times)
  cudaEvent_t ev[10] = {};
  double stage_ms[6] = {0, 0, 0, 0, 0, 0};  // + [5]: lattice-path mode product (events 7-8)
  long long applies = 0;
  long long launches = 0;

  fpbem_cu_comm* comm = nullptr;
  struct SlabPlan* slab = nullptr;  // slab-distributed product (slab.cu), set by fpbem_cu_fmm_set_slabs
};

namespace fpbem_cu {
// operator internals (fpbem_cuda.cu) used by the other translation units
void pair_range(long long n_pairs, int nranks, int rank, double far_pairs, long long& lo, long long& hi);
void set_partition(fpbem_cu_op* op, int rank, int nranks, double far_pairs);
double calibrate_far_pairs(fpbem_cu_op* op);
// y = A x; reduce = false leaves this rank's partial product un-summed
void apply_device(fpbem_cu_op* op, const c64* x, c64* y, int nrhs, bool reduce = true);
void ensure_pinned(fpbem_cu_op* op, size_t bytes);
// collectives over fp64 device buffers, ordered on `s` (comm.cu)
void comm_allreduce(fpbem_cu_comm* c, double* buf, size_t count, cudaStream_t s);
void comm_reduce_scatter(fpbem_cu_comm* c, double* full, double* mine, size_t per_rank, cudaStream_t s);
void comm_allgather(fpbem_cu_comm* c, const double* mine, double* full, size_t per_rank, cudaStream_t s);
// one block of an all-to-all: this rank sends send + sdisp[d] (scount[d] doubles)
// to every rank d and receives rcount[s] doubles from rank s at recv + rdisp[s];
// `all` is the P x P matrix of block sizes [src * P + dst] (every rank's view,
// for the host-staged form)
struct A2aPart {
  const double* send;
  double* recv;
  const size_t *scount, *sdisp, *rcount, *rdisp, *all;
};
// the parts' transfers in one NCCL group (send/recv), or host-staged one after another
void comm_alltoallv(fpbem_cu_comm* c, const A2aPart* parts, int n_parts, cudaStream_t s);
void slab_destroy(fpbem_cu_op* op);
// event i of the handle's stage timing (no-op unless timing is enabled)
void ev_record(fpbem_cu_op* op, int i, cudaStream_t st);
// slab plan (slab.cu): y = (A x) on this rank's planes, device pointers, one right-hand side
void slab_apply(fpbem_cu_op* op, const c64* x, c64* y);
fpbem_cu_comm* slab_comm(const fpbem_cu_op* op);
// rank r's rows [lo, hi) and the padded rows per rank (ceil(planes / P) planes)
void slab_range(const fpbem_cu_op* op, int r, long long* lo, long long* hi, long long* per_rank_rows);
}  // namespace fpbem_cu
