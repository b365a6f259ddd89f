// C-ABI implementation, part 5: restarted GMRES with the Krylov basis
// distributed over the ranks of the handle's communicator (SURVEY.md §8e:
// "GMRES vectors distributed by slab", one batched all-reduce per
// Gram-Schmidt pass instead of MGS's j+1 sequential ones).
//
// Control flow of src/solver.cpp:21-123 (x0 = 0, zero right-hand side =
// converged after 0 iterations, estimate-based inner exit, true residual per
// cycle, reorthogonalisation iff ||w_post|| < ||w_pre|| / 2, non-finite
// product = error). What differs from the reference's MGS is the projection
// pass: classical Gram-Schmidt, h = V^H w in one batched reduction, then
// w -= V h — the second pass of the same test (the Daniel-Gragg-Kaufman-Stewart
// criterion) restores orthogonality where MGS would need it. Rows are split
// in slabs of whole cells; per Arnoldi step:
//   all-gather v_j -> full p ; partial product of this rank's near-field pairs
//   (+ far field on rank 0) ; reduce-scatter -> w on the slab ;
//   dots (+ ||w||^2, non-finite count) -> all-reduce ; update (+ ||w||^2) ->
//   all-reduce ; one read-back of the scalars for the host Givens step.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "givens.hpp"
#include "handle.cuh"

using namespace fpbem_cu;

namespace {

struct Slab {
  int nranks = 1, rank = 0;
  long long rows = 0;    // per rank, padded: ceil(n_cells / nranks) cells
  long long lo = 0, hi = 0;  // this rank's global rows [lo, hi)
};

// the communicator of the distributed solve: the slab plan's, else the pair partition's
fpbem_cu_comm* dist_comm(const fpbem_cu_op* op) { return op->slab ? slab_comm(op) : op->comm; }

Slab slab_of(const fpbem_cu_op* op) {
  Slab sl;
  if (fpbem_cu_comm* c = dist_comm(op)) {
    sl.nranks = c->nranks;
    sl.rank = c->rank;
  }
  if (op->slab) {  // whole planes of the slab plan: ceil(planes / P) per rank
    long long lo = 0, hi = 0, per = 0;
    slab_range(op, sl.rank, &lo, &hi, &per);
    sl.rows = per;
    sl.lo = lo;
    sl.hi = hi;
    return sl;
  }
  const long long cells = (op->n_cells + sl.nranks - 1) / sl.nranks;
  sl.rows = cells * op->n;
  sl.lo = std::min<long long>(op->N, sl.rank * sl.rows);
  sl.hi = std::min<long long>(op->N, (sl.rank + 1) * sl.rows);
  return sl;
}

struct DistOut {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
};

DistOut gmres_dist(fpbem_cu_op* op, const c64* b, bool b_host, c64* x, bool x_host, double tol, int restart,
                   int max_iter) {
  Nvtx range("gmres (distributed, classical Gram-Schmidt)");
  using cd = std::complex<double>;
  cudaStream_t s = op->stream;
  fpbem_cu_comm* comm = dist_comm(op);
  const Slab sl = slab_of(op);
  const long long ns = sl.rows;
  const long long nfull = ns * sl.nranks;
  const int m = std::max(1, restart);
  if (m + 1 >= kCgsMaxCols) fail(FPBEM_CU_EINVAL, "gmres_dist: restart must be < " + std::to_string(kCgsMaxCols - 1));
  DistOut rep;

  // the solver's device buffers live in one arena kept with the handle between
  // solves (the basis alone is (restart + 1) slabs; allocating and freeing it per
  // call cost more than a short solve)
  const size_t vb = static_cast<size_t>(ns) * sizeof(c64);
  const size_t cols_ = static_cast<size_t>(m) + 2;
  auto round256 = [](size_t b) { return (std::max<size_t>(b, 1) + 255) & ~static_cast<size_t>(255); };
  const size_t arena_parts[] = {vb * (m + 1), vb, vb, vb, vb, static_cast<size_t>(nfull) * sizeof(c64),
                                static_cast<size_t>(nfull) * sizeof(c64), (2 * cols_ + 4) * sizeof(c64),
                                cols_ * kCgsMaxBlocks * sizeof(c64), sizeof(unsigned)};
  size_t arena = 0;
  for (size_t b : arena_parts) arena += round256(b);
  if (op->dws_bytes < arena) {
    if (op->dws) check(cudaFree(op->dws), "dist workspace");
    op->dws = nullptr;
    op->dws_bytes = 0;
    check(cudaMalloc(&op->dws, arena), "dist workspace");
    op->dws_bytes = arena;
  }
  size_t arena_off = 0;
  auto alloc = [&](size_t bytes, const char*) {
    void* p = static_cast<char*>(op->dws) + arena_off;
    arena_off += round256(bytes);
    return p;
  };
  c64* V = static_cast<c64*>(alloc(vb * (m + 1), "dist basis"));
  c64* xl = static_cast<c64*>(alloc(vb, "dist x"));
  c64* bl = static_cast<c64*>(alloc(vb, "dist b"));
  c64* rl = static_cast<c64*>(alloc(vb, "dist r"));
  c64* tl = static_cast<c64*>(alloc(vb, "dist Ax"));
  c64* pfull = static_cast<c64*>(alloc(static_cast<size_t>(nfull) * sizeof(c64), "dist gathered vector"));
  c64* ypart = static_cast<c64*>(alloc(static_cast<size_t>(nfull) * sizeof(c64), "dist partial product"));
  // scalars: pass-1 [h_0..h_j | (||w||^2, #non-finite)], pass-2 the same, then doubles
  const size_t cols = static_cast<size_t>(m) + 2;
  c64* red = static_cast<c64*>(alloc((2 * cols + 4) * sizeof(c64), "dist scalars"));
  c64* redc = red + cols;
  double* dd = reinterpret_cast<double*>(red + 2 * cols);  // [0] post ||w||^2, [1] r^2, [2] #non-finite
  c64* partials = static_cast<c64*>(alloc(cols * kCgsMaxBlocks * sizeof(c64), "dist partials"));
  unsigned* counter = static_cast<unsigned*>(alloc(sizeof(unsigned), "dist counter"));
  RedScratch rs{reinterpret_cast<double*>(partials), partials, counter};
  check(cudaMemsetAsync(counter, 0, sizeof(unsigned), s), "counter");
  check(cudaMemsetAsync(ypart, 0, static_cast<size_t>(nfull) * sizeof(c64), s), "pad rows");
  check(cudaMemsetAsync(pfull, 0, static_cast<size_t>(nfull) * sizeof(c64), s), "pad rows");
  check(cudaMemsetAsync(bl, 0, vb, s), "b slab");
  check(cudaMemsetAsync(xl, 0, vb, s), "x0");
  check(cudaMemsetAsync(tl, 0, vb, s), "Ax");  // padding rows of the slab product stay zero
  check(cudaMemsetAsync(V, 0, vb * (m + 1), s), "basis");
  const size_t mine = static_cast<size_t>(sl.hi - sl.lo) * sizeof(c64);
  if (mine)
    check(cudaMemcpyAsync(bl, b + sl.lo, mine, b_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s),
          "b slab");
  const size_t scal_bytes = (2 * cols + 4) * sizeof(c64);
  ensure_pinned(op, scal_bytes);
  char* pin = static_cast<char*>(op->pinned);
  auto fetch = [&]() {
    check(cudaMemcpyAsync(pin, red, scal_bytes, cudaMemcpyDeviceToHost, s), "dist readback");
    check(cudaStreamSynchronize(s), "dist sync");
  };
  auto get_c = [&](const c64* base, size_t i) {
    c64 v;
    std::memcpy(&v, pin + (reinterpret_cast<const char*>(base + i) - reinterpret_cast<const char*>(red)), 16);
    return cd(v.x, v.y);
  };
  auto get_d = [&](int i) {
    double v;
    std::memcpy(&v, pin + 2 * cols * sizeof(c64) + i * sizeof(double), 8);
    return v;
  };
  auto all_d = [&](double* p, size_t count) { comm_allreduce(comm, p, count, s); };
  auto col = [&](int j) { return V + static_cast<long long>(j) * ns; };
  // out (slab) = A in (slab): gather, this rank's partial product, reduce-scatter
  auto product = [&](const c64* in, c64* out) {
    if (op->slab) {  // slab in, slab out: the all-to-all transposes live inside the product
      slab_apply(op, in, out);
      return;
    }
    comm_allgather(comm, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(pfull), 2 * ns, s);
    apply_device(op, pfull, ypart, 1, false);
    comm_reduce_scatter(comm, reinterpret_cast<double*>(ypart), reinterpret_cast<double*>(out), 2 * ns, s);
  };
  auto nonfinite = [&]() { fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value"); };

  // ||b|| (cols = 0: the kernel returns (||b||^2, #non-finite))
  check(launch_cgs_dots(V, ns, 0, bl, ns, partials, counter, red, s), "bnorm");
  all_d(reinterpret_cast<double*>(red), 2);
  op->launches++;
  fetch();
  const double bnorm = std::sqrt(get_c(red, 0).real());
  auto finish = [&]() {  // every rank gets the full x
    comm_allgather(comm, reinterpret_cast<const double*>(xl), reinterpret_cast<double*>(pfull), 2 * ns, s);
    check(cudaMemcpyAsync(x, pfull, static_cast<size_t>(op->N) * sizeof(c64),
                          x_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s),
          "x out");
    check(cudaStreamSynchronize(s), "dist sync");
  };
  if (bnorm == 0.0) {
    rep.converged = true;
    finish();
    return rep;
  }
  GmresCycle cyc(m);
  const c64* r = bl;
  double rnorm = bnorm;
  while (rep.iterations < max_iter) {
    check(launch_div(r, col(0), ns, rnorm, s), "v0");
    op->launches++;
    cyc.start(rnorm);
    int j = 0;
    for (; j < m && rep.iterations < max_iter; ++j) {
      c64* w = col(j + 1);
      product(col(j), w);
      // pass 1: h = V^H w, ||w||^2, non-finite count; all-reduce; w -= V h
      check(launch_cgs_dots(V, ns, j + 1, w, ns, partials, counter, red, s), "cgs dots");
      all_d(reinterpret_cast<double*>(red), 2 * static_cast<size_t>(j + 2));
      check(launch_cgs_update(w, V, ns, j + 1, red, ns, reinterpret_cast<double*>(partials), counter, dd, s),
            "cgs update");
      all_d(dd, 1);
      op->launches += 2;
      fetch();
      if (get_c(red, j + 1).imag() > 0.0) nonfinite();
      for (int i = 0; i <= j; ++i) cyc.h(i, j) = get_c(red, i);
      const double pre2 = get_c(red, j + 1).real();
      double wnorm2 = get_d(0);
      if (std::sqrt(wnorm2) < 0.5 * std::sqrt(pre2)) {  // second pass (:63-69)
        check(launch_cgs_dots(V, ns, j + 1, w, ns, partials, counter, redc, s), "cgs reorth dots");
        all_d(reinterpret_cast<double*>(redc), 2 * static_cast<size_t>(j + 2));
        check(launch_cgs_update(w, V, ns, j + 1, redc, ns, reinterpret_cast<double*>(partials), counter, dd, s),
              "cgs reorth update");
        all_d(dd, 1);
        op->launches += 2;
        fetch();
        for (int i = 0; i <= j; ++i) cyc.h(i, j) += get_c(redc, i);
        wnorm2 = get_d(0);
      }
      const double hlast = std::sqrt(wnorm2);
      cyc.h(j + 1, j) = hlast;
      if (hlast > 0.0) {
        check(launch_div(w, w, ns, hlast, s), "normalise");
        op->launches++;
      }
      ++rep.iterations;
      const double est = cyc.rotate(j) / bnorm;
      rep.history.push_back(est);
      if (est <= tol || hlast == 0.0) {
        ++j;
        break;
      }
    }
    const std::vector<cd> y = cyc.solve(j);
    if (j > 0) {  // x += V y on the slab (:109-110)
      std::vector<c64> yh(j);
      for (int i = 0; i < j; ++i) yh[i] = cmk(y[i].real(), y[i].imag());
      c64* ydev = redc;  // pass-2 scalars are free here
      check(cudaStreamSynchronize(s), "dist sync");
      std::memcpy(pin, yh.data(), j * sizeof(c64));
      check(cudaMemcpyAsync(ydev, pin, j * sizeof(c64), cudaMemcpyHostToDevice, s), "y upload");
      check(launch_update_x(xl, V, ns, ydev, j, ns, s), "x update");
      op->launches++;
    }
    // true residual r = b - A x (:111-112), non-finite product checked
    product(xl, tl);
    check(launch_cgs_dots(V, ns, 0, tl, ns, partials, counter, red, s), "residual finite check");
    check(launch_residual(bl, tl, rl, ns, rs, dd + 1, s), "residual");
    op->launches += 2;
    check(cudaMemcpyAsync(dd + 2, reinterpret_cast<double*>(red) + 1, sizeof(double), cudaMemcpyDeviceToDevice, s),
          "flag");
    all_d(dd + 1, 2);
    fetch();
    if (get_d(2) > 0.0) nonfinite();
    rnorm = std::sqrt(get_d(1));
    r = rl;
    if (rnorm / bnorm <= tol) {
      rep.converged = true;
      break;
    }
  }
  if (!rep.history.empty()) rep.converged = rep.converged || rnorm / bnorm <= tol;
  finish();
  return rep;
}

}  // namespace

extern "C" {

int fpbem_cu_gmres_dist(fpbem_cu_op* op, const fpbem_c64* b, fpbem_c64* x, double tol, int restart, int max_iter,
                        int ptr_kind, int* iterations, int* converged, double* history, int history_cap,
                        int* history_len) {
  return guard([&] {
    if (!op || !b || !x || !iterations || !converged) fail(FPBEM_CU_EINVAL, "gmres_dist: null argument");
    if (!op->slab && !op->comm && op->nranks > 1)
      fail(FPBEM_CU_EINVAL, "gmres_dist: a pair partition needs a communicator (fpbem_cu_fmm_set_comm)");
    check(cudaSetDevice(op->device), "set device");
    const bool host = ptr_kind != FPBEM_CU_PTR_DEVICE;
    DistOut o = gmres_dist(op, reinterpret_cast<const c64*>(b), host, reinterpret_cast<c64*>(x), host, tol, restart,
                           max_iter);
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    if (history_len) *history_len = static_cast<int>(o.history.size());
    if (history)
      for (int i = 0; i < std::min(history_cap, static_cast<int>(o.history.size())); ++i) history[i] = o.history[i];
  });
}

int fpbem_cu_gmres_dist_rows(const fpbem_cu_op* op, long long* lo, long long* hi) {
  return guard([&] {
    if (!op || !lo || !hi) fail(FPBEM_CU_EINVAL, "gmres_dist_rows: null argument");
    const Slab sl = slab_of(op);
    *lo = sl.lo;
    *hi = sl.hi;
  });
}

}  // extern "C"
