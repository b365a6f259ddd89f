// C-ABI implementation, part 2: restarted GMRES with the Krylov basis resident
// in HBM (solver::gmres, src/solver.cpp:21-123) — gmres_one() per right-hand
// side (fused MGS Arnoldi step, one read-back per step), gmres_batched() for
// several right-hand sides in lockstep, and the ApplyFn form fpbem_cu_gmres_fn.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "givens.hpp"
#include "handle.cuh"

using namespace fpbem_cu;

namespace {
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
  Nvtx range("gmres (solver::gmres, one right-hand side)");
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
  GmresCycle cyc(m);
  auto Hm = [&](int i, int j) -> cd& { return cyc.h(i, j); };
  const c64* r = b_dev;  // r = b_eff on the first cycle
  double rnorm = bnorm;
  const bool fused = mgs_fused_supported(n);
  // two pinned slots for the pipelined step read-backs (header + h + hc), after
  // the region fetch() / the y upload use
  const size_t slot_bytes = 128 + 2 * sizeof(c64) * static_cast<size_t>(op->scal_cap);
  const size_t slot0 = (sizeof(c64) * (8 + 3 * static_cast<size_t>(op->scal_cap)) + 64 + 255) / 256 * 256;
  ensure_pinned(op, slot0 + 2 * slot_bytes);
  pin = static_cast<char*>(op->pinned);
  char* slot[2] = {pin + slot0, pin + slot0 + slot_bytes};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (auto& e : ev) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "gmres events");
  std::unique_ptr<cudaEvent_t, void (*)(cudaEvent_t*)> keep_ev(ev, [](cudaEvent_t* e) {
    cudaEventDestroy(e[0]);
    cudaEventDestroy(e[1]);
  });

  while (rep.iterations < max_iter) {
    check(launch_div(r, col(0), n, rnorm, s), "v0");
    op->launches++;
    cyc.start(rnorm);
    int j = 0;
    if (fused) {
      // Pipelined Arnoldi: the device completes each step (MGS, the conditional
      // second pass, h_{j+1,j} and the normalisation: one cooperative launch) and
      // its scalars come back while the next step's product runs; the host
      // applies the Givens rotations and the stopping test of step j with the
      // GPU already on step j + 1. A step enqueued past the stopping point only
      // writes basis column j + 2, never read: same iterations, same solution.
      auto enqueue = [&](int jj) {
        apply(col(jj), col(jj + 1));
        check(launch_mgs_fused(col(jj + 1), V, n, jj, n, h, sd, op->flag, op->rs, true, s, hc), "mgs step");
        op->launches++;
        check(cudaMemcpyAsync(slot[jj & 1], sd, slot_bytes, cudaMemcpyDeviceToHost, s), "gmres readback");
        check(cudaEventRecord(ev[jj & 1], s), "gmres event");
      };
      if (rep.iterations < max_iter) enqueue(0);
      for (; j < m && rep.iterations < max_iter; ++j) {
        if (j + 1 < m && rep.iterations + 1 < max_iter) enqueue(j + 1);
        check(cudaEventSynchronize(ev[j & 1]), "gmres sync");
        const char* p = slot[j & 1];
        int fl;
        std::memcpy(&fl, p + 64, sizeof(int));
        if (fl) {
          check(cudaStreamSynchronize(s), "gmres sync");
          check(cudaMemsetAsync(op->flag, 0, sizeof(int), s), "flag reset");
          fail(FPBEM_CU_ENONFINITE, "gmres: operator returned a non-finite value");
        }
        double nr[6];
        std::memcpy(nr, p, sizeof(nr));
        for (int i = 0; i <= j; ++i) {
          c64 v;
          std::memcpy(&v, p + 128 + i * sizeof(c64), sizeof(c64));
          Hm(i, j) = cd(v.x, v.y);
        }
        if (nr[4] != 0.0)  // reorthogonalised (:63-69): h += hc
          for (int i = 0; i <= j; ++i) {
            c64 v;
            std::memcpy(&v, p + 128 + (op->scal_cap + i) * sizeof(c64), sizeof(c64));
            Hm(i, j) += cd(v.x, v.y);
          }
        const double hlast = nr[5];
        Hm(j + 1, j) = hlast;
        ++rep.iterations;
        const double est = cyc.rotate(j) / bnorm;
        rep.history.push_back(est);
        if (est <= tol || hlast == 0.0) {
          ++j;
          break;
        }
      }
    } else {
      for (; j < m && rep.iterations < max_iter; ++j) {
        c64* w = col(j + 1);
        apply(col(j), w);
        check(launch_sqnorm(w, n, op->rs, sd + 0, op->flag, s), "pre norm");
        // MGS: h_0 = <v_0,w>; (w -= h_i v_i, h_{i+1} = <v_{i+1}, w>)...; w -= h_j v_j, ||w||^2
        check(launch_dotc(col(0), w, n, op->rs, h + 0, s), "mgs dot");
        for (int i = 0; i < j; ++i)
          check(launch_axpy_dotc(w, col(i), h + i, col(i + 1), n, op->rs, h + i + 1, s), "mgs step");
        check(launch_axpy_sqnorm(w, col(j), h + j, n, op->rs, sd + 1, s), "mgs last");
        op->launches += j + 3;
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
          check(launch_dotc(col(0), w, n, op->rs, hc + 0, s), "reorth dot");
          for (int i = 0; i < j; ++i)
            check(launch_axpy_dotc(w, col(i), hc + i, col(i + 1), n, op->rs, hc + i + 1, s), "reorth step");
          check(launch_axpy_sqnorm(w, col(j), hc + j, n, op->rs, sd + 2, s), "reorth last");
          op->launches += j + 2;
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
        ++rep.iterations;
        const double est = cyc.rotate(j) / bnorm;
        rep.history.push_back(est);
        if (est <= tol || hlast == 0.0) {
          ++j;
          break;
        }
      }
    }
    // y = triu(H_jj)^{-1} g ; x += V y (:109-110)
    const std::vector<cd> y = cyc.solve(j);
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
  Nvtx range("gmres (lockstep batch)");
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
  // the basis and the four work vectors stay with the handle between solves
  // (64 right-hand sides of cfg5 at restart 50: 72 GB, whose cudaMalloc / cudaFree
  // per call cost more than many Arnoldi steps)
  const size_t ws_bytes = vecb * G * (m + 5);
  if (op->bws_bytes < ws_bytes) {
    if (op->bws) check(cudaFree(op->bws), "batched workspace");
    op->bws = nullptr;
    op->bws_bytes = 0;
    check(cudaMalloc(&op->bws, ws_bytes), "batched workspace");
    op->bws_bytes = ws_bytes;
  }
  c64* V = static_cast<c64*>(op->bws);
  c64* R = V + static_cast<size_t>(n) * G * (m + 1);
  c64* T = R + static_cast<size_t>(n) * G;
  c64* P = T + static_cast<size_t>(n) * G;
  c64* Q = P + static_cast<size_t>(n) * G;
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
  // per-RHS fused MGS (one cooperative launch per right-hand side and step, w
  // resident in shared memory: each basis vector is streamed once per
  // projection instead of the batched kernels' four vector passes), when the
  // vector fits the cooperative grid; FPBEM_GMRES_BMGS=0 keeps the batched kernels
  static const bool per_rhs_env = [] {
    const char* v = std::getenv("FPBEM_GMRES_BMGS");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  const bool per_rhs = per_rhs_env && mgs_fused_supported(n);
  // [r][m+1] h, [r][m+1] reorth h, [r][4] norms (pre, post, -, post after reorth)
  const size_t o_fh = 0, o_fhc = o_fh + 16 * static_cast<size_t>(G) * (m + 1),
               o_fn = o_fhc + 16 * static_cast<size_t>(G) * (m + 1), ftotal = o_fn + 32 * static_cast<size_t>(G);
  char* fsc = per_rhs ? static_cast<char*>(alloc(ftotal, "per-rhs mgs scalars")) : nullptr;
  ensure_pinned(op, total + 64 + (per_rhs ? ftotal : 0));
  char* fpin = static_cast<char*>(op->pinned) + total + 64;
  auto ffetch = [&](size_t off, size_t bytes) {
    check(cudaMemcpyAsync(fpin + off, fsc + off, bytes, cudaMemcpyDeviceToHost, s), "batched readback");
    check(cudaStreamSynchronize(s), "batched sync");
  };
  auto fget_c = [&](size_t off, size_t idx) {
    c64 v;
    std::memcpy(&v, fpin + off + 16 * idx, 16);
    return cd(v.x, v.y);
  };
  auto fget_d = [&](size_t idx) {
    double v;
    std::memcpy(&v, fpin + o_fn + 8 * idx, 8);
    return v;
  };
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
  std::vector<GmresCycle> cyc(G, GmresCycle(m));
  std::vector<int> jr(G, 0);
  std::vector<char> inner(G, 0);
  const c64* rsrc = Bd;

  // normalise w, then the rotations / Givens / estimate of step j (:74-105) per RHS
  auto finish_step = [&](int j, const std::vector<int>& it, const std::vector<double>& wn2) {
    c64* W = V + static_cast<long long>(j + 1) * G * n;
    std::vector<double> hl(G, 1.0);
    std::vector<int> norm_set;
    for (int r : it) {
      hl[r] = std::sqrt(wn2[r]);
      if (hl[r] > 0.0) norm_set.push_back(r);
    }
    if (!norm_set.empty()) {
      set_mask(norm_set);
      put(o_d, hl.data(), 8 * static_cast<size_t>(G));
      check(launch_b_div(W, W, n, n, G, d_mask, d_d, s), "normalise");
      op->launches++;
    }
    for (int r : it) {  // rotations, Givens, estimate (:74-105), per RHS
      const double hlast = hl[r];
      cyc[r].h(j + 1, j) = hlast;
      const double res = cyc[r].rotate(j);
      ++out.iterations[r];
      const double est = res / bnorm[r];
      out.history[r].push_back(est);
      jr[r] = j + 1;
      if (est <= tol || hlast == 0.0) inner[r] = 0;
    }
  };


  while (true) {
    std::vector<int> act;
    for (int r = 0; r < G; ++r)
      if (!done[r] && out.iterations[r] < max_iter) act.push_back(r);
    if (act.empty()) break;
    set_mask(act);
    put(o_d, rnorm.data(), 8 * static_cast<size_t>(G));
    check(launch_b_div(rsrc, V, n, n, G, d_mask, d_d, s), "v0");  // v0 = r / ||r||
    for (int r : act) {
      cyc[r].start(rnorm[r]);
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
      if (per_rhs) {  // the single-RHS MGS of gmres_one for each right-hand side (same arithmetic)
        const long long ld = static_cast<long long>(G) * n;
        for (int r : it) {
          check(launch_mgs_fused(W + static_cast<long long>(r) * n, V + static_cast<long long>(r) * n, ld, j, n,
                                 reinterpret_cast<c64*>(fsc + o_fh) + static_cast<size_t>(r) * (m + 1),
                                 reinterpret_cast<double*>(fsc + o_fn) + 4 * static_cast<size_t>(r), d_flag + r,
                                 op->rs, true, s),
                "mgs fused");
          op->launches++;
        }
        fetch(0, g8);  // flags
        flags_of(it);
        ffetch(0, ftotal);
        std::vector<int> reo;
        std::vector<double> wn2(G, 0.0);
        for (int r : it) {
          for (int i = 0; i <= j; ++i) cyc[r].h(i, j) = fget_c(o_fh, static_cast<size_t>(r) * (m + 1) + i);
          wn2[r] = fget_d(4 * static_cast<size_t>(r) + 1);
          if (std::sqrt(wn2[r]) < 0.5 * std::sqrt(fget_d(4 * static_cast<size_t>(r)))) reo.push_back(r);  // (:63-69)
        }
        for (int r : reo) {
          check(launch_mgs_fused(W + static_cast<long long>(r) * n, V + static_cast<long long>(r) * n, ld, j, n,
                                 reinterpret_cast<c64*>(fsc + o_fhc) + static_cast<size_t>(r) * (m + 1),
                                 reinterpret_cast<double*>(fsc + o_fn) + 4 * static_cast<size_t>(r) + 2, d_flag + r,
                                 op->rs, false, s),
                "reorth fused");
          op->launches++;
        }
        if (!reo.empty()) {
          ffetch(0, ftotal);
          for (int r : reo) {
            for (int i = 0; i <= j; ++i) cyc[r].h(i, j) += fget_c(o_fhc, static_cast<size_t>(r) * (m + 1) + i);
            wn2[r] = fget_d(4 * static_cast<size_t>(r) + 3);
          }
        }
        finish_step(j, it, wn2);
        continue;
      }
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
        for (int i = 0; i <= j; ++i) cyc[r].h(i, j) = get_c(o_h, static_cast<size_t>(i) * G + r);
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
          for (int i = 0; i <= j; ++i) cyc[r].h(i, j) += get_c(o_hc, static_cast<size_t>(i) * G + r);
          wn2[r] = get_d(o_post2, r);
        }
      }
      finish_step(j, it, wn2);
    }
    // x_r += V_r y_r for every RHS of the cycle, then the true residuals (:109-116)
    std::vector<c64> yh(static_cast<size_t>(m) * G, cmk(0.0, 0.0));
    for (int r : act) {
      const int jj = jr[r];
      const std::vector<cd> y = cyc[r].solve(jj);
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

extern "C" {

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
}  // extern "C"
