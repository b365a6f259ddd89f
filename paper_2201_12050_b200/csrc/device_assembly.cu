// C-ABI implementation, part 3: device assembly of the near-field blocks
// (interaction_block, src/assembly.cpp:214-239), the M2L bank
// (TranslationTable::m2l, src/specfun.cpp:332-351) and field evaluation
// (postproc::evaluate_field, src/postproc.cpp:39-62).
#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "handle.cuh"

using namespace fpbem_cu;

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

extern "C" {

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

}  // extern "C"
