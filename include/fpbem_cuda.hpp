// fpbem_cuda.hpp — header-only C++ shim over the C-ABI (fpbem_cuda.h).
//
// What a maintainer drops into the reference's make_backend
// (/root/reference/proj/src/scene.cpp:323-327): an RAII operator handle whose
// apply() has the semantics of FmmOperators::matvec (src/fmm.cpp:246-271)
// and a gmres() with those of solver::gmres (src/solver.cpp:21-123). C error
// codes become the reference's exceptions: FPBEM_CU_EDIM ->
// std::invalid_argument, everything else -> std::runtime_error (the
// non-finite case carries the reference's message, src/solver.cpp:15).
//
// Vec is any contiguous std::complex<double> container with data()/size()
// and a size constructor (Eigen::VectorXcd, std::vector<std::complex<double>>).
#ifndef FPBEM_CUDA_HPP
#define FPBEM_CUDA_HPP

#include <complex>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "fpbem_cuda.h"

namespace fpbem_cuda {

inline void throw_on(int rc) {
  if (rc == FPBEM_CU_OK) return;
  std::string msg = fpbem_cu_last_error();
  if (rc == FPBEM_CU_EDIM) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct SolveReport {  // include/fpbem/solver.hpp:14-19
  std::vector<std::complex<double>> solution;
  std::vector<double> residual_history;
  int iterations = 0;
  bool converged = false;
};

class DeviceFmm {
 public:
  DeviceFmm(const fpbem_cu_fmm_desc& desc, int device = 0) { throw_on(fpbem_cu_fmm_create(&desc, device, &op_)); }
  ~DeviceFmm() { fpbem_cu_fmm_destroy(op_); }
  DeviceFmm(const DeviceFmm&) = delete;
  DeviceFmm& operator=(const DeviceFmm&) = delete;

  fpbem_cu_op* handle() const { return op_; }

  std::size_t stored_bytes() const {  // FmmOperators::stored_bytes
    std::size_t b = 0;
    throw_on(fpbem_cu_fmm_bytes(op_, &b));
    return b;
  }

  // the near-field path chosen at create (FPBEM_CU_NEAR_DIRECT or _LATTICE) and the
  // Fourier modes per stored block (1 unless cell symmetries were verified)
  int near_path(int* modes_per_block = nullptr) const {
    int path = 0, sizes[3], mpb = 1, mask = 0;
    std::size_t bytes = 0;
    double dev = 0.0;
    throw_on(fpbem_cu_fmm_near_path(op_, &path, sizes, &bytes, &mpb, &mask, &dev));
    if (modes_per_block) *modes_per_block = mpb;
    return path;
  }

  // y = A p (FmmOperators::matvec): host buffers, synchronous
  template <typename Vec>
  Vec apply(const Vec& p, int nrhs = 1) const {
    Vec y(p.size());
    throw_on(fpbem_cu_fmm_apply(op_, reinterpret_cast<const fpbem_c64*>(p.data()),
                                reinterpret_cast<fpbem_c64*>(y.data()), nrhs, FPBEM_CU_PTR_HOST));
    return y;
  }

  // solver::gmres(apply, b, {tol, restart, max_iter}) with the Krylov basis in HBM
  template <typename Vec>
  SolveReport gmres(const Vec& b, double tol = 1e-4, int restart = 100, int max_iter = 1000) const {
    SolveReport rep;
    rep.solution.resize(static_cast<std::size_t>(b.size()));
    std::vector<double> hist(static_cast<std::size_t>(max_iter > 0 ? max_iter : 1));
    int its = 0, conv = 0, len = 0;
    throw_on(fpbem_cu_gmres(op_, reinterpret_cast<const fpbem_c64*>(b.data()),
                            reinterpret_cast<fpbem_c64*>(rep.solution.data()), 1, tol, restart, max_iter,
                            FPBEM_CU_PTR_HOST, &its, &conv, hist.data(), static_cast<int>(hist.size()), &len));
    rep.iterations = its;
    rep.converged = conv != 0;
    rep.residual_history.assign(hist.begin(), hist.begin() + len);
    return rep;
  }

 private:
  fpbem_cu_op* op_ = nullptr;
};

}  // namespace fpbem_cuda

#endif  // FPBEM_CUDA_HPP
