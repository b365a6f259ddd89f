// Host half of one restarted-GMRES cycle (src/solver.cpp:74-110), shared by
// the device solvers (gmres.cu, gmres_dist.cu): the Hessenberg column j is
// rotated by the accumulated Givens rotations, a new rotation zeroes its
// sub-diagonal, g carries the residual estimate, solve() back-substitutes
// y = triu(H_jj)^{-1} g.
#pragma once

#include <cmath>
#include <complex>
#include <vector>

namespace fpbem_cu {

struct GmresCycle {
  using cd = std::complex<double>;
  int m;
  std::vector<cd> H;  // (m + 1) x m, column-major
  std::vector<cd> g;
  std::vector<double> gc;
  std::vector<cd> gs;

  explicit GmresCycle(int m_) : m(m_), H(static_cast<size_t>(m_ + 1) * m_), g(m_ + 1), gc(m_), gs(m_) {}

  cd& h(int i, int j) { return H[static_cast<size_t>(j) * (m + 1) + i]; }

  // new cycle from residual norm rnorm (g = rnorm e_1)
  void start(double rnorm) {
    std::fill(g.begin(), g.end(), cd(0, 0));
    g[0] = rnorm;
  }

  // column j holds the projections h(0..j, j) and h(j+1, j) = ||w||: apply
  // the old rotations (:75-79), make and apply the new one (:80-94), update g
  // (:95-97); returns |g[j+1]|, the unscaled residual estimate
  double rotate(int j) {
    for (int i = 0; i < j; ++i) {
      const cd t = gc[i] * h(i, j) + gs[i] * h(i + 1, j);
      h(i + 1, j) = -std::conj(gs[i]) * h(i, j) + gc[i] * h(i + 1, j);
      h(i, j) = t;
    }
    const cd a = h(j, j);
    const double bb = std::abs(h(j + 1, j));
    const double denom = std::hypot(std::abs(a), bb);
    if (denom == 0.0) {
      gc[j] = 1.0;
      gs[j] = cd(0, 0);
    } else if (std::abs(a) == 0.0) {
      gc[j] = 0.0;
      gs[j] = cd(1, 0);
    } else {
      gc[j] = std::abs(a) / denom;
      gs[j] = (a / std::abs(a)) * std::conj(h(j + 1, j)) / denom;
    }
    h(j, j) = gc[j] * a + gs[j] * h(j + 1, j);
    h(j + 1, j) = cd(0, 0);
    const cd gj = g[j];
    g[j] = gc[j] * gj;
    g[j + 1] = -std::conj(gs[j]) * gj;
    return std::abs(g[j + 1]);
  }

  // y = triu(H(0..j-1, 0..j-1))^{-1} g(0..j-1)   (:109)
  std::vector<cd> solve(int j) {
    std::vector<cd> y(j);
    for (int i = j - 1; i >= 0; --i) {
      cd acc = g[i];
      for (int k = i + 1; k < j; ++k) acc -= h(i, k) * y[k];
      y[i] = acc / h(i, i);
    }
    return y;
  }
};

}  // namespace fpbem_cu
