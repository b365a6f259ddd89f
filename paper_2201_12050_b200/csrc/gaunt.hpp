// Translation-coefficient tables shared by the host producer (host/specfun.cpp)
// and the device M2L bank (csrc/far_bank.cu). Host-only, header-only.
//
// Restates /root/reference/proj/src/specfun.cpp: Wigner 3j by the Racah sum
// (:200-240), the translation coefficient (:242-262) and the M2L term lists of
// TranslationTable (:305-331): entry ((n,m),(n',m')) of the b x b K block is
// sum over l of c_l O_l^{m+m'}(delta; k), c_l = (2n'+1) trans_coeff(n,-m,n',m',l),
// l from |n-n'| to n+n' with n+n'+l even and |m+m'| <= l.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace fpbem_gaunt {

inline constexpr int flat(int n, int m) { return n * n + n + m; }
inline constexpr int coef_count(int n_t) { return (n_t + 1) * (n_t + 1); }

inline double sign_s(int m) { return (m >= 0 && (m & 1)) ? -1.0 : 1.0; }

inline const double* factorial_table() {
  static const std::vector<double> f = [] {
    std::vector<double> t(171);
    t[0] = 1.0;
    for (int i = 1; i < 171; ++i) t[i] = t[i - 1] * i;
    return t;
  }();
  return f.data();
}

inline double wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) {
  if (j1 < 0 || j2 < 0 || j3 < 0) return 0.0;
  if (std::abs(m1) > j1 || std::abs(m2) > j2 || std::abs(m3) > j3) return 0.0;
  if (m1 + m2 + m3 != 0) return 0.0;
  if (j3 < std::abs(j1 - j2) || j3 > j1 + j2) return 0.0;
  const double* f = factorial_table();
  const double tri = f[j1 + j2 - j3] * f[j1 - j2 + j3] * f[-j1 + j2 + j3] / f[j1 + j2 + j3 + 1];
  const double pre = tri * f[j1 + m1] * f[j1 - m1] * f[j2 + m2] * f[j2 - m2] * f[j3 + m3] * f[j3 - m3];
  const int tlo = std::max({0, j2 - j3 - m1, j1 - j3 + m2});
  const int thi = std::min({j1 + j2 - j3, j1 - m1, j2 + m2});
  double sum = 0.0;
  for (int t = tlo; t <= thi; ++t) {
    const double den = f[t] * f[j1 + j2 - j3 - t] * f[j1 - m1 - t] * f[j2 + m2 - t] * f[j3 - j2 + m1 + t] *
                       f[j3 - j1 - m2 + t];
    sum += ((t & 1) ? -1.0 : 1.0) / den;
  }
  return (((j1 - j2 - m3) & 1) ? -1.0 : 1.0) * std::sqrt(pre) * sum;
}

inline double trans_coeff(int n, int m, int np, int mp, int l) {
  const double w0 = wigner3j(n, l, np, 0, 0, 0);
  if (w0 == 0.0) return 0.0;
  const double w1 = wigner3j(n, l, np, -m, m - mp, mp);
  if (w1 == 0.0) return 0.0;
  const double re = (((l + n - np) % 4 + 4) % 4 == 0) ? 1.0 : -1.0;
  return re * (2.0 * l + 1.0) * sign_s(-m) * sign_s(m - mp) * sign_s(mp) * w0 * w1;
}

// M2L term lists in CSR form over the entries of a column-major b x b block
// (entry e = flat(n',m') * b + flat(n,m)): terms [start[e], start[e+1]) with
// O index flat(l, m + m') into the solid harmonics of degree <= 2 n_t.
struct M2lTerms {
  std::vector<int> start, o_index;
  std::vector<double> coef;
};

inline M2lTerms m2l_terms(int n_t) {
  const int p = coef_count(n_t);
  M2lTerms t;
  t.start.assign(static_cast<size_t>(p) * p + 1, 0);
  for (int np = 0; np <= n_t; ++np)
    for (int mp = -np; mp <= np; ++mp)
      for (int n = 0; n <= n_t; ++n)
        for (int m = -n; m <= n; ++m) {
          const size_t e = static_cast<size_t>(flat(np, mp)) * p + flat(n, m);
          const double w = 2.0 * np + 1.0;
          for (int l = std::abs(n - np); l <= n + np; ++l) {
            if ((n + np + l) & 1) continue;
            if (std::abs(m + mp) > l) continue;
            const double c = w * trans_coeff(n, -m, np, mp, l);
            if (c == 0.0) continue;
            t.o_index.push_back(flat(l, m + mp));
            t.coef.push_back(c);
          }
          t.start[e + 1] = static_cast<int>(t.coef.size());
        }
  return t;
}

}  // namespace fpbem_gaunt
