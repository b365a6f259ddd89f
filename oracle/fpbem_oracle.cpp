// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's periodic-FMBEM matvec hot path
// (arXiv 2201.12050, "fpbem"; /root/reference/proj). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this library, and only as the checker or the timed CPU baseline —
// never as the product path.
//
// The reference itself cannot be built in this image (Eigen 3.4, FFTW3,
// doctest, CLI11 and Boost.Multiprecision are absent), so this
// file restates the algorithms it calls, function by function:
//   * BlockToeplitzMatrix::matvec / expand_dense   src/assembly.cpp:62-105
//   * BlockHankelMatrix::matvec / expand_dense     src/assembly.cpp:152-203
//   * fft_friendly, embed_offset, circulant_embed  src/structured.cpp:26-61,
//                                                   include/fpbem/structured.hpp:15
//   * CirculantSpectrum ctor + matvec              src/structured.cpp:63-166
//   * mirror_permute / hankel_spectrum / matvec    src/structured.cpp:168-203
//   * FmmOperators::matvec                         src/fmm.cpp:246-271
//   * solver::gmres (+ checked_apply)              src/solver.cpp:13-123
// Third-party arithmetic restated: Eigen 3.4 GEMV / dot / norm / triangular
// solve (CMakeLists.txt:12) as plain loops; FFTW3's unnormalised multi-dim
// DFT (fftw_plan_many_dft, sign -1 forward / +1 backward; version unpinned,
// CMakeLists.txt:15-16) as an own mixed-radix FFT on the same [q][field]
// interleaved layout.
//
// Parity pinning: the known-answer tests of tests/test_structured.cpp,
// tests/test_solver.cpp, tests/test_assembly.cpp and the byte column of
// acceptance_bench/bench.csv are re-run against this file in
// tests/test_oracle.py (no stored vectors exist in the reference).
//
// Threading mirrors the reference's OpenMP placement (parallel over target
// cells in the Toeplitz product and over modes in the spectral product;
// FFT and level-1 vector operations single-threaded), so the timed
// cpu_baseline reproduces the reference's loop structure.

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace oracle {

using cd = std::complex<double>;

// ---------------------------------------------------------------------------
// error channel for the C-ABI

thread_local std::string g_last_error;

// ---------------------------------------------------------------------------
// block Toeplitz container (include/fpbem/assembly.hpp:24-50)

struct Toeplitz {
  int counts[3] = {1, 1, 1};
  int b = 0;                        // block_dim
  std::vector<int> offsets;         // 3 per stored block, insertion order
  const cd* blocks = nullptr;       // n_off * b * b, column-major each
  int n_off() const { return static_cast<int>(offsets.size() / 3); }
  int cells() const { return counts[0] * counts[1] * counts[2]; }
};

// y = sum_o S_o p_{t-o}; one GEMV per (target, offset) pair, in the stored
// offset order, parallel over target cells (src/assembly.cpp:62-84).
void toeplitz_matvec(const Toeplitz& t, const cd* p, cd* y) {
  const int b = t.b;
  const int m0 = t.counts[0], m1 = t.counts[1], m2 = t.counts[2];
  const long long ncell = static_cast<long long>(m0) * m1 * m2;
  const int no = t.n_off();
#pragma omp parallel for schedule(static)
  for (long long tc = 0; tc < ncell; ++tc) {
    const int tx = static_cast<int>(tc % m0);
    const int ty = static_cast<int>((tc / m0) % m1);
    const int tz = static_cast<int>(tc / (static_cast<long long>(m0) * m1));
    cd* out = y + tc * b;
    for (int i = 0; i < b; ++i) out[i] = 0.0;
    for (int s = 0; s < no; ++s) {
      const int sx = tx - t.offsets[3 * s], sy = ty - t.offsets[3 * s + 1],
                sz = tz - t.offsets[3 * s + 2];
      if (sx < 0 || sx >= m0 || sy < 0 || sy >= m1 || sz < 0 || sz >= m2) continue;
      const long long src = sx + static_cast<long long>(m0) * (sy + static_cast<long long>(m1) * sz);
      const cd* a = t.blocks + static_cast<size_t>(s) * b * b;
      const cd* x = p + src * b;
      // column-major GEMV, accumulated into a temporary then added
      // (Eigen's out.noalias() += A * x evaluates A*x then adds)
      std::vector<cd> tmp(b, cd(0.0, 0.0));
      for (int j = 0; j < b; ++j) {
        const cd xj = x[j];
        const cd* col = a + static_cast<size_t>(j) * b;
        for (int i = 0; i < b; ++i) tmp[i] += col[i] * xj;
      }
      for (int i = 0; i < b; ++i) out[i] += tmp[i];
    }
  }
}

// Dense expansion oracle (src/assembly.cpp:86-105). a is (n*b) x (n*b), column-major.
void toeplitz_expand_dense(const Toeplitz& t, cd* a) {
  const int b = t.b;
  const long long n = static_cast<long long>(t.cells()) * b;
  std::fill(a, a + n * n, cd(0.0, 0.0));
  const int* m = t.counts;
  for (int s = 0; s < t.n_off(); ++s) {
    const int ox = t.offsets[3 * s], oy = t.offsets[3 * s + 1], oz = t.offsets[3 * s + 2];
    const cd* blk = t.blocks + static_cast<size_t>(s) * b * b;
    for (int tz = 0; tz < m[2]; ++tz)
      for (int ty = 0; ty < m[1]; ++ty)
        for (int tx = 0; tx < m[0]; ++tx) {
          const int sx = tx - ox, sy = ty - oy, sz = tz - oz;
          if (sx < 0 || sx >= m[0] || sy < 0 || sy >= m[1] || sz < 0 || sz >= m[2]) continue;
          const long long tcell = tx + static_cast<long long>(m[0]) * (ty + m[1] * tz);
          const long long scell = sx + static_cast<long long>(m[0]) * (sy + m[1] * sz);
          for (int j = 0; j < b; ++j)
            for (int i = 0; i < b; ++i)
              a[(scell * b + j) * n + tcell * b + i] = blk[static_cast<size_t>(j) * b + i];
        }
  }
}

// ---------------------------------------------------------------------------
// block Hankel (mirrored level indexed by the cell-index sum;
// include/fpbem/assembly.hpp:52-75, src/assembly.cpp:152-203)

struct Hankel {
  int counts[3] = {1, 1, 1};
  int b = 0;
  int level = 2;
  std::vector<int> indices;  // 3 per block
  const cd* blocks = nullptr;
  int n_blk() const { return static_cast<int>(indices.size() / 3); }
};

void hankel_matvec_direct(const Hankel& h, const cd* p, cd* y) {
  const int b = h.b;
  const int* m = h.counts;
  const long long ncell = static_cast<long long>(m[0]) * m[1] * m[2];
#pragma omp parallel for schedule(static)
  for (long long tc = 0; tc < ncell; ++tc) {
    int t[3] = {static_cast<int>(tc % m[0]), static_cast<int>((tc / m[0]) % m[1]),
                static_cast<int>(tc / (static_cast<long long>(m[0]) * m[1]))};
    cd* out = y + tc * b;
    for (int i = 0; i < b; ++i) out[i] = 0.0;
    for (int s = 0; s < h.n_blk(); ++s) {
      int src[3];
      bool ok = true;
      for (int d = 0; d < 3 && ok; ++d) {
        src[d] = (d == h.level) ? h.indices[3 * s + d] - t[d] : t[d] - h.indices[3 * s + d];
        ok = src[d] >= 0 && src[d] < m[d];
      }
      if (!ok) continue;
      const long long sc = src[0] + static_cast<long long>(m[0]) * (src[1] + m[1] * src[2]);
      const cd* a = h.blocks + static_cast<size_t>(s) * b * b;
      std::vector<cd> tmp(b, cd(0.0, 0.0));
      for (int j = 0; j < b; ++j) {
        const cd xj = p[sc * b + j];
        for (int i = 0; i < b; ++i) tmp[i] += a[static_cast<size_t>(j) * b + i] * xj;
      }
      for (int i = 0; i < b; ++i) out[i] += tmp[i];
    }
  }
}

// ---------------------------------------------------------------------------
// FFT: own mixed-radix restatement of FFTW's unnormalised DFT.
// X[k] = sum_j x[j] exp(sign * 2 pi i j k / L), sign -1 forward, +1 backward.

int fft_friendly(int n) {  // src/structured.cpp:26-33
  for (int m = n;; ++m) {
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}

struct FftPlan {
  int n = 1;
  std::vector<int> radices;
  std::vector<cd> root;  // exp(sign*2*pi*i*j/n), j in [0, n)
  FftPlan(int len, int sign) : n(len) {
    int r = len;
    for (int f : {4, 2, 3, 5, 7})
      while (r % f == 0) {
        radices.push_back(f);
        r /= f;
      }
    for (int f = 11; r > 1; f += 2)
      while (r % f == 0) {
        radices.push_back(f);
        r /= f;
      }
    root.resize(len);
    for (int j = 0; j < len; ++j) {
      long double ang = static_cast<long double>(sign) * 2.0L * 3.141592653589793238462643383279502884L *
                        static_cast<long double>(j) / static_cast<long double>(len);
      root[j] = cd(static_cast<double>(std::cos(ang)), static_cast<double>(std::sin(ang)));
    }
  }
  // recursive decimation in time; in has stride `stride`, out is contiguous
  void rec(const cd* in, long long stride, cd* out, int len, size_t fi, int step,
           std::vector<cd>& scratch) const {
    if (len == 1) {
      out[0] = in[0];
      return;
    }
    const int r = radices[fi];
    const int m = len / r;
    for (int q = 0; q < r; ++q) rec(in + q * stride, stride * r, out + q * m, m, fi + 1, step * r, scratch);
    // X[k + m s] = sum_q W_len^{q (k + m s)} Y_q[k], W_len = root^step
    cd tmp[64];
    std::vector<cd> big;
    cd* t = tmp;
    if (r > 64) {
      big.resize(r);
      t = big.data();
    }
    for (int k = 0; k < m; ++k) {
      for (int s = 0; s < r; ++s) {
        cd acc(0.0, 0.0);
        for (int q = 0; q < r; ++q) {
          long long e = static_cast<long long>(q) * (k + static_cast<long long>(m) * s) % len;
          acc += out[q * m + k] * root[static_cast<size_t>(e * step)];
        }
        t[s] = acc;
      }
      for (int s = 0; s < r; ++s) out[k + m * s] = t[s];
    }
    (void)scratch;
  }
  void run(const cd* in, long long stride, cd* out) const {
    std::vector<cd> scratch;
    if (n == 1) {
      out[0] = in[0];
      return;
    }
    rec(in, stride, out, n, 0, 1, scratch);
  }
};

// In-place 3-D DFT over sizes {lx, ly, lz} (x fastest) of `howmany`
// interleaved fields: data[q * howmany + f] with q = (qz*ly + qy)*lx + qx.
// Same layout as fftw_plan_many_dft(3, {lz,ly,lx}, howmany, ..., stride
// howmany, dist 1) at src/structured.cpp:93-106.
void dft3(cd* data, const int l[3], int howmany, int sign) {
  const long long stride_axis[3] = {static_cast<long long>(howmany),
                                    static_cast<long long>(howmany) * l[0],
                                    static_cast<long long>(howmany) * l[0] * l[1]};
  for (int axis = 0; axis < 3; ++axis) {
    const int n = l[axis];
    if (n == 1) continue;
    FftPlan plan(n, sign);
    std::vector<cd> line(n), out(n);
    const long long total = static_cast<long long>(l[0]) * l[1] * l[2];
    const long long lines = total / n;
    for (long long li = 0; li < lines; ++li) {
      // decompose the line index into the two other axes
      long long base;
      if (axis == 0) {
        base = li * l[0];
      } else if (axis == 1) {
        long long qx = li % l[0], qz = li / l[0];
        base = qz * l[0] * l[1] + qx;
      } else {
        base = li;  // (qy, qx) plane index
      }
      const long long qstride = stride_axis[axis] / howmany;
      for (int f = 0; f < howmany; ++f) {
        for (int j = 0; j < n; ++j) line[j] = data[(base + j * qstride) * howmany + f];
        plan.run(line.data(), 1, out.data());
        for (int j = 0; j < n; ++j) data[(base + j * qstride) * howmany + f] = out[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// CirculantSpectrum (include/fpbem/structured.hpp:24-50; src/structured.cpp:63-166)

struct Spectrum {
  int counts[3] = {1, 1, 1};
  int sizes[3] = {1, 1, 1};
  int b = 0;
  std::vector<cd> lambda;  // q_total blocks of b*b, column-major
  long long q_total() const { return static_cast<long long>(sizes[0]) * sizes[1] * sizes[2]; }
};

void spectrum_sizes(const int counts[3], int sizes[3]) {
  for (int d = 0; d < 3; ++d) sizes[d] = counts[d] == 1 ? 1 : fft_friendly(2 * counts[d] - 1);
}

int find_offset(const Toeplitz& t, int ox, int oy, int oz) {
  for (int s = 0; s < t.n_off(); ++s)
    if (t.offsets[3 * s] == ox && t.offsets[3 * s + 1] == oy && t.offsets[3 * s + 2] == oz) return s;
  return -1;
}

// Build the spectrum of the circulant embedding; sizes either the
// reference's 7-smooth padding (sizes_in == nullptr) or caller-chosen
// lengths >= 2M-1 (SURVEY.md finding 7).
Spectrum build_spectrum(const Toeplitz& t, const int* sizes_in) {
  Spectrum sp;
  for (int d = 0; d < 3; ++d) sp.counts[d] = t.counts[d];
  if (sizes_in) {
    for (int d = 0; d < 3; ++d) sp.sizes[d] = sizes_in[d];
  } else {
    spectrum_sizes(sp.counts, sp.sizes);
  }
  for (int d = 0; d < 3; ++d)
    if (sp.sizes[d] < 2 * sp.counts[d] - 1 && !(sp.counts[d] == 1 && sp.sizes[d] == 1))
      throw std::invalid_argument("spectrum: embedding length must be >= 2M-1");
  sp.b = t.b;
  const size_t b2 = static_cast<size_t>(t.b) * t.b;
  sp.lambda.assign(sp.q_total() * b2, cd(0.0, 0.0));
  // slot q maps to offset q (q < M), q - L (q > L - M), else padding (src/structured.cpp:73-77)
  auto offset_of = [&](int q, int d, bool& valid) {
    valid = true;
    if (q < sp.counts[d]) return q;
    int o = q - sp.sizes[d];
    if (o > -sp.counts[d]) return o;
    valid = false;
    return 0;
  };
  long long q = 0;
  for (int qz = 0; qz < sp.sizes[2]; ++qz)
    for (int qy = 0; qy < sp.sizes[1]; ++qy)
      for (int qx = 0; qx < sp.sizes[0]; ++qx, ++q) {
        bool v0, v1, v2;
        int ox = offset_of(qx, 0, v0), oy = offset_of(qy, 1, v1), oz = offset_of(qz, 2, v2);
        if (!(v0 && v1 && v2)) continue;
        int s = find_offset(t, ox, oy, oz);
        if (s < 0) continue;
        std::memcpy(sp.lambda.data() + q * b2, t.blocks + s * b2, b2 * sizeof(cd));
      }
  dft3(sp.lambda.data(), sp.sizes, static_cast<int>(b2), -1);
  return sp;
}

// pad -> forward DFT -> per-mode block product -> backward DFT -> 1/q and
// truncate (src/structured.cpp:122-166). nrhs columns are applied one after
// another, exactly as repeated single-vector products.
void spectrum_matvec(const Spectrum& sp, const cd* p, cd* y) {
  const int b = sp.b;
  const int* m = sp.counts;
  const int* l = sp.sizes;
  const long long qt = sp.q_total();
  std::vector<cd> field(qt * b, cd(0.0, 0.0)), image(qt * b);
  for (int iz = 0; iz < m[2]; ++iz)
    for (int iy = 0; iy < m[1]; ++iy)
      for (int ix = 0; ix < m[0]; ++ix) {
        long long q = (static_cast<long long>(iz) * l[1] + iy) * l[0] + ix;
        long long cell = ix + static_cast<long long>(m[0]) * (iy + static_cast<long long>(m[1]) * iz);
        std::copy_n(p + cell * b, b, field.data() + q * b);
      }
  dft3(field.data(), l, b, -1);
  const size_t b2 = static_cast<size_t>(b) * b;
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < qt; ++q) {
    const cd* blk = sp.lambda.data() + q * b2;
    const cd* in = field.data() + q * b;
    cd* out = image.data() + q * b;
    for (int i = 0; i < b; ++i) out[i] = 0.0;
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) out[i] += blk[static_cast<size_t>(j) * b + i] * in[j];
  }
  dft3(image.data(), l, b, +1);
  const double scale = 1.0 / static_cast<double>(qt);
  for (int iz = 0; iz < m[2]; ++iz)
    for (int iy = 0; iy < m[1]; ++iy)
      for (int ix = 0; ix < m[0]; ++ix) {
        long long q = (static_cast<long long>(iz) * l[1] + iy) * l[0] + ix;
        long long cell = ix + static_cast<long long>(m[0]) * (iy + static_cast<long long>(m[1]) * iz);
        for (int c = 0; c < b; ++c) y[cell * b + c] = scale * image[q * b + c];
      }
}

// column reversal along one level (src/structured.cpp:168-183)
void mirror_permute(const int counts[3], int level, int b, const cd* p, cd* out) {
  const int* m = counts;
  for (int iz = 0; iz < m[2]; ++iz)
    for (int iy = 0; iy < m[1]; ++iy)
      for (int ix = 0; ix < m[0]; ++ix) {
        int src[3] = {ix, iy, iz};
        src[level] = m[level] - 1 - src[level];
        long long from = src[0] + static_cast<long long>(m[0]) * (src[1] + static_cast<long long>(m[1]) * src[2]);
        long long to = ix + static_cast<long long>(m[0]) * (iy + static_cast<long long>(m[1]) * iz);
        std::copy_n(p + from * b, b, out + to * b);
      }
}

// H P is block Toeplitz along the mirrored level with o = idx - (M - 1)
// (src/structured.cpp:185-198)
Spectrum hankel_spectrum(const Hankel& h) {
  Toeplitz t;
  for (int d = 0; d < 3; ++d) t.counts[d] = h.counts[d];
  t.b = h.b;
  t.offsets = h.indices;
  for (int s = 0; s < h.n_blk(); ++s) t.offsets[3 * s + h.level] -= h.counts[h.level] - 1;
  t.blocks = h.blocks;
  return build_spectrum(t, nullptr);
}

// ---------------------------------------------------------------------------
// FmmOperators::matvec (src/fmm.cpp:246-271)

struct Fmm {
  Toeplitz near;           // S
  int n_coef = 0;          // (n_t+1)^2
  const cd* u0 = nullptr;  // n_dof x n_coef column-major
  const cd* v0 = nullptr;  // n_coef x n_dof column-major
  Spectrum k;              // spectrum of K
  // optional half-space split (src/fmm.cpp:262-263, 269)
  bool has_image = false;
  int mirrored_level = -1;
  Spectrum k_image;  // spectrum of K_hat P
  Hankel s_hat;
};

void fmm_matvec(const Fmm& f, const cd* p, cd* y) {
  const int b = f.near.b;
  const int pc = f.n_coef;
  const long long ncell = f.near.cells();
  toeplitz_matvec(f.near, p, y);
  std::vector<cd> moments(ncell * pc), local(ncell * pc);
#pragma omp parallel for schedule(static)
  for (long long c = 0; c < ncell; ++c) {
    cd* mo = moments.data() + c * pc;
    for (int i = 0; i < pc; ++i) mo[i] = 0.0;
    for (int j = 0; j < b; ++j) {
      const cd pj = p[c * b + j];
      for (int i = 0; i < pc; ++i) mo[i] += f.v0[static_cast<size_t>(j) * pc + i] * pj;
    }
  }
  spectrum_matvec(f.k, moments.data(), local.data());
  if (f.has_image) {
    std::vector<cd> perm(ncell * pc), extra(ncell * pc);
    mirror_permute(f.k_image.counts, f.mirrored_level, pc, moments.data(), perm.data());
    spectrum_matvec(f.k_image, perm.data(), extra.data());
    for (long long i = 0; i < ncell * pc; ++i) local[i] += extra[i];
  }
#pragma omp parallel for schedule(static)
  for (long long c = 0; c < ncell; ++c) {
    std::vector<cd> tmp(b, cd(0.0, 0.0));
    for (int j = 0; j < pc; ++j) {
      const cd lj = local[c * pc + j];
      for (int i = 0; i < b; ++i) tmp[i] += f.u0[static_cast<size_t>(j) * b + i] * lj;
    }
    for (int i = 0; i < b; ++i) y[c * b + i] += tmp[i];
  }
  if (f.has_image) {
    std::vector<cd> extra(ncell * b);
    hankel_matvec_direct(f.s_hat, p, extra.data());
    for (long long i = 0; i < ncell * b; ++i) y[i] += extra[i];
  }
}

// ---------------------------------------------------------------------------
// restarted GMRES (include/fpbem/solver.hpp:14-33; src/solver.cpp:13-123)

using ApplyCb = int (*)(void* ctx, const cd* v, cd* w, long long n);

struct GmresResult {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
};

// Level-1 operations. By default single-threaded, like Eigen's level-1 code
// in the reference (Eigen parallelises only GEMM). CHECKER mode
// (oracle_set_level1_parallel) splits them into fixed chunks over the OpenMP
// threads with the partial sums combined in chunk order (deterministic for a
// fixed thread count): only for stated-size GMRES parity checks, never for the
// timed CPU baseline.
int g_level1_parallel = 0;

template <typename T, typename F>
T chunked_sum(long long n, F f) {
  if (!g_level1_parallel || n < (1 << 15)) return f(0LL, n);
#ifdef _OPENMP
  const int nt = omp_get_max_threads();
#else
  const int nt = 1;
#endif
  std::vector<T> part(nt, T(0));
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int c = 0; c < nt; ++c) part[c] = f(n * c / nt, n * (c + 1) / nt);
  T s(0);
  for (int c = 0; c < nt; ++c) s += part[c];
  return s;
}

template <typename F>
void chunked_for(long long n, F f) {
  if (!g_level1_parallel || n < (1 << 15)) {
    f(0LL, n);
    return;
  }
#pragma omp parallel for schedule(static)
  for (long long c = 0; c < 64; ++c) f(n * c / 64, n * (c + 1) / 64);
}

double norm2(const cd* v, long long n) {
  const double s = chunked_sum<double>(n, [&](long long lo, long long hi) {
    double t = 0.0;
    for (long long i = lo; i < hi; ++i) t += std::norm(v[i]);
    return t;
  });
  return std::sqrt(s);
}

// Eigen's x.dot(y) conjugates the first argument
cd dotc(const cd* a, const cd* b, long long n) {
  return chunked_sum<cd>(n, [&](long long lo, long long hi) {
    cd t(0.0, 0.0);
    for (long long i = lo; i < hi; ++i) t += std::conj(a[i]) * b[i];
    return t;
  });
}

// w -= h v
void axpy_sub(cd* w, cd h, const cd* v, long long n) {
  chunked_for(n, [&](long long lo, long long hi) {
    for (long long k = lo; k < hi; ++k) w[k] -= h * v[k];
  });
}

bool all_finite(const cd* v, long long n) {
  for (long long i = 0; i < n; ++i)
    if (!std::isfinite(v[i].real()) || !std::isfinite(v[i].imag())) return false;
  return true;
}

struct NonFinite : std::runtime_error {
  NonFinite() : std::runtime_error("gmres: operator returned a non-finite value") {}
};

void checked_apply(ApplyCb apply, void* ctx, const cd* v, cd* w, long long n) {  // :13-17
  if (apply(ctx, v, w, n) != 0) throw std::runtime_error("gmres: operator callback failed");
  if (!all_finite(w, n)) throw NonFinite();
}

GmresResult gmres(ApplyCb apply, void* actx, ApplyCb precond, void* pctx, const cd* b, cd* x_out,
                  long long n, double tol, int restart, int max_iter) {
  GmresResult rep;
  std::fill(x_out, x_out + n, cd(0.0, 0.0));
  std::vector<cd> tmpw(n);
  auto apply_eff = [&](const cd* v, cd* w) {
    if (precond) {
      checked_apply(apply, actx, v, tmpw.data(), n);
      checked_apply(precond, pctx, tmpw.data(), w, n);
    } else {
      checked_apply(apply, actx, v, w, n);
    }
  };
  std::vector<cd> b_eff(b, b + n);
  if (precond) checked_apply(precond, pctx, b, b_eff.data(), n);

  const double bnorm = norm2(b_eff.data(), n);
  if (bnorm == 0.0) {
    rep.converged = true;
    return rep;
  }
  const int m = std::max(1, restart);
  std::vector<cd> basis(static_cast<size_t>(n) * (m + 1));
  auto col = [&](int j) { return basis.data() + static_cast<size_t>(j) * n; };
  std::vector<cd> hess(static_cast<size_t>(m + 1) * m, cd(0.0, 0.0));  // column-major (m+1) x m
  auto H = [&](int i, int j) -> cd& { return hess[static_cast<size_t>(j) * (m + 1) + i]; };
  std::vector<cd> g(m + 1);
  std::vector<double> giv_c(m);
  std::vector<cd> giv_s(m);
  std::vector<cd> x(n, cd(0.0, 0.0)), r(b_eff), w(n);
  double rnorm = bnorm;

  while (rep.iterations < max_iter) {
    chunked_for(n, [&](long long lo, long long hi) {
      for (long long k = lo; k < hi; ++k) col(0)[k] = r[k] / rnorm;
    });
    std::fill(g.begin(), g.end(), cd(0.0, 0.0));
    g[0] = rnorm;
    int j = 0;
    for (; j < m && rep.iterations < max_iter; ++j) {
      apply_eff(col(j), w.data());
      const double pre_norm = norm2(w.data(), n);
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt (:58-62)
        cd hij = dotc(col(i), w.data(), n);
        H(i, j) = hij;
        axpy_sub(w.data(), hij, col(i), n);
      }
      if (norm2(w.data(), n) < 0.5 * pre_norm) {  // one reorthogonalisation pass (:63-69)
        for (int i = 0; i <= j; ++i) {
          cd corr = dotc(col(i), w.data(), n);
          H(i, j) += corr;
          axpy_sub(w.data(), corr, col(i), n);
        }
      }
      const double hlast = norm2(w.data(), n);
      H(j + 1, j) = hlast;
      if (hlast > 0.0)
        chunked_for(n, [&](long long lo, long long hi) {
          for (long long k = lo; k < hi; ++k) col(j + 1)[k] = w[k] / hlast;
        });
      for (int i = 0; i < j; ++i) {  // old rotations (:75-79)
        cd t = giv_c[i] * H(i, j) + giv_s[i] * H(i + 1, j);
        H(i + 1, j) = -std::conj(giv_s[i]) * H(i, j) + giv_c[i] * H(i + 1, j);
        H(i, j) = t;
      }
      const cd a = H(j, j);  // new rotation (:80-94)
      const double bb = std::abs(H(j + 1, j));
      const double denom = std::hypot(std::abs(a), bb);
      if (denom == 0.0) {
        giv_c[j] = 1.0;
        giv_s[j] = cd(0.0, 0.0);
      } else if (std::abs(a) == 0.0) {
        giv_c[j] = 0.0;
        giv_s[j] = cd(1.0, 0.0);
      } else {
        giv_c[j] = std::abs(a) / denom;
        giv_s[j] = (a / std::abs(a)) * std::conj(H(j + 1, j)) / denom;
      }
      H(j, j) = giv_c[j] * a + giv_s[j] * H(j + 1, j);
      H(j + 1, j) = cd(0.0, 0.0);
      const cd gj = g[j];
      g[j] = giv_c[j] * gj;
      g[j + 1] = -std::conj(giv_s[j]) * gj;

      ++rep.iterations;
      const double est = std::abs(g[j + 1]) / bnorm;
      rep.history.push_back(est);
      if (est <= tol || hlast == 0.0) {
        ++j;
        break;
      }
    }
    // upper-triangular solve of the j x j system, then x += V y (:109-110)
    std::vector<cd> y(j);
    for (int i = j - 1; i >= 0; --i) {
      cd s = g[i];
      for (int k = i + 1; k < j; ++k) s -= H(i, k) * y[k];
      y[i] = s / H(i, i);
    }
    for (int i = 0; i < j; ++i) {
      const cd* vi = col(i);
      const cd yi = y[i];
      chunked_for(n, [&](long long lo, long long hi) {
        for (long long k = lo; k < hi; ++k) x[k] += vi[k] * yi;
      });
    }
    apply_eff(x.data(), w.data());  // true residual (:111-112)
    chunked_for(n, [&](long long lo, long long hi) {
      for (long long k = lo; k < hi; ++k) r[k] = b_eff[k] - w[k];
    });
    rnorm = norm2(r.data(), n);
    if (rnorm / bnorm <= tol) {
      rep.converged = true;
      break;
    }
  }
  std::copy(x.begin(), x.end(), x_out);
  if (!rep.history.empty()) rep.converged = rep.converged || rnorm / bnorm <= tol;
  return rep;
}

}  // namespace oracle

// ---------------------------------------------------------------------------
// C-ABI for the test harness (ctypes). Complex numbers are interleaved
// (re, im) doubles, layout-identical to std::complex<double>.

using oracle::cd;

extern "C" {

const char* oracle_last_error() { return oracle::g_last_error.c_str(); }

int oracle_num_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_fft_friendly(int n) { return oracle::fft_friendly(n); }

// CHECKER mode of the GMRES level-1 operations (see chunked_sum); returns the previous setting
int oracle_set_level1_parallel(int on) {
  const int prev = oracle::g_level1_parallel;
  oracle::g_level1_parallel = on != 0;
  return prev;
}

static oracle::Toeplitz make_toeplitz(const int* counts, int b, int n_off, const int* offsets,
                                      const double* blocks) {
  oracle::Toeplitz t;
  for (int d = 0; d < 3; ++d) t.counts[d] = counts[d];
  t.b = b;
  t.offsets.assign(offsets, offsets + 3 * n_off);
  t.blocks = reinterpret_cast<const cd*>(blocks);
  return t;
}

int oracle_toeplitz_matvec(const int* counts, int b, int n_off, const int* offsets,
                           const double* blocks, const double* p, double* y) {
  try {
    oracle::toeplitz_matvec(make_toeplitz(counts, b, n_off, offsets, blocks),
                            reinterpret_cast<const cd*>(p), reinterpret_cast<cd*>(y));
    return 0;
  } catch (const std::exception& e) {
    oracle::g_last_error = e.what();
    return 1;
  }
}

int oracle_toeplitz_expand_dense(const int* counts, int b, int n_off, const int* offsets,
                                 const double* blocks, double* dense) {
  oracle::toeplitz_expand_dense(make_toeplitz(counts, b, n_off, offsets, blocks),
                                reinterpret_cast<cd*>(dense));
  return 0;
}

int oracle_hankel_matvec(const int* counts, int b, int level, int n_blk, const int* indices,
                         const double* blocks, const double* p, double* y) {
  oracle::Hankel h;
  for (int d = 0; d < 3; ++d) h.counts[d] = counts[d];
  h.b = b;
  h.level = level;
  h.indices.assign(indices, indices + 3 * n_blk);
  h.blocks = reinterpret_cast<const cd*>(blocks);
  oracle::hankel_matvec_direct(h, reinterpret_cast<const cd*>(p), reinterpret_cast<cd*>(y));
  return 0;
}

// sizes_out[3]; if lambda_out is null only the sizes are returned.
// sizes_in may be null (reference 7-smooth padding).
int oracle_spectrum_build(const int* counts, int b, int n_off, const int* offsets,
                          const double* blocks, const int* sizes_in, int* sizes_out,
                          double* lambda_out) {
  try {
    oracle::Toeplitz t = make_toeplitz(counts, b, n_off, offsets, blocks);
    if (!lambda_out) {
      if (sizes_in)
        for (int d = 0; d < 3; ++d) sizes_out[d] = sizes_in[d];
      else
        oracle::spectrum_sizes(t.counts, sizes_out);
      return 0;
    }
    oracle::Spectrum sp = oracle::build_spectrum(t, sizes_in);
    for (int d = 0; d < 3; ++d) sizes_out[d] = sp.sizes[d];
    std::memcpy(lambda_out, sp.lambda.data(), sp.lambda.size() * sizeof(cd));
    return 0;
  } catch (const std::exception& e) {
    oracle::g_last_error = e.what();
    return 1;
  }
}

static oracle::Spectrum make_spectrum(const int* counts, const int* sizes, int b, const double* lambda) {
  oracle::Spectrum sp;
  for (int d = 0; d < 3; ++d) {
    sp.counts[d] = counts[d];
    sp.sizes[d] = sizes[d];
  }
  sp.b = b;
  const cd* lam = reinterpret_cast<const cd*>(lambda);
  sp.lambda.assign(lam, lam + sp.q_total() * static_cast<long long>(b) * b);
  return sp;
}

int oracle_spectrum_matvec(const int* counts, const int* sizes, int b, const double* lambda,
                           const double* p, double* y) {
  oracle::spectrum_matvec(make_spectrum(counts, sizes, b, lambda), reinterpret_cast<const cd*>(p),
                          reinterpret_cast<cd*>(y));
  return 0;
}

int oracle_dft3(double* data, const int* sizes, int howmany, int sign) {
  oracle::dft3(reinterpret_cast<cd*>(data), sizes, howmany, sign);
  return 0;
}

int oracle_mirror_permute(const int* counts, int level, int b, const double* p, double* out) {
  oracle::mirror_permute(counts, level, b, reinterpret_cast<const cd*>(p), reinterpret_cast<cd*>(out));
  return 0;
}

// Operator handle: copies nothing large; the caller keeps the arrays alive.
struct oracle_fmm {
  oracle::Fmm f;
};

oracle_fmm* oracle_fmm_create(const int* counts, int n_dof, int n_coef, int n_near,
                              const int* near_offsets, const double* near_blocks, const double* u0,
                              const double* v0, const int* fft_sizes, const double* lambda) {
  auto* h = new oracle_fmm();
  h->f.near = make_toeplitz(counts, n_dof, n_near, near_offsets, near_blocks);
  h->f.n_coef = n_coef;
  h->f.u0 = reinterpret_cast<const cd*>(u0);
  h->f.v0 = reinterpret_cast<const cd*>(v0);
  h->f.k = make_spectrum(counts, fft_sizes, n_coef, lambda);
  return h;
}

// optional half-space split image pair (S_hat block Hankel, spectrum of K_hat P)
int oracle_fmm_set_image(oracle_fmm* h, int mirrored_level, int n_hat, const int* hat_indices,
                         const double* hat_blocks, const int* img_sizes, const double* img_lambda) {
  h->f.has_image = true;
  h->f.mirrored_level = mirrored_level;
  for (int d = 0; d < 3; ++d) h->f.s_hat.counts[d] = h->f.near.counts[d];
  h->f.s_hat.b = h->f.near.b;
  h->f.s_hat.level = mirrored_level;
  h->f.s_hat.indices.assign(hat_indices, hat_indices + 3 * n_hat);
  h->f.s_hat.blocks = reinterpret_cast<const cd*>(hat_blocks);
  h->f.k_image = make_spectrum(h->f.near.counts, img_sizes, h->f.n_coef, img_lambda);
  return 0;
}

void oracle_fmm_destroy(oracle_fmm* h) { delete h; }

// nrhs right-hand sides stored one after another (x[r*N + i]).
int oracle_fmm_matvec(const oracle_fmm* h, const double* p, double* y, int nrhs) {
  try {
    const long long n = static_cast<long long>(h->f.near.cells()) * h->f.near.b;
    for (int r = 0; r < nrhs; ++r)
      oracle::fmm_matvec(h->f, reinterpret_cast<const cd*>(p) + r * n, reinterpret_cast<cd*>(y) + r * n);
    return 0;
  } catch (const std::exception& e) {
    oracle::g_last_error = e.what();
    return 1;
  }
}

static int fmm_apply_cb(void* ctx, const cd* v, cd* w, long long) {
  oracle::fmm_matvec(static_cast<oracle_fmm*>(ctx)->f, v, w);
  return 0;
}

// returns 0 ok, 1 error, 2 non-finite operator output (runtime_error in the reference)
static int run_gmres(oracle::ApplyCb apply, void* actx, oracle::ApplyCb pre, void* pctx,
                     const double* b, double* x, long long n, double tol, int restart, int max_iter,
                     int* iterations, int* converged, double* history, int history_cap,
                     int* history_len) {
  try {
    oracle::GmresResult r = oracle::gmres(apply, actx, pre, pctx, reinterpret_cast<const cd*>(b),
                                          reinterpret_cast<cd*>(x), n, tol, restart, max_iter);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    int len = static_cast<int>(r.history.size());
    if (history_len) *history_len = len;
    if (history)
      for (int i = 0; i < std::min(len, history_cap); ++i) history[i] = r.history[i];
    return 0;
  } catch (const oracle::NonFinite& e) {
    oracle::g_last_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    oracle::g_last_error = e.what();
    return 1;
  }
}

int oracle_gmres_cb(oracle::ApplyCb apply, void* actx, oracle::ApplyCb pre, void* pctx,
                    const double* b, double* x, long long n, double tol, int restart, int max_iter,
                    int* iterations, int* converged, double* history, int history_cap,
                    int* history_len) {
  return run_gmres(apply, actx, pre, pctx, b, x, n, tol, restart, max_iter, iterations, converged,
                   history, history_cap, history_len);
}

int oracle_fmm_gmres(oracle_fmm* h, const double* b, double* x, double tol, int restart,
                     int max_iter, int* iterations, int* converged, double* history,
                     int history_cap, int* history_len) {
  const long long n = static_cast<long long>(h->f.near.cells()) * h->f.near.b;
  return run_gmres(fmm_apply_cb, h, nullptr, nullptr, b, x, n, tol, restart, max_iter, iterations,
                   converged, history, history_cap, history_len);
}

}  // extern "C"
