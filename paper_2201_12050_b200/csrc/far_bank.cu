// Device M2L bank: the b x b translation blocks K(delta) of the far-field
// offsets, for many translation vectors at once.
//
// Reference: TranslationTable::m2l (src/specfun.cpp:332-351), called once per
// far offset by assemble_periodic_fmm (src/fmm.cpp:180-191; image terms of a
// folded half space :186-190, split-half-space K_hat blocks :204-242):
//   K[(n,m),(n',m')] = sum_l c_l O_l^{m+m'}(delta; k),
//   O_l^mu = h_l(k r) Y_l^mu(theta, phi),  h_l = j_l + i y_l,
// Y without the Condon-Shortley phase, normalised by sqrt((l-|mu|)!/(l+|mu|)!)
// (src/specfun.cpp:12-160). The c_l term lists come from csrc/gaunt.hpp (the
// same code the host producer uses).
//
// One CTA per block: thread 0 evaluates the (2 n_t + 1)^2 singular solid
// harmonics (and those of the image vector) into shared memory with the host
// recurrences (Miller downward j_l, upward y_l, packed associated Legendre),
// then every thread sums the term lists of its block entries.
#include <cmath>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "gaunt.hpp"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {

constexpr int kMaxDeg = 2 * 15;  // 2 n_t for n_t <= 15 (b <= 256)
constexpr int kBankThreads = 128;

__device__ __forceinline__ int flat_nm(int n, int m) { return n * n + n + m; }

// out[flat(l, mu)] = h_l(k r) Y_l^mu(v), l <= n_max; work: 2 (n_max + 1) + (n_max + 1)(n_max + 2) / 2 doubles
__device__ void solid_singular(int n_max, double vx, double vy, double vz, double k, c64* out, double* work) {
  double* jv = work;
  double* yv = jv + (n_max + 1);
  double* p = yv + (n_max + 1);
  const double r = sqrt(vx * vx + vy * vy + vz * vz);
  const double x = k * r;
  // spherical Bessel j: Miller downward recurrence, normalised by j0 or j1
  const double j0 = sin(x) / x;
  if (n_max == 0) {
    jv[0] = j0;
  } else {
    const double xe = fmax(static_cast<double>(n_max), x);
    const int start = static_cast<int>(xe + 16.0 + 2.0 * sqrt(xe));
    double hi = 0.0, cur = 1.0e-300;
    for (int n = 0; n <= n_max; ++n) jv[n] = 0.0;
    for (int m = start; m >= 1; --m) {
      const double lo = (2.0 * m + 1.0) / x * cur - hi;
      hi = cur;
      cur = lo;
      if (fabs(cur) > 1.0e250) {
        cur *= 1.0e-250;
        hi *= 1.0e-250;
        for (int n = 0; n <= n_max; ++n) jv[n] *= 1.0e-250;
      }
      if (m - 1 <= n_max) jv[m - 1] = cur;
    }
    const double j1 = j0 / x - cos(x) / x;
    const double scale = fabs(j0) >= fabs(j1) ? j0 / jv[0] : j1 / jv[1];
    for (int n = 0; n <= n_max; ++n) jv[n] *= scale;
  }
  // spherical Bessel y: upward recurrence
  yv[0] = -cos(x) / x;
  if (n_max > 0) yv[1] = yv[0] / x - sin(x) / x;
  for (int n = 1; n < n_max; ++n) yv[n + 1] = (2.0 * n + 1.0) / x * yv[n] - yv[n - 1];
  // associated Legendre P_n^m(cos theta), packed at n(n+1)/2 + m
  const double ct = vz / r;
  const double st = hypot(vx, vy) / r;
  const double phi = st > 0.0 ? atan2(vy, vx) : 0.0;
  p[0] = 1.0;
  double pmm = 1.0;
  for (int m = 0; m <= n_max; ++m) {
    const int mm = m * (m + 1) / 2 + m;
    if (m > 0) {
      pmm *= (2.0 * m - 1.0) * st;
      p[mm] = pmm;
    }
    if (m < n_max) p[(m + 1) * (m + 2) / 2 + m] = (2.0 * m + 1.0) * ct * p[mm];
    for (int n = m + 2; n <= n_max; ++n)
      p[n * (n + 1) / 2 + m] =
          ((2.0 * n - 1.0) * ct * p[(n - 1) * n / 2 + m] - (n + m - 1.0) * p[(n - 2) * (n - 1) / 2 + m]) / (n - m);
  }
  // Y_n^m with e^{i m phi} by repeated multiplication, times h_n
  const c64 e1 = cmk(cos(phi), sin(phi));
  for (int n = 0; n <= n_max; ++n) {
    const c64 h = cmk(jv[n], yv[n]);
    out[flat_nm(n, 0)] = cmul(cmk(p[n * (n + 1) / 2], 0.0), h);
    double nrm = 1.0;
    c64 em = cmk(1.0, 0.0);
    for (int m = 1; m <= n; ++m) {
      em = cmul(em, e1);
      nrm /= sqrt(static_cast<double>((n - m + 1) * (n + m)));
      const double a = nrm * p[n * (n + 1) / 2 + m];
      const c64 y = cmk(a * em.x, a * em.y);
      out[flat_nm(n, m)] = cmul(y, h);
      out[flat_nm(n, -m)] = cmul(cmk(y.x, -y.y), h);
    }
  }
}

// out[s] = [K(delta_s)] + refl * K(image_s) P_axis, column-major b x b
//   P_axis: the mirror parity map (src/fmm.cpp:108-123) as a signed permutation
//   of columns: (K P)[:, flat(n, m)] = v K[:, flat(n, m')] with
//   axis 2: m' = m, v = (-1)^(n+m); axis 0/1: m' = -m, v = (-1)^m on axis 0 only
__global__ void __launch_bounds__(kBankThreads)
far_bank_kernel(int n_t, double k, int n_blk, const double* __restrict__ delta, const double* __restrict__ image,
                int parity_axis, c64 refl, const int* __restrict__ t_start, const int* __restrict__ t_o,
                const double* __restrict__ t_c, c64* __restrict__ out) {
  __shared__ c64 o_main[(kMaxDeg + 1) * (kMaxDeg + 1)];
  __shared__ c64 o_img[(kMaxDeg + 1) * (kMaxDeg + 1)];
  __shared__ double work[2 * (kMaxDeg + 1) + (kMaxDeg + 1) * (kMaxDeg + 2) / 2];
  const int s = blockIdx.x;
  const int p = (n_t + 1) * (n_t + 1);
  const int n_max = 2 * n_t;
  if (threadIdx.x == 0) {
    if (delta) solid_singular(n_max, delta[3 * s], delta[3 * s + 1], delta[3 * s + 2], k, o_main, work);
    if (image) solid_singular(n_max, image[3 * s], image[3 * s + 1], image[3 * s + 2], k, o_img, work);
  }
  __syncthreads();
  c64* blk = out + static_cast<long long>(s) * p * p;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    c64 acc = cmk(0.0, 0.0);
    if (delta)
      for (int t = t_start[e]; t < t_start[e + 1]; ++t) {
        const c64 o = o_main[t_o[t]];
        const double c = t_c[t];
        acc = cmk(acc.x + c * o.x, acc.y + c * o.y);
      }
    if (image) {
      const int col = e / p, row = e - col * p;
      int n = 0;
      while ((n + 1) * (n + 1) <= col) ++n;
      const int m = col - n * n - n;
      int mc;
      double v;
      if (parity_axis == 2) {
        mc = m;
        v = ((n + m) & 1) ? -1.0 : 1.0;
      } else {
        mc = -m;
        v = (parity_axis == 0 && (m & 1)) ? -1.0 : 1.0;
      }
      const int ei = flat_nm(n, mc) * p + row;
      c64 ki = cmk(0.0, 0.0);
      for (int t = t_start[ei]; t < t_start[ei + 1]; ++t) {
        const c64 o = o_img[t_o[t]];
        const double c = t_c[t];
        ki = cmk(ki.x + c * o.x, ki.y + c * o.y);
      }
      acc = cadd(acc, cscale(cmul(refl, ki), v));
    }
    blk[e] = acc;
  }
}

struct DeviceTerms {
  int* start = nullptr;
  int* o_index = nullptr;
  double* coef = nullptr;
};

// term lists per (device, n_t), uploaded once and kept for the process
cudaError_t device_terms(int device, int n_t, DeviceTerms* out) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, DeviceTerms> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({device, n_t});
  if (it != cache.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  const fpbem_gaunt::M2lTerms t = fpbem_gaunt::m2l_terms(n_t);
  DeviceTerms d;
  cudaError_t e = cudaMalloc(&d.start, t.start.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&d.o_index, (t.o_index.size() + 1) * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&d.coef, (t.coef.size() + 1) * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(d.start, t.start.data(), t.start.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !t.o_index.empty())
    e = cudaMemcpy(d.o_index, t.o_index.data(), t.o_index.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !t.coef.empty())
    e = cudaMemcpy(d.coef, t.coef.data(), t.coef.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d.start);
    cudaFree(d.o_index);
    cudaFree(d.coef);
    return e;
  }
  cache[{device, n_t}] = d;
  *out = d;
  return cudaSuccess;
}

}  // namespace

int far_bank_max_nt() { return kMaxDeg / 2; }

cudaError_t launch_far_bank(int device, int n_t, double k, int n_blk, const double* delta, const double* image,
                            int parity_axis, c64 refl, c64* out, cudaStream_t stream) {
  if (n_blk == 0) return cudaSuccess;
  DeviceTerms t;
  cudaError_t e = device_terms(device, n_t, &t);
  if (e != cudaSuccess) return e;
  far_bank_kernel<<<n_blk, kBankThreads, 0, stream>>>(n_t, k, n_blk, delta, image, parity_axis, refl, t.start,
                                                      t.o_index, t.coef, out);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
