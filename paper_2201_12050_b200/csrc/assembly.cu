// Near-field block assembly on the device.
//
// One thread per matrix entry (target collocation point i, source element j,
// block slot s): the Burton-Miller collocation entry of
// src/assembly.cpp:214-239 (bm_entry / interaction_block) with the quadrature
// of src/kernels.cpp:98-261 — 6x6 Gauss tensor rule on the bilinear element
// map, 4-fold adaptive subdivision (depth <= 6) when the collocation point is
// closer than 3 element diameters, and for the self entry the closed-form
// planar static parts plus the order-8 polar (Duffy) fan for the smooth
// remainders. Triangles are quads with the fourth corner collapsed, as on the
// host (paper_2201_12050_b200/host/kernels.cpp). A slot carries a target
// shift, a source shift, an optional mirror of the source element (half-space
// images: folded Toeplitz terms and the block-Hankel S_hat) and a complex
// scale (the reflection coefficient); "accumulate" adds into the output.
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace fpbem_cu {

namespace {

constexpr double kPiD = 3.14159265358979323846;
constexpr int kRegular = 6;
constexpr int kSelf = 8;
constexpr double kNear = 3.0;
constexpr int kMaxDepth = 6;

__constant__ double c_gx6[kRegular], c_gw6[kRegular], c_gx8[kSelf], c_gw8[kSelf];

struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 p3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ P3 operator+(P3 a, P3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ P3 operator-(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ P3 operator*(double s, P3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot3(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ P3 cross3(P3 a, P3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double len3(P3 a) { return sqrt(dot3(a, a)); }

struct Quad {
  P3 c[4];
};

struct Elem {
  Quad q;
  P3 cen, nrm;
  double diam;
  c64 beta;
};

// sum over the 6x6 tensor rule of one bilinear patch of the BM integrands
__device__ void tensor_accum(const Quad& q, P3 x, P3 nx, P3 ny, double k, c64 alpha, c64& h, c64& g) {
  const double nxny = dot3(nx, ny);
  for (int i = 0; i < kRegular; ++i) {
    const double u = c_gx6[i];
    for (int jj = 0; jj < kRegular; ++jj) {
      const double v = c_gx6[jj];
      const double s0 = 0.25 * (1 - u) * (1 - v), s1 = 0.25 * (1 + u) * (1 - v), s2 = 0.25 * (1 + u) * (1 + v),
                   s3 = 0.25 * (1 - u) * (1 + v);
      const P3 y = s0 * q.c[0] + s1 * q.c[1] + s2 * q.c[2] + s3 * q.c[3];
      const P3 du = 0.25 * ((1 - v) * (q.c[1] - q.c[0]) + (1 + v) * (q.c[2] - q.c[3]));
      const P3 dv = 0.25 * ((1 - u) * (q.c[3] - q.c[0]) + (1 + u) * (q.c[2] - q.c[1]));
      const double w = c_gw6[i] * c_gw6[jj] * len3(cross3(du, dv));
      const P3 d = x - y;
      const double r = len3(d);
      const double inv = 1.0 / r;
      const double cx = dot3(d, nx) * inv, cy = dot3(d, ny) * inv;
      double sn, cs;
      sincos(k * r, &sn, &cs);
      const c64 gg = cmk(cs * inv / (4.0 * kPiD), sn * inv / (4.0 * kPiD));  // e^{ikr}/(4 pi r)
      const c64 qd = cmk(-inv, k);                                             // dG/dr = q G
      const c64 qg = cmul(qd, gg);
      const c64 dgdny = cscale(qg, -cy);
      const c64 dgdnx = cscale(qg, cx);
      // d2G = G (k^2 + 3ik/r - 3/r^2) cx cy - G q / r nx.ny
      const c64 f1 = cmk(k * k - 3.0 * inv * inv, 3.0 * k * inv);
      const c64 d2g = csub(cscale(cmul(gg, f1), cx * cy), cscale(qg, inv * nxny));
      h = cadd(h, cscale(cadd(dgdny, cmul(alpha, d2g)), w));
      g = cadd(g, cscale(cadd(gg, cmul(alpha, dgdnx)), w));
    }
  }
}

// influence of one element seen from x: tensor rule, or adaptive quartering
// (depth-first, the host's recursion order) when x is near (kernels.cpp:98-128, 214-226)
__device__ void influence(const Elem& e, P3 x, P3 nx, double k, c64 alpha, c64& h, c64& g) {
  h = g = cmk(0.0, 0.0);
  if (len3(x - e.cen) >= kNear * e.diam) {
    tensor_accum(e.q, x, nx, e.nrm, k, alpha, h, g);
    return;
  }
  Quad stack[3 * kMaxDepth + 1];
  int depth[3 * kMaxDepth + 1];
  int top = 0;
  stack[0] = e.q;
  depth[0] = kMaxDepth;
  while (top >= 0) {
    const Quad q = stack[top];
    const int dep = depth[top];
    --top;
    const P3 mid = 0.25 * (q.c[0] + q.c[1] + q.c[2] + q.c[3]);
    const double diam = fmax(len3(q.c[2] - q.c[0]), len3(q.c[3] - q.c[1]));
    if (dep <= 0 || len3(x - mid) >= kNear * diam) {
      tensor_accum(q, x, nx, e.nrm, k, alpha, h, g);
      continue;
    }
    const P3 m01 = 0.5 * (q.c[0] + q.c[1]), m12 = 0.5 * (q.c[1] + q.c[2]), m23 = 0.5 * (q.c[2] + q.c[3]),
             m30 = 0.5 * (q.c[3] + q.c[0]);
    // push in reverse so the children are visited in the host's order
    stack[++top] = Quad{{m30, mid, m23, q.c[3]}};
    depth[top] = dep - 1;
    stack[++top] = Quad{{mid, m12, q.c[2], m23}};
    depth[top] = dep - 1;
    stack[++top] = Quad{{m01, q.c[1], m12, mid}};
    depth[top] = dep - 1;
    stack[++top] = Quad{{q.c[0], m01, mid, m30}};
    depth[top] = dep - 1;
  }
}

__device__ c64 sl_remainder(double k, double r) {  // (e^{ikr} - 1)/(4 pi r)
  const double kr = k * r;
  if (kr >= 0.5) {
    double sn, cs;
    sincos(kr, &sn, &cs);
    return cmk((cs - 1.0) / (4.0 * kPiD * r), sn / (4.0 * kPiD * r));
  }
  c64 sum = cmk(0.0, 0.0), pw = cmk(1.0, 0.0);
  const c64 ikr = cmk(0.0, kr);
  double fact = 1.0;
  for (int j = 1; j <= 24; ++j) {
    fact *= j;
    sum = cadd(sum, cscale(pw, 1.0 / fact));
    pw = cmul(pw, ikr);
  }
  return cmul(cmk(0.0, k / (4.0 * kPiD)), sum);
}

__device__ c64 hyper_remainder(double k, double r) {  // [e^{ikr}(1 - ikr) - 1 - (kr)^2/2] / (4 pi r^3)
  const double kr = k * r;
  if (kr >= 0.5) {
    double sn, cs;
    sincos(kr, &sn, &cs);
    const c64 e = cmk(cs, sn);
    const c64 t = cmul(e, cmk(1.0, -kr));
    const double den = 4.0 * kPiD * r * r * r;
    return cmk((t.x - 1.0 - 0.5 * kr * kr) / den, t.y / den);
  }
  c64 sum = cmk(0.0, 0.0);
  const c64 ik = cmk(0.0, k);
  c64 pw = cmul(cmul(ik, ik), ik);
  double fact = 2.0;
  for (int j = 3; j <= 26; ++j) {
    fact *= j;
    sum = cadd(sum, cscale(pw, (1.0 - j) / fact));
    pw = cmul(pw, cmk(0.0, k * r));
  }
  return cscale(sum, 1.0 / (4.0 * kPiD));
}

// self entry at the element's own centroid (kernels.cpp:228-261)
__device__ void influence_self(const Elem& e, double k, c64 alpha, c64& h, c64& g) {
  const P3 x = e.cen;
  P3 ng = cross3(e.q.c[2] - e.q.c[0], e.q.c[3] - e.q.c[1]);
  ng = (1.0 / len3(ng)) * ng;
  double sl0 = 0.0, hyp0 = 0.0;
  for (int edge = 0; edge < 4; ++edge) {
    const P3 a = e.q.c[edge] - x, b = e.q.c[(edge + 1) % 4] - x;
    const P3 ab = b - a;
    const double len = len3(ab);
    if (len == 0.0) continue;
    const P3 t = (1.0 / len) * ab;
    const double sa = dot3(a, t), sb = dot3(b, t), da = len3(a), db = len3(b);
    const double hh = dot3(ng, cross3(a, b)) / len;
    sl0 += hh * log((db + sb) / (da + sa));
    hyp0 -= (sb / db - sa / da) / hh;
  }
  sl0 /= 4.0 * kPiD;
  hyp0 /= 4.0 * kPiD;
  c64 g_rem = cmk(0.0, 0.0), h_rem = cmk(0.0, 0.0);
  for (int edge = 0; edge < 4; ++edge) {
    const P3 a = e.q.c[edge] - x, b = e.q.c[(edge + 1) % 4] - x;
    if (len3(b - a) == 0.0) continue;
    const double jac2 = dot3(cross3(a, b), ng);
    for (int i = 0; i < kSelf; ++i) {
      const double u = 0.5 * (c_gx8[i] + 1.0);
      for (int jj = 0; jj < kSelf; ++jj) {
        const double v = 0.5 * (c_gx8[jj] + 1.0);
        const P3 y = u * ((1.0 - v) * a + v * b);
        const double wq = 0.25 * c_gw8[i] * c_gw8[jj] * u * jac2;
        const double rr = len3(y);
        g_rem = cadd(g_rem, cscale(sl_remainder(k, rr), wq));
        h_rem = cadd(h_rem, cscale(hyper_remainder(k, rr), wq));
      }
    }
  }
  g = cadd(cmk(sl0, 0.0), g_rem);
  h = cmul(alpha, cadd(cmk(hyp0 + 0.5 * k * k * sl0, 0.0), h_rem));
}

__device__ __forceinline__ P3 load_p3(const double* a, long long i) { return p3(a[3 * i], a[3 * i + 1], a[3 * i + 2]); }

__device__ __forceinline__ P3 mirror_p(P3 p, int axis, double off) {
  if (axis == 0) p.x = 2.0 * off - p.x;
  if (axis == 1) p.y = 2.0 * off - p.y;
  if (axis == 2) p.z = 2.0 * off - p.z;
  return p;
}

// entries of block slot s: out[s][j*n + i] (+)= scale_s * bm_entry(src_j', x_i + tshift_s)
__global__ void __launch_bounds__(128)
assemble_kernel(const double* __restrict__ corners, const int* __restrict__ nv, const double* __restrict__ cen,
                const double* __restrict__ nrm, const double* __restrict__ diam, const c64* __restrict__ beta, int n,
                const AssemblySlot* __restrict__ slots, double k, c64 alpha, int hs_axis, double hs_offset,
                c64* __restrict__ out, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const AssemblySlot sl = slots[blockIdx.z];
  if (i >= n) return;
  // source element j, shifted, optionally mirrored (geometry.cpp:164-178)
  Elem e;
  const P3 ss = p3(sl.sshift[0], sl.sshift[1], sl.sshift[2]);
  P3 c[4];
  for (int a = 0; a < 4; ++a) c[a] = load_p3(corners, 4LL * j + a) + ss;
  e.cen = load_p3(cen, j) + ss;
  e.nrm = load_p3(nrm, j);
  e.diam = diam[j];
  e.beta = beta ? beta[j] : cmk(0.0, 0.0);
  if (sl.mirror) {
    for (int a = 0; a < 4; ++a) c[a] = mirror_p(c[a], hs_axis, hs_offset);
    e.cen = mirror_p(e.cen, hs_axis, hs_offset);
    if (hs_axis == 0) e.nrm.x = -e.nrm.x;
    if (hs_axis == 1) e.nrm.y = -e.nrm.y;
    if (hs_axis == 2) e.nrm.z = -e.nrm.z;
    if (nv[j] == 3) {  // (c0, c2, c1, c1)
      e.q = Quad{{c[0], c[2], c[1], c[1]}};
    } else {           // (c0, c3, c2, c1)
      e.q = Quad{{c[0], c[3], c[2], c[1]}};
    }
  } else {
    e.q = Quad{{c[0], c[1], c[2], c[3]}};
  }
  const P3 x = load_p3(cen, i) + p3(sl.tshift[0], sl.tshift[1], sl.tshift[2]);
  const P3 nx = load_p3(nrm, i);
  const c64 ikb = cmul(cmk(0.0, k), e.beta);
  c64 h, g, val;
  if (sl.self && i == j) {
    influence_self(e, k, alpha, h, g);
    // 0.5 + 0.5 alpha ikb + h - ikb g (assembly.cpp:217-219)
    val = cadd(cadd(cmk(0.5, 0.0), cscale(cmul(alpha, ikb), 0.5)), csub(h, cmul(ikb, g)));
  } else {
    influence(e, x, nx, k, alpha, h, g);
    val = csub(h, cmul(ikb, g));
  }
  val = cmul(sl.scale, val);
  c64* dst = out + (static_cast<long long>(blockIdx.z) * n + j) * n + i;
  *dst = accumulate ? cadd(*dst, val) : val;
}

}  // namespace

cudaError_t assembly_set_rules(const double* x6, const double* w6, const double* x8, const double* w8) {
  cudaError_t e = cudaMemcpyToSymbol(c_gx6, x6, sizeof(double) * kRegular);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_gw6, w6, sizeof(double) * kRegular);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_gx8, x8, sizeof(double) * kSelf);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_gw8, w8, sizeof(double) * kSelf);
  return e;
}

cudaError_t launch_assemble(const double* corners, const int* nv, const double* cen, const double* nrm,
                            const double* diam, const c64* beta, int n, const AssemblySlot* slots, int n_slots,
                            double k, c64 alpha, int hs_axis, double hs_offset, c64* out, bool accumulate,
                            cudaStream_t stream) {
  if (n_slots == 0 || n == 0) return cudaSuccess;
  dim3 grid((n + 127) / 128, n, n_slots);
  assemble_kernel<<<grid, 128, 0, stream>>>(corners, nv, cen, nrm, diam, beta, n, slots, k, alpha, hs_axis,
                                            hs_offset, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace fpbem_cu
