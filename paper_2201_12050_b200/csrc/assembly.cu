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
constexpr int kFieldThreads = 128;
constexpr int kFieldPerThread = 8;

__constant__ double c_gx6[kRegular], c_gw6[kRegular], c_gx8[kSelf], c_gw8[kSelf];

struct P3 {
  double x, y, z;
};
__host__ __device__ __forceinline__ P3 p3(double x, double y, double z) { return {x, y, z}; }
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
// (kBM = false: the plain layer potentials, h = int dG/dn_y, g = int G, as the
// representation formula of src/postproc.cpp:18-35 needs them)
template <bool kBM = true>
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
      if (!kBM) {
        h = cadd(h, cscale(dgdny, w));
        g = cadd(g, cscale(gg, w));
        continue;
      }
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
template <bool kBM = true>
__device__ void influence(const Elem& e, P3 x, P3 nx, double k, c64 alpha, c64& h, c64& g) {
  h = g = cmk(0.0, 0.0);
  if (len3(x - e.cen) >= kNear * e.diam) {
    tensor_accum<kBM>(e.q, x, nx, e.nrm, k, alpha, h, g);
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
      tensor_accum<kBM>(q, x, nx, e.nrm, k, alpha, h, g);
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

// element j of the replicated mesh (cell-major, x fastest; src/geometry.cpp
// replicate): the unit-cell element j % n shifted by the lattice vector of cell
// j / n, optionally mirrored (mirror_mesh: mirrored corners, reversed loop,
// mirrored normal)
__device__ Elem full_element(const double* __restrict__ corners, const int* __restrict__ nv,
                             const double* __restrict__ cen, const double* __restrict__ nrm,
                             const double* __restrict__ diam, const c64* __restrict__ beta, int n, int cx, int cy,
                             P3 pitch, long long j, bool mirror, int hs_axis, double hs_offset) {
  const long long cell = j / n;
  const int e = static_cast<int>(j - cell * n);
  const int ix = static_cast<int>(cell % cx), iy = static_cast<int>((cell / cx) % cy),
            iz = static_cast<int>(cell / (static_cast<long long>(cx) * cy));
  const P3 sh = p3(ix * pitch.x, iy * pitch.y, iz * pitch.z);
  Elem el;
  P3 c[4];
  for (int a = 0; a < 4; ++a) c[a] = load_p3(corners, 4LL * e + a) + sh;
  el.cen = load_p3(cen, e) + sh;
  el.nrm = load_p3(nrm, e);
  el.diam = diam[e];
  el.beta = beta ? beta[e] : cmk(0.0, 0.0);
  if (mirror) {
    for (int a = 0; a < 4; ++a) c[a] = mirror_p(c[a], hs_axis, hs_offset);
    el.cen = mirror_p(el.cen, hs_axis, hs_offset);
    if (hs_axis == 0) el.nrm.x = -el.nrm.x;
    if (hs_axis == 1) el.nrm.y = -el.nrm.y;
    if (hs_axis == 2) el.nrm.z = -el.nrm.z;
    el.q = nv[e] == 3 ? Quad{{c[0], c[2], c[1], c[1]}} : Quad{{c[0], c[3], c[2], c[1]}};
  } else {
    el.q = Quad{{c[0], c[1], c[2], c[3]}};
  }
  return el;
}

// representation-formula contribution of one element (postproc.cpp:18-35):
// int [-dG/dn_y p + G i k beta p]
__device__ __forceinline__ c64 field_contribution(const Elem& e, P3 x, double k, c64 pressure) {
  c64 h, g;
  influence<false>(e, x, p3(0.0, 0.0, 1.0), k, cmk(0.0, 0.0), h, g);
  const c64 ikb_p = cmul(cmul(cmk(0.0, k), e.beta), pressure);
  return cadd(cmul(csub(cmk(0.0, 0.0), h), pressure), cmul(g, ikb_p));
}

// partial[chunk][pt] = sum over the chunk's elements of the contributions at
// point pt (+ reflection x the mirrored elements'); fixed order: each thread
// sums its strided elements, then a fixed tree over the CTA
__global__ void __launch_bounds__(kFieldThreads)
field_kernel(const double* __restrict__ corners, const int* __restrict__ nv, const double* __restrict__ cen,
             const double* __restrict__ nrm, const double* __restrict__ diam, const c64* __restrict__ beta, int n,
             int cx, int cy, P3 pitch, long long n_total, const c64* __restrict__ sol, const double* __restrict__ pts,
             int n_pts, double k, int with_image, int hs_axis, double hs_offset, c64 refl,
             c64* __restrict__ partial) {
  __shared__ c64 red[kFieldThreads];
  const int pt = blockIdx.y;
  const P3 x = load_p3(pts, pt);
  const long long j0 = static_cast<long long>(blockIdx.x) * kFieldThreads * kFieldPerThread;
  c64 acc = cmk(0.0, 0.0);
  for (int u = 0; u < kFieldPerThread; ++u) {
    const long long j = j0 + static_cast<long long>(u) * kFieldThreads + threadIdx.x;
    if (j >= n_total) break;
    const c64 pj = sol[j];
    acc = cadd(acc, field_contribution(full_element(corners, nv, cen, nrm, diam, beta, n, cx, cy, pitch, j, false,
                                                    hs_axis, hs_offset), x, k, pj));
    if (with_image)
      acc = cadd(acc, cmul(refl, field_contribution(full_element(corners, nv, cen, nrm, diam, beta, n, cx, cy, pitch,
                                                                 j, true, hs_axis, hs_offset), x, k, pj)));
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kFieldThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[static_cast<long long>(blockIdx.x) * n_pts + pt] = red[0];
}

// out[pt] = p_inc[pt] + sum over chunks, in chunk order
__global__ void field_sum_kernel(const c64* __restrict__ partial, int n_chunks, int n_pts,
                                 const c64* __restrict__ p_inc, c64* __restrict__ out) {
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  if (pt >= n_pts) return;
  c64 acc = p_inc ? p_inc[pt] : cmk(0.0, 0.0);
  for (int c = 0; c < n_chunks; ++c) acc = cadd(acc, partial[static_cast<long long>(c) * n_pts + pt]);
  out[pt] = acc;
}

}  // namespace

int field_chunks(long long n_total) {
  return static_cast<int>((n_total + kFieldThreads * kFieldPerThread - 1) / (kFieldThreads * kFieldPerThread));
}

cudaError_t launch_field(const double* corners, const int* nv, const double* cen, const double* nrm,
                         const double* diam, const c64* beta, int n, const int counts[3], const double pitch[3],
                         const c64* solution, const double* pts, int n_pts, const c64* p_inc, double k,
                         bool with_image, int hs_axis, double hs_offset, c64 refl, c64* partial, c64* out,
                         cudaStream_t stream) {
  if (n_pts == 0) return cudaSuccess;
  const long long n_total = static_cast<long long>(n) * counts[0] * counts[1] * counts[2];
  const int chunks = field_chunks(n_total);
  for (int p0 = 0; p0 < n_pts; p0 += 65535) {  // grid.y limit
    const int np = n_pts - p0 < 65535 ? n_pts - p0 : 65535;
    field_kernel<<<dim3(chunks, np), kFieldThreads, 0, stream>>>(
        corners, nv, cen, nrm, diam, beta, n, counts[0], counts[1], p3(pitch[0], pitch[1], pitch[2]), n_total,
        solution, pts + 3LL * p0, n_pts, k, with_image ? 1 : 0, hs_axis, hs_offset, refl, partial + p0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  field_sum_kernel<<<(n_pts + 127) / 128, 128, 0, stream>>>(partial, chunks, n_pts, p_inc, out);
  return cudaGetLastError();
}

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
