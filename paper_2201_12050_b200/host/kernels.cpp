// Burton-Miller collocation kernels, element quadrature and incident fields.
// Restates /root/reference/proj/src/kernels.cpp:13-325 (regular tensor rule,
// 4-fold adaptive subdivision near the collocation point, closed-form planar
// self-term static parts plus Duffy-fan smooth remainders) and the entry
// formula of src/assembly.cpp:214-251. Triangles (nv == 3) reuse the quad
// rules with the collapsed fourth corner; the self-term skips the
// zero-length edge (extension, parity unpinned).
#include <algorithm>
#include <mutex>
#include <stdexcept>

#include "fpbem_host.hpp"

namespace fpbem_host {

namespace {

// (e^{ikr} - 1)/(4 pi r), series below kr = 0.5 (kernels.cpp:15-30)
cd sl_remainder(double k, double r) {
  const double kr = k * r;
  if (kr >= 0.5) return (std::exp(kI * kr) - 1.0) / (4.0 * kPi * r);
  cd sum(0.0, 0.0), pw(1.0, 0.0);
  const cd ikr = kI * kr;
  double fact = 1.0;
  for (int j = 1; j <= 24; ++j) {
    fact *= j;
    sum += pw / fact;
    pw *= ikr;
  }
  return kI * k / (4.0 * kPi) * sum;
}

// [e^{ikr}(1 - ikr) - 1 - (kr)^2/2] / (4 pi r^3) (kernels.cpp:32-50)
cd hyper_remainder(double k, double r) {
  const double kr = k * r;
  if (kr >= 0.5) {
    const cd e = std::exp(kI * kr);
    return (e * (1.0 - kI * kr) - 1.0 - 0.5 * kr * kr) / (4.0 * kPi * r * r * r);
  }
  cd sum(0.0, 0.0);
  const cd ik = kI * k;
  cd pw = ik * ik * ik;
  double fact = 2.0;
  for (int j = 3; j <= 26; ++j) {
    fact *= j;
    sum += (1.0 - j) / fact * pw;
    pw *= ik * r;
  }
  return sum / (4.0 * kPi);
}

struct QuadRule {
  std::vector<double> x, w;
};

const QuadRule& rule(int order) {
  static std::once_flag once;
  static std::vector<QuadRule> rules(17);
  std::call_once(once, [] {
    for (int n = 1; n <= 16; ++n) gauss_legendre(n, rules[n].x, rules[n].w);
  });
  if (order < 1 || order > 16) throw std::invalid_argument("gauss rule order in [1,16]");
  return rules[order];
}

void tensor_corners(const std::array<V3, 4>& c, int order, std::vector<QPoint>& out) {
  const QuadRule& r = rule(order);
  const size_t n = r.x.size();
  for (size_t i = 0; i < n; ++i) {
    const double u = r.x[i];
    for (size_t j = 0; j < n; ++j) {
      const double v = r.x[j];
      const double s0 = 0.25 * (1 - u) * (1 - v), s1 = 0.25 * (1 + u) * (1 - v),
                   s2 = 0.25 * (1 + u) * (1 + v), s3 = 0.25 * (1 - u) * (1 + v);
      V3 y = s0 * c[0] + s1 * c[1] + s2 * c[2] + s3 * c[3];
      V3 du = 0.25 * ((1 - v) * (c[1] - c[0]) + (1 + v) * (c[2] - c[3]));
      V3 dv = 0.25 * ((1 - u) * (c[3] - c[0]) + (1 + u) * (c[2] - c[1]));
      out.push_back({y, r.w[i] * r.w[j] * norm(cross(du, dv))});
    }
  }
}

void subdivide(const std::array<V3, 4>& c, const V3& x, int order, int depth, std::vector<QPoint>& out) {
  V3 mid = 0.25 * (c[0] + c[1] + c[2] + c[3]);
  double diam = std::max(norm(c[2] - c[0]), norm(c[3] - c[1]));
  if (depth <= 0 || norm(x - mid) >= kNearFactor * diam) {
    tensor_corners(c, order, out);
    return;
  }
  V3 m01 = 0.5 * (c[0] + c[1]), m12 = 0.5 * (c[1] + c[2]), m23 = 0.5 * (c[2] + c[3]),
     m30 = 0.5 * (c[3] + c[0]);
  subdivide({c[0], m01, mid, m30}, x, order, depth - 1, out);
  subdivide({m01, c[1], m12, mid}, x, order, depth - 1, out);
  subdivide({mid, m12, c[2], m23}, x, order, depth - 1, out);
  subdivide({m30, mid, m23, c[3]}, x, order, depth - 1, out);
}

}  // namespace

// Golub-Welsch-free Newton iteration on Legendre roots (kernels.cpp:162-194)
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(n, 0.0);
  weights.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 0; j < n; ++j) {
        double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j + 1.0) * x * p1 - j * p2) / (j + 1);
      }
      dp = n * (x * p0 - p1) / (x * x - 1.0);
      double dx = p0 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    nodes[i] = -x;
    nodes[n - 1 - i] = x;
    weights[i] = weights[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

void tensor_points(const Element& e, int order, std::vector<QPoint>& out) {
  tensor_corners(e.c, order, out);
}

void influence_points(const Element& e, const V3& x, int order, std::vector<QPoint>& out) {
  if (norm(x - e.centroid) < kNearFactor * e.diameter)
    subdivide(e.c, x, order, kMaxSubdivision, out);
  else
    tensor_corners(e.c, order, out);
}

// h = int dG/dn_y + alpha d2G/dn_x dn_y ; g = int G + alpha dG/dn_x
// with closed-form derivatives of e^{ikr}/(4 pi r) (kernels.cpp:143-160, 214-226)
Influence influence(const Wave& w, const Element& src, const V3& x, const V3& nx) {
  thread_local std::vector<QPoint> pts;
  pts.clear();
  influence_points(src, x, kRegularOrder, pts);
  const double k = w.k;
  const V3& ny = src.normal;
  const double nxny = dot(nx, ny);
  Influence out;
  for (const QPoint& q : pts) {
    V3 d = x - q.y;
    double r = norm(d);
    if (r <= 0.0) throw std::domain_error("influence: coincident points");
    double inv = 1.0 / r;
    double cx = dot(d, nx) * inv, cy = dot(d, ny) * inv;
    cd g = std::exp(kI * (k * r)) * (inv / (4.0 * kPi));
    cd qd = kI * k - inv;  // dG/dr = q G
    cd dgdny = -qd * g * cy;
    cd dgdnx = qd * g * cx;
    cd d2g = g * (k * k + 3.0 * kI * k * inv - 3.0 * inv * inv) * cx * cy - g * qd * inv * nxny;
    out.h += q.w * (dgdny + w.alpha * d2g);
    out.g += q.w * (g + w.alpha * dgdnx);
  }
  return out;
}

// Self term at the element's own centroid (kernels.cpp:228-261).
Influence influence_self(const Wave& w, const Element& e) {
  const V3& x = e.centroid;
  const double k = w.k;
  const V3 ng = unit(cross(e.c[2] - e.c[0], e.c[3] - e.c[1]));
  double sl0 = 0.0, hyp0 = 0.0;
  for (int edge = 0; edge < 4; ++edge) {
    V3 a = e.c[edge] - x, b = e.c[(edge + 1) % 4] - x;
    V3 ab = b - a;
    double len = norm(ab);
    if (len == 0.0) continue;  // collapsed edge of a triangle
    V3 t = ab / len;
    double sa = dot(a, t), sb = dot(b, t), da = norm(a), db = norm(b);
    double h = dot(ng, cross(a, b)) / len;
    sl0 += h * std::log((db + sb) / (da + sa));
    hyp0 -= (sb / db - sa / da) / h;
  }
  sl0 /= 4.0 * kPi;
  hyp0 /= 4.0 * kPi;

  // polar (Duffy) fan around the centroid for the smooth remainders
  const QuadRule& r = rule(kSelfOrder);
  cd g_rem(0.0, 0.0), h_rem(0.0, 0.0);
  for (int edge = 0; edge < 4; ++edge) {
    V3 a = e.c[edge] - x, b = e.c[(edge + 1) % 4] - x;
    if (norm(b - a) == 0.0) continue;
    double jac2 = dot(cross(a, b), ng);
    for (size_t i = 0; i < r.x.size(); ++i) {
      double u = 0.5 * (r.x[i] + 1.0);
      for (size_t j = 0; j < r.x.size(); ++j) {
        double v = 0.5 * (r.x[j] + 1.0);
        V3 y = u * ((1.0 - v) * a + v * b);
        double wq = 0.25 * r.w[i] * r.w[j] * u * jac2;
        double rr = norm(y);
        g_rem += wq * sl_remainder(k, rr);
        h_rem += wq * hyper_remainder(k, rr);
      }
    }
  }
  Influence out;
  out.g = sl0 + g_rem;
  out.h = w.alpha * (hyp0 + 0.5 * k * k * sl0 + h_rem);
  return out;
}

// assembly.cpp:214-223
cd bm_entry(const Wave& w, const Element& src, const V3& x, const V3& nx, bool self) {
  const cd ikb = kI * w.k * src.beta;
  if (self) {
    Influence s = influence_self(w, src);
    return 0.5 + 0.5 * w.alpha * ikb + s.h - ikb * s.g;
  }
  Influence p = influence(w, src, x, nx);
  return p.h - ikb * p.g;
}

namespace {
void add_source(const Source& s, double k, const V3& x, const V3& nx, cd& p, cd& dpdn) {
  if (s.plane) {  // kernels.cpp:289-292
    cd e = s.amp * std::exp(kI * (k * dot(s.v, x)));
    p += e;
    dpdn += kI * k * dot(s.v, nx) * e;
  } else {  // monopole normalised to |p| = amp at 1 m (kernels.cpp:293-300)
    V3 d = x - s.v;
    double r = norm(d);
    if (r <= 0.0) throw std::domain_error("incident: point coincides with a monopole");
    cd e = s.amp * std::exp(kI * (k * r)) / r;
    p += e;
    dpdn += (kI * k - 1.0 / r) * e * (dot(d, nx) / r);
  }
}
}  // namespace

// superposition with optional mirror images (kernels.cpp:302-325)
void incident(const std::vector<Source>& src, double k, const V3& x, const V3& nx, cd& p, cd& dpdn,
              const HalfSpace* hs) {
  p = dpdn = cd(0.0, 0.0);
  for (const Source& s : src) {
    add_source(s, k, x, nx, p, dpdn);
    if (hs && hs->active()) {
      Source img = s;
      img.amp *= hs->reflection;
      if (s.plane) {  // mirrored direction with the plane-offset phase
        img.v[hs->axis] = -img.v[hs->axis];
        img.amp *= std::exp(kI * (k * 2.0 * hs->offset * s.v[hs->axis]));
      } else {
        img.v = mirror_point(s.v, *hs);
      }
      add_source(img, k, x, nx, p, dpdn);
    }
  }
}

std::vector<cd> assemble_rhs(const Mesh& full, const Wave& w, const std::vector<Source>& src,
                             const HalfSpace* hs) {
  std::vector<cd> rhs(full.size());
#pragma omp parallel for schedule(static)
  for (int i = 0; i < full.size(); ++i) {
    const Element& e = full.el[i];
    cd p, dpdn;
    incident(src, w.k, e.centroid, -e.normal, p, dpdn, hs);
    rhs[i] = p + w.alpha * dpdn;
  }
  return rhs;
}

}  // namespace fpbem_host
