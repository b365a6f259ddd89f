// Field evaluation by the representation formula and the insertion loss.
// Restates /root/reference/proj/src/postproc.cpp:18-81: for each observation
// point x, p(x) = p_inc(x) + sum_j int_{e_j} [-dG/dn_y(x, y) p_j + G(x, y) i k beta_j p_j] dy
// over the BIE-oriented elements (influence quadrature of src/kernels.cpp:205-212,
// order 6 with adaptive subdivision near x), plus reflection * the same sum
// over the mirrored mesh when a half space is active; IL = 20 log10(sum |p_inc| / sum |p|).
// This is the checker for the device kernel (csrc/assembly.cu field_kernel).
#include <cmath>
#include <stdexcept>

#include "fpbem_host.hpp"

namespace fpbem_host {

namespace {

constexpr double kPi = 3.14159265358979323846;

cd element_contribution(const Wave& w, const Element& e, const V3& x, cd pressure) {
  const double k = w.k;
  const cd ikb_p = cd(0.0, k) * e.beta * pressure;
  std::vector<QPoint> pts;
  influence_points(e, x, 6, pts);
  cd acc(0.0, 0.0);
  for (const QPoint& qp : pts) {
    const V3 d = x - qp.y;
    const double r = norm(d);
    const cd g = std::exp(cd(0.0, k * r)) / (4.0 * kPi * r);
    const cd dgdn = -(cd(0.0, k) - 1.0 / r) * g * (dot(d, e.normal) / r);
    acc += qp.w * (-dgdn * pressure + g * ikb_p);
  }
  return acc;
}

}  // namespace

std::vector<cd> evaluate_field(const Mesh& full, const std::vector<cd>& solution, const Wave& w,
                               const std::vector<Source>& src, const std::vector<V3>& points, const HalfSpace* hs) {
  if (static_cast<int>(solution.size()) != full.size())
    throw std::invalid_argument("evaluate_field: solution length mismatch");
  const Mesh bie = bie_oriented(full);
  const bool with_image = hs && hs->active();
  Mesh image;
  if (with_image) image = mirror_mesh(bie, *hs);
  std::vector<cd> out(points.size());
#pragma omp parallel for schedule(dynamic, 8)
  for (int ip = 0; ip < static_cast<int>(points.size()); ++ip) {
    const V3& x = points[ip];
    cd p, dpdn;
    incident(src, w.k, x, V3{0.0, 0.0, 1.0}, p, dpdn, hs);
    cd acc = p;
    for (int j = 0; j < bie.size(); ++j) {
      acc += element_contribution(w, bie.el[j], x, solution[j]);
      if (with_image) acc += hs->reflection * element_contribution(w, image.el[j], x, solution[j]);
    }
    out[ip] = acc;
  }
  return out;
}

double insertion_loss(const std::vector<cd>& p_inc, const std::vector<cd>& p) {
  if (p_inc.size() != p.size() || p.empty())
    throw std::invalid_argument("insertion_loss: paired non-empty vectors required");
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < p.size(); ++i) {
    num += std::abs(p_inc[i]);
    den += std::abs(p[i]);
  }
  if (den == 0.0) throw std::domain_error("insertion_loss: vanishing total pressure");
  return 20.0 * std::log10(num / den);
}

}  // namespace fpbem_host
