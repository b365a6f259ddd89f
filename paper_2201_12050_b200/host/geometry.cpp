// Unit-cell meshes, lattices and the near/far box grid.
// Restates /root/reference/proj/src/geometry.cpp:14-196 (quads, cube-sphere,
// wall cell, replication, box grid, admissibility); icosphere, closed
// cylinder, closed box and triangles are extensions for BASELINE.json's
// configs (parity unpinned).
#include <algorithm>
#include <limits>
#include <map>
#include <stdexcept>

#include "fpbem_host.hpp"

namespace fpbem_host {

// geometry.cpp:14-28: area = two triangle halves, normal = their normalised
// sum, area-weighted centroid, diameter = longest diagonal.
Element make_quad(const V3& a, const V3& b, const V3& c, const V3& d, cd beta) {
  Element e;
  e.c = {a, b, c, d};
  e.nv = 4;
  V3 n1 = cross(b - a, c - a), n2 = cross(c - a, d - a);
  double a1 = 0.5 * norm(n1), a2 = 0.5 * norm(n2);
  e.area = a1 + a2;
  if (!(e.area > 0.0)) throw std::runtime_error("make_quad: degenerate element");
  e.normal = unit(n1 + n2);
  e.centroid = (a1 * (a + b + c) + a2 * (a + c + d)) / (3.0 * e.area);
  e.diameter = std::max(norm(c - a), norm(d - b));
  e.beta = beta;
  return e;
}

// Triangle: the quad formulas with the fourth corner collapsed onto the
// third (the bilinear map then is the Duffy map of the triangle); the
// diameter is the longest edge.
Element make_tri(const V3& a, const V3& b, const V3& c, cd beta) {
  Element e;
  e.c = {a, b, c, c};
  e.nv = 3;
  V3 n1 = cross(b - a, c - a);
  e.area = 0.5 * norm(n1);
  if (!(e.area > 0.0)) throw std::runtime_error("make_tri: degenerate element");
  e.normal = unit(n1);
  e.centroid = (a + b + c) / 3.0;
  e.diameter = std::max({norm(b - a), norm(c - b), norm(a - c)});
  e.beta = beta;
  return e;
}

// Symmetry-consistent corner order (extension). The axis
// sign maps g (bit d of g flips axis d about the bounding-box centre; the 7
// mirrors, pi-rotations and the inversion) under which the cell mesh is
// invariant as a set of elements form a group; every orbit of elements gets
// corners that are the images of its representative's corners, reordered
// (b', a', [d', c'] / c') for orientation-reversing g, so the bilinear element
// map of an image is the image of the representative's map composed with
// u -> 1 - u. Gauss nodes, weights and the 4-fold subdivision are symmetric
// under u -> 1 - u, so images carry the images of the representative's
// quadrature nodes and every interaction satisfies
// S_{A_g o}[P_g i, P_g j] = S_o[i, j] up to rounding (normals and relative
// vectors map by g, all kernel terms are invariant). A representative fixed by
// some g gets the corner rotation that g maps to itself (a triangle on a mirror
// plane: the vertex on the plane last). The element order, the corner sets and
// the orientation are unchanged; without a consistent choice the mesh is left
// as it is. The lattice near field uses the symmetries after verifying them on
// the assembled blocks.
int cell_symmetries(const Mesh& m, std::vector<std::vector<int>>& perm) {
  const int n = m.size();
  perm.assign(8, {});
  if (n < 2) return 0;
  V3 lo, hi;
  m.bbox(lo, hi);
  const V3 ctr = 0.5 * (lo + hi);
  const double tol = 1e-9 * std::max(1e-300, norm(hi - lo));
  auto img = [&](int g, const V3& p) {
    V3 r = p;
    for (int d = 0; d < 3; ++d)
      if (g >> d & 1) r[d] = 2.0 * ctr[d] - p[d];
    return r;
  };
  int valid = 1;
  perm[0].resize(n);
  for (int j = 0; j < n; ++j) perm[0][j] = j;
  for (int g = 1; g < 8; ++g) {
    std::vector<int> p(n, -1);
    bool ok = true;
    for (int j = 0; j < n && ok; ++j) {
      const V3 r = img(g, m.el[j].centroid);
      for (int k = 0; k < n && p[j] < 0; ++k)
        if (m.el[k].nv == m.el[j].nv && norm(m.el[k].centroid - r) < tol) p[j] = k;
      const int k = p[j];
      ok = k >= 0;
      for (int a = 0; a < m.el[j].nv && ok; ++a) {  // the image corners are k's corners
        bool found = false;
        for (int b = 0; b < m.el[k].nv && !found; ++b) found = norm(m.el[k].c[b] - img(g, m.el[j].c[a])) < tol;
        ok = found;
      }
    }
    if (ok) {
      perm[g] = p;
      valid |= 1 << g;
    }
  }
  for (bool changed = true; changed;) {  // keep a group: drop g whose products leave the set
    changed = false;
    for (int g1 = 1; g1 < 8; ++g1)
      for (int g2 = 1; g2 < 8; ++g2)
        if ((valid >> g1 & 1) && (valid >> g2 & 1) && !(valid >> (g1 ^ g2) & 1)) {
          valid &= ~(1 << std::max(g1, g2));
          changed = true;
        }
  }
  return valid;
}

void symmetrize_group(Mesh& m) {
  std::vector<std::vector<int>> perm;
  const int valid = cell_symmetries(m, perm);
  if (valid <= 1) return;
  const int n = m.size();
  V3 lo, hi;
  m.bbox(lo, hi);
  const V3 ctr = 0.5 * (lo + hi);
  const double tol = 1e-9 * std::max(1e-300, norm(hi - lo));
  auto img = [&](int g, const V3& p) {
    V3 r = p;
    for (int d = 0; d < 3; ++d)
      if (g >> d & 1) r[d] = 2.0 * ctr[d] - p[d];
    return r;
  };
  auto reversing = [](int g) { return (__builtin_popcount(g) & 1) != 0; };
  // corners of the image of an element with corners c[0..nv) under g
  auto image = [&](int g, const std::array<V3, 4>& c, int nv) {
    std::array<V3, 4> r;
    if (reversing(g)) {
      r = {img(g, c[1]), img(g, c[0]), img(g, nv == 3 ? c[2] : c[3]), img(g, c[2])};
      if (nv == 3) r[3] = r[2];
    } else {
      r = {img(g, c[0]), img(g, c[1]), img(g, c[2]), img(g, c[3])};
    }
    return r;
  };
  auto same = [&](const std::array<V3, 4>& a, const std::array<V3, 4>& b, int nv, int shift) {
    for (int k = 0; k < nv; ++k)
      if (norm(a[k] - b[(k + shift) % nv]) >= tol) return false;
    return true;
  };
  std::vector<std::array<V3, 4>> out(n);
  std::vector<char> done(n, 0);
  for (int j = 0; j < n; ++j) {
    if (done[j]) continue;
    const Element& e = m.el[j];
    const int nv = e.nv;
    // the representative's corner rotation that its stabiliser maps to itself
    // (a pi-rotation fixing a quad may also map it to its half-turn)
    std::array<V3, 4> rep{};
    bool found = false;
    for (int rot = 0; rot < nv && !found; ++rot) {
      std::array<V3, 4> c;
      for (int k = 0; k < nv; ++k) c[k] = e.c[(k + rot) % nv];
      if (nv == 3) c[3] = c[2];
      bool ok = true;
      for (int g = 1; g < 8 && ok; ++g)
        if ((valid >> g & 1) && perm[g][j] == j) {
          const std::array<V3, 4> im = image(g, c, nv);
          ok = same(im, c, nv, 0) || (!reversing(g) && nv == 4 && same(im, c, nv, 2));
        }
      if (ok) {
        rep = c;
        found = true;
      }
    }
    if (!found) return;  // no consistent choice: leave the mesh unchanged
    for (int g = 0; g < 8; ++g) {
      if (!(valid >> g & 1)) continue;
      const int k = perm[g][j];
      if (done[k]) continue;
      out[k] = g == 0 ? rep : image(g, rep, nv);
      done[k] = 1;
    }
  }
  for (int k = 0; k < n; ++k) {
    const Element& e = m.el[k];
    const auto& c = out[k];
    m.el[k] = e.nv == 3 ? make_tri(c[0], c[1], c[2], e.beta) : make_quad(c[0], c[1], c[2], c[3], e.beta);
  }
}

void Mesh::bbox(V3& lo, V3& hi) const {
  const double big = std::numeric_limits<double>::max();
  lo = {big, big, big};
  hi = {-big, -big, -big};
  for (const Element& e : el)
    for (int k = 0; k < e.nv; ++k)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], e.c[k][d]);
        hi[d] = std::max(hi[d], e.c[k][d]);
      }
}

// Cube-projected sphere of 6 r^2 flat panels (geometry.cpp:67-109).
Mesh cube_sphere(double radius, int refinement, cd beta) {
  if (radius <= 0.0 || refinement < 1) throw std::invalid_argument("cube_sphere: bad arguments");
  struct Face {
    int u, v, w;
    double s;
  };
  const Face faces[6] = {{0, 1, 2, 1.0}, {1, 0, 2, -1.0}, {2, 0, 1, 1.0},
                         {0, 2, 1, -1.0}, {1, 2, 0, 1.0}, {2, 1, 0, -1.0}};
  Mesh m;
  for (const Face& f : faces)
    for (int i = 0; i < refinement; ++i)
      for (int j = 0; j < refinement; ++j) {
        auto node = [&](int a, int b) {
          V3 p;
          p[f.u] = -1.0 + 2.0 * a / refinement;
          p[f.v] = -1.0 + 2.0 * b / refinement;
          p[f.w] = f.s;
          return radius * unit(p);
        };
        V3 c[4] = {node(i, j), node(i + 1, j), node(i + 1, j + 1), node(i, j + 1)};
        V3 mid = 0.25 * (c[0] + c[1] + c[2] + c[3]);
        V3 n = unit(cross(c[2] - c[0], c[3] - c[1]));
        if (dot(n, mid) < 0.0) {
          std::swap(c[1], c[3]);
          n = -n;
        }
        for (V3& p : c) p = p - dot(n, p - mid) * n;  // flatten onto the panel plane
        m.el.push_back(make_quad(c[0], c[1], c[2], c[3], beta));
      }
  return m;
}

// Two-layer open wall slice (geometry.cpp:111-135).
Mesh wall_cell(double ly, double lz, double t, int div, cd beta) {
  if (ly <= 0 || lz <= 0 || t <= 0 || div < 1) throw std::invalid_argument("wall_cell: bad arguments");
  Mesh m;
  const double dy = ly / div, dz = lz / div;
  for (int layer = 0; layer < 2; ++layer) {
    const double x = layer == 0 ? -0.5 * t : 0.5 * t;
    for (int j = 0; j < div; ++j)
      for (int i = 0; i < div; ++i) {
        double y0 = -0.5 * ly + i * dy, y1 = y0 + dy, z0 = j * dz, z1 = z0 + dz;
        if (layer == 0)
          m.el.push_back(make_quad({x, y0, z0}, {x, y0, z1}, {x, y1, z1}, {x, y1, z0}, beta));
        else
          m.el.push_back(make_quad({x, y0, z0}, {x, y1, z0}, {x, y1, z1}, {x, y0, z1}, beta));
      }
  }
  return m;
}

// Icosahedron refined by edge bisection, nodes projected to the sphere;
// 20 * 4^s flat triangles, outward counter-clockwise corner loops.
Mesh icosphere(double radius, int subdivisions, cd beta) {
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<V3> nodes = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                           {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  for (V3& p : nodes) p = unit(p);
  std::vector<std::array<int, 3>> tris = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
      {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6}, {3, 6, 8},
      {3, 8, 9},  {4, 9, 5},  {2, 4, 11},  {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
  for (int s = 0; s < subdivisions; ++s) {
    std::map<std::pair<int, int>, int> mid;
    auto midpoint = [&](int a, int b) {
      auto key = std::make_pair(std::min(a, b), std::max(a, b));
      auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      nodes.push_back(unit(0.5 * (nodes[a] + nodes[b])));
      int id = static_cast<int>(nodes.size()) - 1;
      mid[key] = id;
      return id;
    };
    std::vector<std::array<int, 3>> next;
    for (const auto& tr : tris) {
      int a = midpoint(tr[0], tr[1]), b = midpoint(tr[1], tr[2]), c = midpoint(tr[2], tr[0]);
      next.push_back({tr[0], a, c});
      next.push_back({tr[1], b, a});
      next.push_back({tr[2], c, b});
      next.push_back({a, b, c});
    }
    tris.swap(next);
  }
  Mesh m;
  for (const auto& tr : tris) {
    V3 a = radius * nodes[tr[0]], b = radius * nodes[tr[1]], c = radius * nodes[tr[2]];
    if (dot(cross(b - a, c - a), a + b + c) < 0.0) std::swap(b, c);
    m.el.push_back(make_tri(a, b, c, beta));
  }
  symmetrize_group(m);
  return m;
}

// Closed cylinder along z on [0, height]: n_theta x n_z side quads each split
// into two triangles, plus a triangle fan per cap; 2 n_theta (n_z + 1) triangles.
// The split diagonal runs (theta_i, z_j)-(theta_i+1, z_j+1) in the lower half and
// the other way in the upper half (the middle row of an odd n_z: half of the
// ring each way), so for even n_theta the triangulation is symmetric under the
// point reflection about the cylinder's centre, like the cylinder itself.
Mesh closed_cylinder(double radius, double height, int n_theta, int n_z, cd beta) {
  Mesh m;
  auto ring = [&](int i, double z) {
    double a = 2.0 * kPi * i / n_theta;
    return V3{radius * std::cos(a), radius * std::sin(a), z};
  };
  for (int j = 0; j < n_z; ++j) {
    double z0 = height * j / n_z, z1 = height * (j + 1) / n_z;
    for (int i = 0; i < n_theta; ++i) {
      V3 p00 = ring(i, z0), p10 = ring(i + 1, z0), p11 = ring(i + 1, z1), p01 = ring(i, z1);
      const bool lower = 2 * j + 1 < n_z || (2 * j + 1 == n_z && 2 * i < n_theta);
      // outward (radial) orientation: theta then z is counter-clockwise seen from outside
      if (lower) {
        m.el.push_back(make_tri(p00, p10, p11, beta));
        m.el.push_back(make_tri(p00, p11, p01, beta));
      } else {
        m.el.push_back(make_tri(p00, p10, p01, beta));
        m.el.push_back(make_tri(p10, p11, p01, beta));
      }
    }
  }
  V3 bottom{0, 0, 0}, top{0, 0, height};
  for (int i = 0; i < n_theta; ++i) {
    m.el.push_back(make_tri(bottom, ring(i + 1, 0.0), ring(i, 0.0), beta));      // normal -z
    m.el.push_back(make_tri(top, ring(i, height), ring(i + 1, height), beta));   // normal +z
  }
  symmetrize_group(m);
  return m;
}

// Closed axis-aligned box [-lx/2,lx/2] x [-ly/2,ly/2] x [0,lz] meshed with
// squares of side ~h on every face (outward normals), optionally each split
// into two triangles.
Mesh closed_box(double lx, double ly, double lz, double h, bool split, cd beta) {
  Mesh m;
  const double lo[3] = {-0.5 * lx, -0.5 * ly, 0.0}, hi[3] = {0.5 * lx, 0.5 * ly, lz};
  for (int axis = 0; axis < 3; ++axis)
    for (int side = 0; side < 2; ++side) {
      const int u = (axis + 1) % 3, v = (axis + 2) % 3;
      const int nu = std::max(1, static_cast<int>(std::lround((hi[u] - lo[u]) / h)));
      const int nv = std::max(1, static_cast<int>(std::lround((hi[v] - lo[v]) / h)));
      for (int j = 0; j < nv; ++j)
        for (int i = 0; i < nu; ++i) {
          auto pt = [&](int a, int b) {
            V3 p;
            p[axis] = side ? hi[axis] : lo[axis];
            p[u] = lo[u] + (hi[u] - lo[u]) * a / nu;
            p[v] = lo[v] + (hi[v] - lo[v]) * b / nv;
            return p;
          };
          V3 q[4] = {pt(i, j), pt(i + 1, j), pt(i + 1, j + 1), pt(i, j + 1)};
          // (u, v, axis) is right-handed, so this loop has normal +axis
          if (!side) std::swap(q[1], q[3]);
          if (split) {
            m.el.push_back(make_tri(q[0], q[1], q[2], beta));
            m.el.push_back(make_tri(q[0], q[2], q[3], beta));
          } else {
            m.el.push_back(make_quad(q[0], q[1], q[2], q[3], beta));
          }
        }
    }
  symmetrize_group(m);
  return m;
}

// cell-major replication, x fastest (geometry.cpp:137-155)
Mesh replicate(const Mesh& cell, const Lattice& lat) {
  Mesh m;
  m.el.reserve(static_cast<size_t>(lat.cells()) * cell.el.size());
  for (int iz = 0; iz < lat.counts[2]; ++iz)
    for (int iy = 0; iy < lat.counts[1]; ++iy)
      for (int ix = 0; ix < lat.counts[0]; ++ix) {
        V3 s = lat.shift(ix, iy, iz);
        for (const Element& e : cell.el) {
          Element t = e;
          for (V3& c : t.c) c = c + s;
          t.centroid = t.centroid + s;
          m.el.push_back(t);
        }
      }
  return m;
}

V3 mirror_point(const V3& p, const HalfSpace& hs) {
  V3 q = p;
  q[hs.axis] = 2.0 * hs.offset - p[hs.axis];
  return q;
}

// mirrored copy with reversed corner loop; the stored normal is the mirrored
// source normal, so BIE-flipped meshes stay flipped (geometry.cpp:164-178)
Mesh mirror_mesh(const Mesh& m, const HalfSpace& hs) {
  Mesh out;
  out.el.reserve(m.el.size());
  for (const Element& e : m.el) {
    Element t;
    if (e.nv == 3)
      t = make_tri(mirror_point(e.c[0], hs), mirror_point(e.c[2], hs), mirror_point(e.c[1], hs), e.beta);
    else
      t = make_quad(mirror_point(e.c[0], hs), mirror_point(e.c[3], hs), mirror_point(e.c[2], hs),
                    mirror_point(e.c[1], hs), e.beta);
    V3 n = e.normal;
    n[hs.axis] = -n[hs.axis];
    t.normal = n;
    out.el.push_back(t);
  }
  return out;
}

Mesh bie_oriented(const Mesh& m) {
  Mesh out = m;
  for (Element& e : out.el) e.normal = -e.normal;
  return out;
}

BoxGrid make_box_grid(const Mesh& cell, const Lattice& lat) {
  V3 lo, hi;
  cell.bbox(lo, hi);
  V3 size;
  for (int d = 0; d < 3; ++d) size[d] = lat.counts[d] > 1 ? lat.pitch[d] : hi[d] - lo[d];
  BoxGrid g;
  g.base_center = 0.5 * (lo + hi);
  g.radius = 0.5 * norm(size);
  return g;
}

bool admissible(const V3& a, const V3& b, double r) {
  if (r <= 0.0) throw std::invalid_argument("admissible: r > 0 required");
  return norm(a - b) >= 2.0 * r;
}

}  // namespace fpbem_host
