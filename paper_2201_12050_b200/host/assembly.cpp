// Operator assembly: near-field Toeplitz blocks, far-field M2L bank, shared
// P2M/L2P matrices, dense reference system and the BASELINE scenes.
// Restates /root/reference/proj/src/fmm.cpp:22-65 (p2m/l2p), :125-190
// (assemble_periodic_fmm: bie orientation, box grid, offset loop z,y,x
// ascending, admissible -> M2L block else interaction block) and
// src/assembly.cpp:225-276 (interaction_block, dense assembly).
#include <algorithm>
#include <memory>
#include <mutex>
#include <stdexcept>

#include "fpbem_host.hpp"

namespace fpbem_host {

// V0(idx, j) = int_j [conj(dI_n^m/dn)(y-c) - ik beta_j conj(I_n^m)(y-c)] dGamma
void p2m_matrix(const Mesh& cell_bie, const Wave& w, int n_t, const V3& center, cd* v0) {
  const int p = coef_count(n_t);
  const int n = cell_bie.size();
  const double k = w.k;
  std::fill(v0, v0 + static_cast<size_t>(p) * n, cd(0.0, 0.0));
#pragma omp parallel for schedule(dynamic, 4)
  for (int j = 0; j < n; ++j) {
    const Element& e = cell_bie.el[j];
    const cd ikb = kI * k * e.beta;
    std::vector<QPoint> pts;
    tensor_points(e, kRegularOrder, pts);
    cd* col = v0 + static_cast<size_t>(j) * p;
    for (const QPoint& q : pts) {
      SolidGrad g = solid_regular_gradients(n_t, q.y - center, k);
      for (int i = 0; i < p; ++i) {
        cd dn = g.dx[i] * e.normal.x + g.dy[i] * e.normal.y + g.dz[i] * e.normal.z;
        col[i] += q.w * (std::conj(dn) - ikb * std::conj(g.val[i]));
      }
    }
  }
}

// U0(i, (n,m)) = (ik/4pi)(2n+1) [conj(I_n^m)(x_i-c) + alpha conj(dI_n^m/dn)(x_i-c)]
void l2p_matrix(const Mesh& cell_bie, const Wave& w, int n_t, const V3& center, cd* u0) {
  const int p = coef_count(n_t);
  const int n = cell_bie.size();
  const double k = w.k;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    const Element& e = cell_bie.el[i];
    SolidGrad g = solid_regular_gradients(n_t, e.centroid - center, k);
    for (int deg = 0; deg <= n_t; ++deg)
      for (int ord = -deg; ord <= deg; ++ord) {
        const int idx = flat(deg, ord);
        cd dn = g.dx[idx] * e.normal.x + g.dy[idx] * e.normal.y + g.dz[idx] * e.normal.z;
        u0[static_cast<size_t>(idx) * n + i] =
            kI * k / (4.0 * kPi) * (2.0 * deg + 1.0) * (std::conj(g.val[idx]) + w.alpha * std::conj(dn));
      }
  }
}

void interaction_block(const Wave& w, const Mesh& tgt, const V3& shift, const Mesh& src, bool self_terms,
                       cd* out) {
  const int rows = tgt.size(), cols = src.size();
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < rows; ++i) {
    const V3 x = tgt.el[i].centroid + shift;
    const V3& nx = tgt.el[i].normal;
    for (int j = 0; j < cols; ++j)
      out[static_cast<size_t>(j) * rows + i] = bm_entry(w, src.el[j], x, nx, self_terms && i == j);
  }
}

static const Translation& table(int n_t) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<Translation>> cache(64);
  std::lock_guard<std::mutex> lock(mu);
  if (n_t < 0 || n_t >= 64) throw std::invalid_argument("n_t out of range");
  if (!cache[n_t]) cache[n_t] = std::make_unique<Translation>(n_t);
  return *cache[n_t];
}

void classify_offsets(const Mesh& cell, const Lattice& lat, std::vector<int>& near, std::vector<int>& far) {
  const BoxGrid grid = make_box_grid(cell, lat);
  const auto& m = lat.counts;
  near.clear();
  far.clear();
  for (int oz = 1 - m[2]; oz <= m[2] - 1; ++oz)
    for (int oy = 1 - m[1]; oy <= m[1] - 1; ++oy)
      for (int ox = 1 - m[0]; ox <= m[0] - 1; ++ox) {
        // center(o) - base_center, evaluated as the reference does (fmm.cpp:160)
        const V3 center = grid.base_center + lat.shift(ox, oy, oz);
        std::vector<int>& dst = admissible(center, grid.base_center, grid.radius) ? far : near;
        dst.insert(dst.end(), {ox, oy, oz});
      }
}

void mirror_parity_map(int n_t, int axis, cd* out) {  // fmm.cpp:108-123
  const int p = coef_count(n_t);
  std::fill(out, out + static_cast<size_t>(p) * p, cd(0.0, 0.0));
  for (int n = 0; n <= n_t; ++n)
    for (int m = -n; m <= n; ++m) {
      const int row = flat(n, m);
      int col;
      double v;
      if (axis == 2) {
        col = row;
        v = ((n + m) & 1) ? -1.0 : 1.0;
      } else {
        col = flat(n, -m);
        v = (axis == 0 && (m & 1)) ? -1.0 : 1.0;
      }
      out[static_cast<size_t>(col) * p + row] = v;
    }
}

namespace {
// c = a * b for p x p column-major blocks
void matmul(int p, const cd* a, const cd* b, cd* c) {
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < p; ++i) {
      cd s(0.0, 0.0);
      for (int k = 0; k < p; ++k) s += a[static_cast<size_t>(k) * p + i] * b[static_cast<size_t>(j) * p + k];
      c[static_cast<size_t>(j) * p + i] = s;
    }
}
Mesh shifted(const Mesh& m, const V3& s) {
  Mesh out = m;
  for (Element& e : out.el) {
    for (V3& c : e.c) c = c + s;
    e.centroid = e.centroid + s;
  }
  return out;
}
}  // namespace

// assemble_periodic_fmm (fmm.cpp:125-244): offsets in z, y, x order split by
// admissibility into the near blocks S_o and the M2L bank K_o; a half space
// parallel to every periodic direction folds its image into S and K, one
// whose axis is periodic yields the block-Hankel image pair (S_hat, K_hat).
FmmData assemble_fmm(const Mesh& cell, const Lattice& lat, const Wave& w, int n_t, bool skip_near_values,
                     const HalfSpace* hs, bool skip_far_values) {
  if (n_t < 0 || n_t > 30) throw std::invalid_argument("assemble_fmm: n_t in [0, 30] required");
  for (int d = 0; d < 3; ++d)
    if (lat.counts[d] < 1) throw std::invalid_argument("assemble_fmm: counts must be >= 1");
  FmmData op;
  op.counts = lat.counts;
  op.n_dof = cell.size();
  op.n_t = n_t;
  op.n_coef = coef_count(n_t);
  op.grid = make_box_grid(cell, lat);
  const Mesh bie = bie_oriented(cell);
  classify_offsets(cell, lat, op.near_offsets, op.far_offsets);
  const bool with_image = hs && hs->active();
  const bool split = with_image && lat.counts[hs->axis] > 1;
  const bool folded = with_image && !split;
  const int b = op.n_dof, p = op.n_coef;
  const size_t bb = static_cast<size_t>(b) * b, pp = static_cast<size_t>(p) * p;
  std::vector<cd> parity;
  Mesh image_cell;
  if (with_image) {
    parity.resize(pp);
    mirror_parity_map(n_t, hs->axis, parity.data());
    image_cell = mirror_mesh(bie, *hs);
  }

  if (!skip_near_values) {
    op.near_blocks.resize(static_cast<size_t>(op.n_near()) * bb);
    std::vector<cd> tmp(folded ? bb : 0);
    for (int s = 0; s < op.n_near(); ++s) {
      const int* o = &op.near_offsets[3 * s];
      const bool self = o[0] == 0 && o[1] == 0 && o[2] == 0;
      cd* blk = op.near_blocks.data() + s * bb;
      const V3 delta = lat.shift(o[0], o[1], o[2]);
      interaction_block(w, bie, delta, bie, self, blk);
      if (folded) {
        interaction_block(w, bie, delta, image_cell, false, tmp.data());
        for (size_t e = 0; e < bb; ++e) blk[e] += hs->reflection * tmp[e];
      }
    }
  }
  const Translation& tt = table(n_t);
  op.far_blocks.resize(skip_far_values ? 0 : static_cast<size_t>(op.n_far()) * pp);
#pragma omp parallel for schedule(static)
  for (int s = 0; s < (skip_far_values ? 0 : op.n_far()); ++s) {
    const int* o = &op.far_offsets[3 * s];
    cd* blk = op.far_blocks.data() + s * pp;
    tt.m2l(lat.shift(o[0], o[1], o[2]), w.k, blk);
    if (folded) {  // image boxes of far cells are at least as far as the cells
      const V3 center = op.grid.base_center + lat.shift(o[0], o[1], o[2]);
      std::vector<cd> k_img(pp), prod(pp);
      tt.m2l(center - mirror_point(op.grid.base_center, *hs), w.k, k_img.data());
      matmul(p, k_img.data(), parity.data(), prod.data());
      for (size_t e = 0; e < pp; ++e) blk[e] += hs->reflection * prod[e];
    }
  }
  op.u0.resize(static_cast<size_t>(b) * p);
  op.v0.resize(static_cast<size_t>(b) * p);
  l2p_matrix(bie, w, n_t, op.grid.base_center, op.u0.data());
  p2m_matrix(bie, w, n_t, op.grid.base_center, op.v0.data());

  if (split) {  // fmm.cpp:192-242
    const int ax = hs->axis;
    const auto& m = lat.counts;
    op.mirrored_level = ax;
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = d == ax ? 0 : 1 - m[d];
      hi[d] = d == ax ? 2 * m[d] - 2 : m[d] - 1;
    }
    const V3 base_image = mirror_point(op.grid.base_center, *hs);
    std::vector<cd> k_img(pp), prod(pp);
    for (int i2 = lo[2]; i2 <= hi[2]; ++i2)
      for (int i1 = lo[1]; i1 <= hi[1]; ++i1)
        for (int i0 = lo[0]; i0 <= hi[0]; ++i0) {
          int idx[3] = {i0, i1, i2};
          int tgt[3] = {i0, i1, i2}, src[3] = {0, 0, 0};
          tgt[ax] = std::min(idx[ax], m[ax] - 1);
          src[ax] = idx[ax] - tgt[ax];
          const V3 tshift = lat.shift(tgt[0], tgt[1], tgt[2]);
          const V3 sshift = lat.shift(src[0], src[1], src[2]);
          const V3 target_center = op.grid.base_center + tshift;
          V3 image_center = base_image;
          for (int d = 0; d < 3; ++d) image_center[d] += d == ax ? -sshift[d] : sshift[d];
          if (admissible(target_center, image_center, op.grid.radius)) {
            op.far_hat_indices.insert(op.far_hat_indices.end(), {i0, i1, i2});
            if (skip_far_values) continue;
            tt.m2l(target_center - image_center, w.k, k_img.data());
            matmul(p, k_img.data(), parity.data(), prod.data());
            for (size_t e = 0; e < pp; ++e) op.far_hat_blocks.push_back(hs->reflection * prod[e]);
          } else {
            op.hat_indices.insert(op.hat_indices.end(), {i0, i1, i2});
            if (skip_near_values) continue;
            const Mesh src_image = mirror_mesh(shifted(bie, sshift), *hs);
            const size_t at = op.hat_blocks.size();
            op.hat_blocks.resize(at + bb);
            interaction_block(w, bie, tshift, src_image, false, op.hat_blocks.data() + at);
            for (size_t e = 0; e < bb; ++e) op.hat_blocks[at + e] *= hs->reflection;
          }
        }
  }
  return op;
}

std::vector<cd> assemble_dense(const Mesh& full, const Wave& w, const HalfSpace* hs) {
  const Mesh bie = bie_oriented(full);
  const size_t n = static_cast<size_t>(full.size());
  std::vector<cd> a(n * n);
  interaction_block(w, bie, V3{0, 0, 0}, bie, true, a.data());
  if (hs && hs->active()) {  // assembly.cpp:260-271
    const Mesh image = mirror_mesh(bie, *hs);
#pragma omp parallel for schedule(dynamic, 4)
    for (long long i = 0; i < static_cast<long long>(n); ++i)
      for (size_t j = 0; j < n; ++j)
        a[j * n + i] += hs->reflection * bm_entry(w, image.el[j], bie.el[i].centroid, bie.el[i].normal, false);
  }
  return a;
}

// ---------------------------------------------------------------------------
// BASELINE.json configurations. variant 0 = the config as
// stated (triangle meshes: extension, parity unpinned); variant 1 = the
// reference-pinned quad variant (cube-sphere / quad box) where one exists;
// variant 2 = a shrunk lattice of the same cell for fast CPU checks.

static std::vector<Source> plane(V3 d) { return {Source{true, unit(d), cd(1.0, 0.0)}}; }
static std::vector<Source> monopole(V3 x) { return {Source{false, x, cd(1.0, 0.0)}}; }

Scene make_scene(int id, int variant) {
  Scene s;
  switch (id) {
    case 1:  // 8 spheres on a row, period 1.0, k = 2
      s.name = "cfg1";
      s.cell = variant == 1 ? cube_sphere(0.25, 7) : icosphere(0.25, 2);
      s.lat = Lattice{{variant == 2 ? 4 : 8, 1, 1}, {1.0, 0.0, 0.0}};
      s.wave = Wave::from_k(2.0);
      s.rhs_fields = {plane({1, 0, 0})};
      break;
    case 2: {  // 4 x 32 closed cylinders, square lattice 0.22 m, 1000 Hz
      s.name = "cfg2";
      s.cell = variant == 1 ? closed_cylinder(0.08, 2.0, 16, 31) : closed_cylinder(0.08, 2.0, 16, 31);
      if (variant == 2) s.cell = closed_cylinder(0.08, 2.0, 8, 7);
      s.lat = Lattice{{4, variant == 2 ? 8 : 32, 1}, {0.22, 0.22, 0.0}};
      s.wave = Wave::from_frequency(1000.0, 343.0);
      const double mid_y = 0.5 * 0.22 * (s.lat.counts[1] - 1);
      s.rhs_fields = {monopole({-5.0, mid_y, 1.0})};
      break;
    }
    case 3:  // 16^3 spheres, period 0.5, k * period = 3
      s.name = "cfg3";
      s.cell = variant == 1 ? cube_sphere(0.15, 7) : icosphere(0.15, 2);
      if (variant == 2) {
        s.lat = Lattice{{4, 4, 4}, {0.5, 0.5, 0.5}};
      } else {
        s.lat = Lattice{{16, 16, 16}, {0.5, 0.5, 0.5}};
      }
      s.wave = Wave::from_k(6.0);
      s.rhs_fields = {plane({1, 1, 1})};
      break;
    case 4: {  // 256 closed boxes on a row along y; period 1.05 m
      s.name = "cfg4";
      if (variant == 2)
        s.cell = closed_box(0.1, 1.0, 2.0, 0.25, true);
      else
        s.cell = closed_box(0.1, 1.0, 2.0, 0.05, variant != 1);
      s.lat = Lattice{{1, variant == 2 ? 16 : 256, 1}, {0.0, 1.05, 0.0}};
      s.wave = Wave::from_frequency(100.0, 343.0);
      for (int i = 1; i <= 10; ++i) s.sweep_hz.push_back(100.0 * i);
      const double mid_y = 0.5 * 1.05 * (s.lat.counts[1] - 1);
      s.rhs_fields = {monopole({-10.0, mid_y, 1.0})};
      break;
    }
    case 5: {  // 32 x 32 x 4 spheres, k * period = 2, 64 Fibonacci plane waves
      s.name = "cfg5";
      s.cell = variant == 1 ? cube_sphere(0.15, 7) : icosphere(0.15, 2);
      if (variant == 2)
        s.lat = Lattice{{6, 6, 2}, {0.5, 0.5, 0.5}};
      else
        s.lat = Lattice{{32, 32, 4}, {0.5, 0.5, 0.5}};
      s.wave = Wave::from_k(4.0);
      const double golden = kPi * (3.0 - std::sqrt(5.0));
      for (int i = 0; i < 64; ++i) {
        double z = 1.0 - (2.0 * i + 1.0) / 64.0;
        double rxy = std::sqrt(std::max(0.0, 1.0 - z * z));
        double phi = i * golden;
        s.rhs_fields.push_back(plane({rxy * std::cos(phi), rxy * std::sin(phi), z}));
      }
      break;
    }
    case 6:  // reference acceptance criterion 6 cell: cube-sphere r=0.1 ref 2, 1 x My x 1, 500 Hz
      s.name = "crit6";
      s.cell = cube_sphere(0.1, 2);
      s.lat = Lattice{{1, variant > 0 ? variant : 8, 1}, {0.35, 0.35, 0.35}};
      s.wave = Wave::from_frequency(500.0, 343.0);
      s.rhs_fields = {plane({1, 0, 0})};
      break;
    default:
      throw std::invalid_argument("make_scene: config id in 1..6");
  }
  return s;
}

}  // namespace fpbem_host
