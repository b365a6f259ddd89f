// C-ABI of the host operator producer, for the Python layer (ctypes).
// Complex arrays are interleaved (re, im) doubles.
#include <cstring>
#include <exception>
#include <string>

#include "fpbem_host.hpp"

using namespace fpbem_host;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct SceneH {
  Scene s;
};
struct FmmH {
  FmmData d;
};
}  // namespace

extern "C" {

const char* fh_last_error() { return g_err.c_str(); }

void* fh_scene_create(int id, int variant) {
  SceneH* h = nullptr;
  guarded([&] { h = new SceneH{make_scene(id, variant)}; });
  return h;
}

// kind: 0 cube_sphere(r, refinement) 1 icosphere(r, subdiv) 2 cylinder(r, h, n_theta, n_z)
//       3 closed box(lx, ly, lz, h, split) 4 wall cell(ly, lz, t, div)
void* fh_scene_custom(int kind, const double* p, const int* counts, const double* pitch, double k) {
  SceneH* h = nullptr;
  guarded([&] {
    Scene s;
    s.name = "custom";
    switch (kind) {
      case 0: s.cell = cube_sphere(p[0], static_cast<int>(p[1])); break;
      case 1: s.cell = icosphere(p[0], static_cast<int>(p[1])); break;
      case 2: s.cell = closed_cylinder(p[0], p[1], static_cast<int>(p[2]), static_cast<int>(p[3])); break;
      case 3: s.cell = closed_box(p[0], p[1], p[2], p[3], p[4] != 0.0); break;
      case 4: s.cell = wall_cell(p[0], p[1], p[2], static_cast<int>(p[3])); break;
      default: throw std::invalid_argument("fh_scene_custom: unknown kind");
    }
    for (int d = 0; d < 3; ++d) {
      s.lat.counts[d] = counts[d];
      s.lat.pitch[d] = pitch[d];
    }
    s.wave = Wave::from_k(k);
    s.rhs_fields = {{Source{true, V3{1, 0, 0}, cd(1.0, 0.0)}}};
    h = new SceneH{s};
  });
  return h;
}

void fh_scene_destroy(void* h) { delete static_cast<SceneH*>(h); }

// info: counts[3], n_dof, n_rhs, n_sweep ; dinfo: pitch[3], k
void fh_scene_info(void* hp, int* info, double* dinfo) {
  const Scene& s = static_cast<SceneH*>(hp)->s;
  for (int d = 0; d < 3; ++d) {
    info[d] = s.lat.counts[d];
    dinfo[d] = s.lat.pitch[d];
  }
  info[3] = s.cell.size();
  info[4] = static_cast<int>(s.rhs_fields.size());
  info[5] = static_cast<int>(s.sweep_hz.size());
  dinfo[3] = s.wave.k;
}

void fh_scene_set_k(void* hp, double k) { static_cast<SceneH*>(hp)->s.wave = Wave::from_k(k); }

// half space: mirror axis, plane offset, complex reflection (0 disables)
void fh_scene_set_halfspace(void* hp, int axis, double offset, double re, double im) {
  HalfSpace& h = static_cast<SceneH*>(hp)->s.half_space;
  h.axis = axis;
  h.offset = offset;
  h.reflection = cd(re, im);
}

// shift the unit cell (e.g. raise it above a ground plane)
void fh_scene_shift_cell(void* hp, const double* s) {
  Mesh& m = static_cast<SceneH*>(hp)->s.cell;
  for (Element& e : m.el) {
    for (V3& c : e.c) c = c + V3{s[0], s[1], s[2]};
    e.centroid = e.centroid + V3{s[0], s[1], s[2]};
  }
}

void fh_scene_sweep(void* hp, double* hz) {
  const Scene& s = static_cast<SceneH*>(hp)->s;
  for (size_t i = 0; i < s.sweep_hz.size(); ++i) hz[i] = s.sweep_hz[i];
}

// replace the right-hand-side fields: kinds[i] 1 = plane wave (direction), 0 = monopole (position)
void fh_scene_set_sources(void* hp, int n, const int* kinds, const double* vecs) {
  Scene& s = static_cast<SceneH*>(hp)->s;
  s.rhs_fields.clear();
  for (int i = 0; i < n; ++i) {
    V3 v{vecs[3 * i], vecs[3 * i + 1], vecs[3 * i + 2]};
    s.rhs_fields.push_back({Source{kinds[i] != 0, kinds[i] != 0 ? unit(v) : v, cd(1.0, 0.0)}});
  }
}

int fh_scene_rhs(void* hp, int field, double* out) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    Mesh full = replicate(s.cell, s.lat);
    std::vector<cd> r = assemble_rhs(full, s.wave, s.rhs_fields.at(field), &s.half_space);
    std::memcpy(out, r.data(), r.size() * sizeof(cd));
  });
}

// incident pressure of field `field` at n points (incident_values(...).first, kernels.cpp:305-325)
int fh_scene_incident(void* hp, int field, int n, const double* pts, double* out) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    const std::vector<Source>& src = s.rhs_fields.at(field);
    for (int i = 0; i < n; ++i) {
      cd p, dpdn;
      incident(src, s.wave.k, V3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]}, V3{0.0, 0.0, 1.0}, p, dpdn,
               &s.half_space);
      out[2 * i] = p.real();
      out[2 * i + 1] = p.imag();
    }
  });
}

// evaluate_field on the host (postproc.cpp:39-62): the checker for fpbem_cu_evaluate_field
int fh_scene_field(void* hp, int field, const double* solution, int n, const double* pts, double* out) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    const Mesh full = replicate(s.cell, s.lat);
    std::vector<cd> sol(reinterpret_cast<const cd*>(solution), reinterpret_cast<const cd*>(solution) + full.size());
    std::vector<V3> points(n);
    for (int i = 0; i < n; ++i) points[i] = V3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    const std::vector<cd> r = evaluate_field(full, sol, s.wave, s.rhs_fields.at(field), points, &s.half_space);
    std::memcpy(out, r.data(), r.size() * sizeof(cd));
  });
}

int fh_insertion_loss(int n, const double* p_inc, const double* p, double* il) {
  return guarded([&] {
    std::vector<cd> a(reinterpret_cast<const cd*>(p_inc), reinterpret_cast<const cd*>(p_inc) + n);
    std::vector<cd> b(reinterpret_cast<const cd*>(p), reinterpret_cast<const cd*>(p) + n);
    *il = insertion_loss(a, b);
  });
}

int fh_scene_dense(void* hp, double* out) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    std::vector<cd> a = assemble_dense(replicate(s.cell, s.lat), s.wave, &s.half_space);
    std::memcpy(out, a.data(), a.size() * sizeof(cd));
  });
}

// per element of the unit cell: corners (4x3), centroid (3), normal (3), area, diameter, nv
int fh_scene_cell(void* hp, double* corners, double* centroid, double* normal, double* area, double* diam, int* nv) {
  return guarded([&] {
    const Mesh& m = static_cast<SceneH*>(hp)->s.cell;
    for (int i = 0; i < m.size(); ++i) {
      const Element& e = m.el[i];
      for (int c = 0; c < 4; ++c)
        for (int d = 0; d < 3; ++d) corners[(i * 4 + c) * 3 + d] = e.c[c][d];
      for (int d = 0; d < 3; ++d) {
        centroid[3 * i + d] = e.centroid[d];
        normal[3 * i + d] = e.normal[d];
      }
      area[i] = e.area;
      diam[i] = e.diameter;
      nv[i] = e.nv;
    }
  });
}

// axis sign symmetries of the cell (cell_symmetries): returns the bitmask of
// valid g (bit 0 = identity) and perms[g * n + j] = image of element j (valid g)
int fh_cell_symmetries(void* hp, int* perms) {
  int mask = -1;
  const int rc = guarded([&] {
    const Mesh& m = static_cast<SceneH*>(hp)->s.cell;
    std::vector<std::vector<int>> perm;
    mask = cell_symmetries(m, perm);
    for (int g = 0; g < 8; ++g)
      if (mask >> g & 1)
        for (int j = 0; j < m.size(); ++j) perms[static_cast<size_t>(g) * m.size() + j] = perm[g][j];
  });
  return rc ? -1 : mask;
}

// rows = BIE-oriented cell collocation points shifted by `shift`, columns = cell elements
int fh_interaction_block(void* hp, const double* shift, int self, double* out) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    Mesh bie = bie_oriented(s.cell);
    interaction_block(s.wave, bie, V3{shift[0], shift[1], shift[2]}, bie, self != 0, reinterpret_cast<cd*>(out));
  });
}

int fh_classify(void* hp, int* n_near, int* n_far, int* near, int* far, int cap, double* grid) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    std::vector<int> nr, fr;
    classify_offsets(s.cell, s.lat, nr, fr);
    *n_near = static_cast<int>(nr.size() / 3);
    *n_far = static_cast<int>(fr.size() / 3);
    if (near && static_cast<int>(nr.size()) <= 3 * cap) std::memcpy(near, nr.data(), nr.size() * sizeof(int));
    if (far && static_cast<int>(fr.size()) <= 3 * cap) std::memcpy(far, fr.data(), fr.size() * sizeof(int));
    if (grid) {
      BoxGrid g = make_box_grid(s.cell, s.lat);
      grid[0] = g.base_center.x;
      grid[1] = g.base_center.y;
      grid[2] = g.base_center.z;
      grid[3] = g.radius;
    }
  });
}

// flags: 1 = leave the near / S_hat values empty, 2 = leave the K bank / K_hat values empty
void* fh_fmm_assemble(void* hp, int n_t, int flags) {
  FmmH* h = nullptr;
  guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    h = new FmmH{assemble_fmm(s.cell, s.lat, s.wave, n_t, (flags & 1) != 0, &s.half_space, (flags & 2) != 0)};
  });
  return h;
}

void fh_fmm_destroy(void* h) { delete static_cast<FmmH*>(h); }

// info: counts[3], n_dof, n_coef, n_near, n_far, has_near_values, mirrored_level, n_hat, n_far_hat
void fh_fmm_info(void* hp, int* info) {
  const FmmData& d = static_cast<FmmH*>(hp)->d;
  for (int k = 0; k < 3; ++k) info[k] = d.counts[k];
  info[3] = d.n_dof;
  info[4] = d.n_coef;
  info[5] = d.n_near();
  info[6] = d.n_far();
  info[7] = d.near_blocks.empty() ? 0 : 1;
  info[8] = d.mirrored_level;
  info[9] = d.n_hat();
  info[10] = d.n_far_hat();
  info[11] = (d.far_blocks.empty() && d.n_far() > 0) || (d.far_hat_blocks.empty() && d.n_far_hat() > 0) ? 0 : 1;
}

void fh_fmm_image_arrays(void* hp, const int** hat_idx, const double** hat_blk, const int** far_hat_idx,
                         const double** far_hat_blk) {
  const FmmData& d = static_cast<FmmH*>(hp)->d;
  *hat_idx = d.hat_indices.data();
  *hat_blk = reinterpret_cast<const double*>(d.hat_blocks.data());
  *far_hat_idx = d.far_hat_indices.data();
  *far_hat_blk = reinterpret_cast<const double*>(d.far_hat_blocks.data());
}

// borrowed pointers into the handle (valid until fh_fmm_destroy)
void fh_fmm_arrays(void* hp, const int** near_off, const double** near_blk, const int** far_off,
                   const double** far_blk, const double** u0, const double** v0) {
  const FmmData& d = static_cast<FmmH*>(hp)->d;
  *near_off = d.near_offsets.data();
  *near_blk = reinterpret_cast<const double*>(d.near_blocks.data());
  *far_off = d.far_offsets.data();
  *far_blk = reinterpret_cast<const double*>(d.far_blocks.data());
  *u0 = reinterpret_cast<const double*>(d.u0.data());
  *v0 = reinterpret_cast<const double*>(d.v0.data());
}

// ---- special-function probes (tests)
void fh_sph_bessel(int n_max, double x, double* j, double* y) {
  sph_bessel_j_all(n_max, x, j);
  if (y && x > 0) sph_bessel_y_all(n_max, x, y);
}
double fh_wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) { return wigner3j(j1, j2, j3, m1, m2, m3); }
int fh_solid_gradients(int n_max, const double* v, double k, double* val, double* dx, double* dy, double* dz) {
  return guarded([&] {
    SolidGrad g = solid_regular_gradients(n_max, V3{v[0], v[1], v[2]}, k);
    std::memcpy(val, g.val.data(), g.val.size() * sizeof(cd));
    std::memcpy(dx, g.dx.data(), g.dx.size() * sizeof(cd));
    std::memcpy(dy, g.dy.data(), g.dy.size() * sizeof(cd));
    std::memcpy(dz, g.dz.data(), g.dz.size() * sizeof(cd));
  });
}
int fh_solid_singular(int n_max, const double* v, double k, double* out) {
  return guarded([&] { solid_singular_all(n_max, V3{v[0], v[1], v[2]}, k, reinterpret_cast<cd*>(out)); });
}
int fh_m2l_block(int n_t, const double* delta, double k, double* out) {
  return guarded([&] {
    Translation t(n_t);
    t.m2l(V3{delta[0], delta[1], delta[2]}, k, reinterpret_cast<cd*>(out));
  });
}
int fh_expansions(void* hp, int n_t, const double* center, double* u0, double* v0) {
  return guarded([&] {
    const Scene& s = static_cast<SceneH*>(hp)->s;
    Mesh bie = bie_oriented(s.cell);
    V3 c{center[0], center[1], center[2]};
    l2p_matrix(bie, s.wave, n_t, c, reinterpret_cast<cd*>(u0));
    p2m_matrix(bie, s.wave, n_t, c, reinterpret_cast<cd*>(v0));
  });
}

}  // extern "C"
