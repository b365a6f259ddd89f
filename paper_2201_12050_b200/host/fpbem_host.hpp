// Host-side operator producer for the periodic FMBEM hot path.
//
// This is the C++ layer that sits ABOVE the CUDA C-ABI (include/fpbem_cuda.h):
// it builds the unit-cell mesh, classifies lattice offsets into near / far,
// assembles the near-field Toeplitz blocks S_o, the far-field M2L bank K_o and
// the shared expansion matrices U0 (L2P) and V0 (P2M), and the right-hand side.
// It restates the reference's host assembly (out of the hot-path scope, but
// needed to produce realistic operator data):
//   geometry   /root/reference/proj/src/geometry.cpp:14-196
//   kernels    /root/reference/proj/src/kernels.cpp:13-325
//   specfun    /root/reference/proj/src/specfun.cpp:12-372
//   assembly   /root/reference/proj/src/assembly.cpp:17-21, 214-251
//   fmm build  /root/reference/proj/src/fmm.cpp:22-65, 125-190
// Extensions the BASELINE configs need and the reference lacks (parity
// unpinned): flat triangles (stored as a 3-corner
// polygon; the planar self-term runs edge by edge), icosphere / closed
// cylinder / closed box generators.
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <string>
#include <vector>

namespace fpbem_host {

using cd = std::complex<double>;
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr cd kI{0.0, 1.0};

struct V3 {
  double x = 0, y = 0, z = 0;
  V3() = default;
  V3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int d) const { return d == 0 ? x : (d == 1 ? y : z); }
  double& operator[](int d) { return d == 0 ? x : (d == 1 ? y : z); }
};
inline V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator-(const V3& a) { return {-a.x, -a.y, -a.z}; }
inline V3 operator*(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator*(const V3& a, double s) { return s * a; }
inline V3 operator/(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const V3& a) { return std::sqrt(dot(a, a)); }
inline V3 unit(const V3& a) { return a / norm(a); }

// Frequency-dependent scalars (include/fpbem/types.hpp:24-49). alpha = -i/k.
struct Wave {
  double k = 1.0;
  cd alpha{0.0, -1.0};
  static Wave from_k(double k) { return {k, cd(0.0, -1.0 / k)}; }
  static Wave from_frequency(double f, double c) { return from_k(2.0 * kPi * f / c); }
};

// Flat polygon element with constant collocation: 4 corners (quad), or a
// triangle stored with corner[3] == corner[2] and nv == 3.
struct Element {
  std::array<V3, 4> c;
  int nv = 4;
  V3 centroid;
  V3 normal;
  double area = 0;
  double diameter = 0;
  cd beta{0.0, 0.0};
};

Element make_quad(const V3& a, const V3& b, const V3& c, const V3& d, cd beta = {});
Element make_tri(const V3& a, const V3& b, const V3& c, cd beta = {});

struct Mesh {
  std::vector<Element> el;
  int size() const { return static_cast<int>(el.size()); }
  void bbox(V3& lo, V3& hi) const;
};

// generators
Mesh cube_sphere(double radius, int refinement, cd beta = {});           // geometry.cpp:67-109
Mesh wall_cell(double ly, double lz, double t, int div, cd beta = {});    // geometry.cpp:111-135
Mesh icosphere(double radius, int subdivisions, cd beta = {});            // extension
// axis sign maps g (bit d flips axis d about the bbox centre) leaving the mesh invariant:
// bitmask of valid g (bit 0 = identity), perm[g][j] = image element of j (extension)
int cell_symmetries(const Mesh& m, std::vector<std::vector<int>>& perm);
// images of each orbit's representative get the images of its quadrature nodes (extension)
void symmetrize_group(Mesh& m);
Mesh closed_cylinder(double radius, double height, int n_theta, int n_z, cd beta = {});  // extension
Mesh closed_box(double lx, double ly, double lz, double h, bool split_triangles,
                cd beta = {});  // extension; box [-lx/2,lx/2]x[-ly/2,ly/2]x[0,lz]

struct Lattice {
  std::array<int, 3> counts{1, 1, 1};
  std::array<double, 3> pitch{0, 0, 0};
  int cells() const { return counts[0] * counts[1] * counts[2]; }
  V3 shift(int ix, int iy, int iz) const { return {ix * pitch[0], iy * pitch[1], iz * pitch[2]}; }
};

Mesh replicate(const Mesh& cell, const Lattice& lat);

// Axis-aligned mirror plane with a constant complex reflection coefficient
// (geometry.hpp:66-78); mirror_mesh reverses the corner loop and keeps the
// source orientation with the mirrored normal (geometry.cpp:157-178).
struct HalfSpace {
  int axis = 2;
  double offset = 0.0;
  cd reflection{0.0, 0.0};
  bool active() const { return reflection != cd(0.0, 0.0); }
};
V3 mirror_point(const V3& p, const HalfSpace& hs);
Mesh mirror_mesh(const Mesh& m, const HalfSpace& hs);
Mesh bie_oriented(const Mesh& m);  // normals flipped once (assembly.cpp:17-21)

struct BoxGrid {  // geometry.cpp:180-191
  V3 base_center;
  double radius = 0;
};
BoxGrid make_box_grid(const Mesh& cell, const Lattice& lat);
bool admissible(const V3& a, const V3& b, double r);  // |a-b| >= 2r, inclusive (geometry.cpp:193-196)

// quadrature (kernels.hpp:17-20, kernels.cpp:162-212)
inline constexpr int kRegularOrder = 6;
inline constexpr int kSelfOrder = 8;
inline constexpr double kNearFactor = 3.0;
inline constexpr int kMaxSubdivision = 6;
struct QPoint {
  V3 y;
  double w;
};
void gauss_legendre(int order, std::vector<double>& nodes, std::vector<double>& weights);
void tensor_points(const Element& e, int order, std::vector<QPoint>& out);
void influence_points(const Element& e, const V3& x, int order, std::vector<QPoint>& out);

// Burton-Miller influence of one BIE-oriented element (kernels.cpp:214-261,
// assembly.cpp:214-223)
struct Influence {
  cd h{0, 0}, g{0, 0};
};
Influence influence(const Wave& w, const Element& src, const V3& x, const V3& nx);
Influence influence_self(const Wave& w, const Element& src);
cd bm_entry(const Wave& w, const Element& src, const V3& x, const V3& nx, bool self);

// incident field (kernels.cpp:263-325, without half-space images)
struct Source {
  bool plane = true;
  V3 v;  // unit direction or position
  cd amp{1.0, 0.0};
};
void incident(const std::vector<Source>& src, double k, const V3& x, const V3& nx, cd& p, cd& dpdn,
              const HalfSpace* hs = nullptr);
// rhs = p_inc + alpha dp_inc/dn at centroids with BIE normals (assembly.cpp:241-251)
std::vector<cd> assemble_rhs(const Mesh& full, const Wave& w, const std::vector<Source>& src,
                             const HalfSpace* hs = nullptr);

// representation formula at observation points and the insertion loss
// (postproc.cpp:18-81); `full` is the replicated mesh in its stored orientation
std::vector<cd> evaluate_field(const Mesh& full, const std::vector<cd>& solution, const Wave& w,
                               const std::vector<Source>& src, const std::vector<V3>& points,
                               const HalfSpace* hs = nullptr);
double insertion_loss(const std::vector<cd>& p_inc, const std::vector<cd>& p);

// special functions (specfun.hpp)
inline constexpr int flat(int n, int m) { return n * n + n + m; }
inline constexpr int coef_count(int n_t) { return (n_t + 1) * (n_t + 1); }
void sph_bessel_j_all(int n_max, double x, double* out);
void sph_bessel_y_all(int n_max, double x, double* out);
double wigner3j(int j1, int j2, int j3, int m1, int m2, int m3);
double trans_coeff(int n, int m, int np, int mp, int l);
void solid_regular_all(int n_max, const V3& v, double k, cd* out);
void solid_singular_all(int n_max, const V3& v, double k, cd* out);
struct SolidGrad {
  std::vector<cd> val, dx, dy, dz;
};
SolidGrad solid_regular_gradients(int n_max, const V3& v, double k);

// M2L / regular-shift translation table (specfun.cpp:305-372)
class Translation {
 public:
  explicit Translation(int n_t);
  int n_t() const { return n_t_; }
  // b x b column-major block, b = (n_t+1)^2
  void m2l(const V3& delta, double k, cd* out) const;
  void regular_shift(const V3& s, double k, cd* out) const;

 private:
  struct Term {
    int l;
    double c;
  };
  int n_t_;
  std::vector<std::vector<Term>> m2l_, shift_;
};

// shared expansion matrices (fmm.cpp:22-65); column-major
void p2m_matrix(const Mesh& cell_bie, const Wave& w, int n_t, const V3& center, cd* v0 /*b x n*/);
void l2p_matrix(const Mesh& cell_bie, const Wave& w, int n_t, const V3& center, cd* u0 /*n x b*/);

// interaction block: rows = collocation points of target (shifted), columns =
// source elements; column-major n_t x n_s (assembly.cpp:225-239)
void interaction_block(const Wave& w, const Mesh& target_bie, const V3& shift, const Mesh& source_bie,
                       bool self_terms, cd* out);

// Assembled operator data consumed by the CUDA C-ABI (fmm.hpp:54-71, minus Λ:
// the GPU builds the spectrum from the far bank, or the caller supplies it).
struct FmmData {
  std::array<int, 3> counts{1, 1, 1};
  int n_dof = 0;
  int n_t = 4;
  int n_coef = 25;
  BoxGrid grid;
  std::vector<int> near_offsets;  // 3 per block, loop order z, y, x ascending
  std::vector<cd> near_blocks;    // n_near * n_dof^2
  std::vector<int> far_offsets;   // 3 per block
  std::vector<cd> far_blocks;     // n_far * n_coef^2
  std::vector<cd> u0, v0;
  // half space whose mirror axis is periodic: block Hankel image pair
  // (S_hat, K_hat), indexed by the cell-index sum along the mirrored level
  int mirrored_level = -1;
  std::vector<int> hat_indices;      // 3 per S_hat block
  std::vector<cd> hat_blocks;        // n_hat * n_dof^2
  std::vector<int> far_hat_indices;  // 3 per K_hat block
  std::vector<cd> far_hat_blocks;    // n_far_hat * n_coef^2
  int n_near() const { return static_cast<int>(near_offsets.size() / 3); }
  int n_far() const { return static_cast<int>(far_offsets.size() / 3); }
  int n_hat() const { return static_cast<int>(hat_indices.size() / 3); }
  int n_far_hat() const { return static_cast<int>(far_hat_indices.size() / 3); }
};

// Offset classification only (no block values); same loop as the assembly.
void classify_offsets(const Mesh& cell, const Lattice& lat, std::vector<int>& near,
                      std::vector<int>& far);

// assemble_periodic_fmm (fmm.cpp:125-242). skip_near_values leaves the near
// (and S_hat) blocks empty, skip_far_values the K bank (and K_hat) blocks, for
// runs that assemble those on the device; offsets and indices are always set.
FmmData assemble_fmm(const Mesh& cell, const Lattice& lat, const Wave& w, int n_t,
                     bool skip_near_values = false, const HalfSpace* hs = nullptr, bool skip_far_values = false);

// action of an axis mirror on moment vectors (fmm.cpp:108-123); b x b column-major
void mirror_parity_map(int n_t, int axis, cd* out);

// Dense collocation matrix of a full mesh (assembly.cpp:253-276)
std::vector<cd> assemble_dense(const Mesh& full, const Wave& w, const HalfSpace* hs = nullptr);

// The five BASELINE.json configurations (and reference-pinned quad variants).
struct Scene {
  std::string name;
  Mesh cell;
  Lattice lat;
  Wave wave;
  std::vector<std::vector<Source>> rhs_fields;  // one field per right-hand side
  std::vector<double> sweep_hz;                 // cfg4 frequency sweep (empty otherwise)
  HalfSpace half_space;                         // inactive unless reflection != 0
  double sound_speed = 343.0;
};
Scene make_scene(int config_id, int variant);

}  // namespace fpbem_host
