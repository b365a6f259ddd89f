// C++-only drop-in path: the host side stays C++ (scene, assembly — the
// reference's FmmOperators producer, restated in paper_2201_12050_b200/host)
// and calls the device through the C-ABI shim (include/fpbem_cuda.hpp), as
// make_backend + run_scene would (src/scene.cpp:291-329, 446): assemble the
// operator, hand its data to fpbem_cu_fmm_create, apply it once, solve the
// first right-hand side with the device GMRES. Writes the product and the
// solution as raw complex128 so a test can compare them with the oracle.
//
//   cpp_scene_solve <config> <variant> <x.bin in> <y.bin out> <solution.bin out>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "fpbem_cuda.hpp"
#include "fpbem_host.hpp"

using namespace fpbem_host;

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s config variant x.bin y.bin solution.bin\n", argv[0]);
    return 2;
  }
  const int cid = std::atoi(argv[1]), var = std::atoi(argv[2]);
  const Scene sc = make_scene(cid, var);
  const FmmData op = assemble_fmm(sc.cell, sc.lat, sc.wave, 4, false, &sc.half_space);
  const Mesh full = replicate(sc.cell, sc.lat);
  const std::vector<cd> rhs = assemble_rhs(full, sc.wave, sc.rhs_fields.at(0), &sc.half_space);
  const size_t N = rhs.size();

  // FmmOperators -> fpbem_cu_fmm_desc
  fpbem_cu_fmm_desc d{};
  for (int k = 0; k < 3; ++k) d.counts[k] = op.counts[k];
  d.n_dof = op.n_dof;
  d.n_coef = op.n_coef;
  d.n_near = op.n_near();
  d.near_offsets = op.near_offsets.data();
  d.near_blocks = reinterpret_cast<const fpbem_c64*>(op.near_blocks.data());
  d.u0 = reinterpret_cast<const fpbem_c64*>(op.u0.data());
  d.v0 = reinterpret_cast<const fpbem_c64*>(op.v0.data());
  d.n_far = op.n_far();
  d.far_offsets = op.far_offsets.data();
  d.far_blocks = reinterpret_cast<const fpbem_c64*>(op.far_blocks.data());
  d.mirrored_level = op.mirrored_level;
  d.max_rhs = 1;
  // the cell's axis-sign symmetries (verified by the library on the blocks)
  std::vector<std::vector<int>> perm;
  const int mask = cell_symmetries(sc.cell, perm);
  std::vector<int> axes, perms;
  for (int g = 1; g < 8; ++g)
    if (mask >> g & 1) {
      axes.push_back(g);
      perms.insert(perms.end(), perm[g].begin(), perm[g].end());
    }
  d.n_sym = static_cast<int>(axes.size());
  d.sym_axes = axes.data();
  d.sym_perms = perms.data();

  fpbem_cuda::DeviceFmm dev(d, 0);
  int per_block = 1;
  const int path = dev.near_path(&per_block);

  std::vector<std::complex<double>> x(N);
  std::ifstream(argv[3], std::ios::binary).read(reinterpret_cast<char*>(x.data()), N * sizeof(cd));
  const std::vector<std::complex<double>> y = dev.apply(x);
  std::ofstream(argv[4], std::ios::binary).write(reinterpret_cast<const char*>(y.data()), N * sizeof(cd));

  const fpbem_cuda::SolveReport rep = dev.gmres(rhs, 1e-6, 50, 1000);
  std::ofstream(argv[5], std::ios::binary)
      .write(reinterpret_cast<const char*>(rep.solution.data()), N * sizeof(cd));
  std::printf("N %zu near_path %s modes_per_block %d iterations %d converged %d\n", N,
              path == FPBEM_CU_NEAR_LATTICE ? "lattice" : "direct", per_block, rep.iterations, rep.converged ? 1 : 0);
  return 0;
}
