// Launchers of the sm_100a kernels (near_field.cu, m2l.cu, krylov.cu, assembly.cu, far_bank.cu).
#pragma once

#include "common.cuh"

namespace fpbem_cu {

// ---- near field (near_field.cu)
// jobs: (block slot, first column, column count | width class << 8, pair base);
// columns are (pair, rhs) with rhs fastest, or (cell, rhs) when pair_src is null.
cudaError_t launch_block_gemm(const c64* A, long long a_stride, int lda, int M, const c64* x, c64* out, int ldo,
                              const int* pair_src, const int4* jobs, int n_jobs, int K, int n, long long N, int nrhs,
                              cudaStream_t stream, long long out_rhs_stride = 0, const int* perm = nullptr,
                              const int* items = nullptr, long long n_items = 0);
// out_rhs_stride > 0: column (unit, rhs) lands at out[rhs * out_rhs_stride + unit * ldo] (rhs-major);
// jobs with g = bits 12-14 of .z nonzero gather B rows and scatter output rows through
// perm + (g - 1) * K (the lattice near field's symmetry images)
// near field as a lattice convolution, items t in [t_lo, t_hi): for each image
// (q_i, g_i) of the item (items[t*8 + i], items[(n_items + t)*8 + i]),
// yh[r][q_i] = P_g shat_t P_g xh[r][q_i]; nrhs * nimg <= kModeGemvMaxAcc
constexpr int kModeGemvMaxAcc = 8;
// The same product on DMMA tiles with a bulk-copy ring of the stored blocks
// (nrhs * nimg <= 8 columns, n % 8 == 0; mode_mma_shape says whether it applies)
bool mode_mma_shape(int n, int ncols, int* nw, int* kc, int* ring, size_t* smem);
cudaError_t launch_mode_mma(const c64* shat, const int* items, long long n_items, const int* perm, const c64* xh,
                            c64* yh, int n, long long t_lo, long long t_hi, long long q_stride, int nrhs, int nimg,
                            cudaStream_t stream);
// out[col] (+)= A in[col] per (cell, rhs) column col = cell * nrhs + r, A[m][k] =
// a[m a_ms + k a_ks] (M x K): the P2M product on DMMA (csrc/cellwise.cu)
bool cellwise_supported(int M, int K);
cudaError_t launch_cellwise(const c64* a, long long a_ms, long long a_ks, int M, int K, const c64* in, long long in_rs,
                            long long in_cs, c64* out, long long out_rs, long long out_cs, int nrhs, long long ncols,
                            bool accumulate, cudaStream_t stream);
cudaError_t launch_mode_gemv(const c64* shat, const int* items, long long n_items, const int* perm, const c64* xh,
                             c64* yh, int n, long long t_lo, long long t_hi, long long q_stride, int nrhs, int nimg,
                             cudaStream_t stream);
// cell-symmetry check: out2[0] = max |S_mirror[s][P i, P j] - S_s[i, j]|, out2[1] = max |S| (double bits)
cudaError_t launch_near_symmetry(const c64* S, int n, int n_blk, const int* mirror, const int* perm,
                                 unsigned long long* out2, cudaStream_t stream);
// y += U0 L per (cell, rhs) (the lattice path's L2P; bitwise = the reduction with no pairs)
cudaError_t launch_l2p_add(const c64* u0, const c64* local, c64* y, int n, int n_coef, int n_cells, long long N,
                           int nrhs, cudaStream_t stream);
cudaError_t launch_near_reduce_l2p(const c64* W, const int* tgt_ptr, const int* tgt_pairs, const c64* u0,
                                   const c64* local, c64* y, int n, int n_coef, int n_cells, long long N,
                                   int nrhs, bool accumulate, cudaStream_t stream);

// ---- M2L / P2M (m2l.cu)
// The last inverse near-field pass (x axis) with the L2P fused: out = scale DFT(in)
// + U0 L_cell (n_in <= 32, b <= 32; lines a = r * (My Mz) + line, nrhs | n_a)
bool dft_l2p_supported(int n_in, int n_out, int b);
cudaError_t launch_dft_axis_l2p(const c64* in, c64* out, const c64* tw, long long n_a, int n_in, int n_out,
                                long long n_inner, int L, double scale, const c64* u0, const c64* loc, int b, int nrhs,
                                cudaStream_t stream);
cudaError_t launch_dft_axis(const c64* in, c64* out, const c64* tw, long long n_a, int n_in, int n_out,
                            long long n_inner, int L, bool backward, double scale, cudaStream_t stream);
cudaError_t launch_mode_product(const c64* lambda, const c64* field, c64* image, long long q_total, int b,
                                int nrhs, cudaStream_t stream);
// fused forward-z DFT + mode product + inverse-z DFT, one CTA per (qy, qx) column
// ring depth (Λ mode blocks in shared memory) of the fused z kernel, 0 when
// the column's fields leave no room for >= 4 (then the unfused passes run)
// the flat Λ stream (in place on the z-extended field): ring slots, 0 when the shape is not supported
int mode_stream_ring(int E, int b);
// quad: the spectrum also has the z-reflection parity, units run over qz <= Lz/2 only
cudaError_t launch_mode_stream(c64* field, const c64* lambda, int Lz, long long plane, int E, int b,
                               const int2* items, int n_items, bool quad, cudaStream_t stream);
int m2l_zfused_ring(int Mz, int Lz, int E, int b);
cudaError_t launch_m2l_zfused(const c64* in, c64* out, const c64* lambda, const c64* tw, int Mz, int Lz,
                              long long plane, int E, int b, double scale, const int2* items, int n_items,
                              cudaStream_t stream);
// Λ(-q) = D Λ(q) D check (D = diag((-1)^n)): out2[0] = max deviation, out2[1] = max |Λ|, as double bits
cudaError_t launch_lambda_parity(const c64* lam, const int L[3], int b, bool zflip, unsigned long long* out2,
                                 cudaStream_t stream);
cudaError_t launch_mirror_permute(const c64* in, c64* out, const int counts[3], int level, long long E,
                                  cudaStream_t stream);
cudaError_t launch_add(c64* acc, const c64* v, long long n, cudaStream_t stream);
cudaError_t launch_scatter_bank(const c64* blocks, const int* offsets, int n_blk, int b2, int lx, int ly, int lz,
                                c64* field, cudaStream_t stream);

// ---- near-field block assembly (assembly.cu)
struct AssemblySlot {
  double tshift[3];  // target (collocation point) shift
  double sshift[3];  // source element shift, applied before the optional mirror
  c64 scale;         // entry multiplier (1, or the reflection coefficient)
  int mirror;        // source element mirrored in the half-space plane
  int self;          // slot holds the self block (i == j -> singular self term)
};
cudaError_t assembly_set_rules(const double* x6, const double* w6, const double* x8, const double* w8);
cudaError_t launch_assemble(const double* corners, const int* nv, const double* cen, const double* nrm,
                            const double* diam, const c64* beta, int n, const AssemblySlot* slots, int n_slots,
                            double k, c64 alpha, int hs_axis, double hs_offset, c64* out, bool accumulate,
                            cudaStream_t stream);

// ---- Krylov vector ops (krylov.cu)
constexpr int kRedBlocks = 2 * kNumSMs;
struct RedScratch {
  double* partial_d;  // kRedBlocks
  c64* partial_c;     // kRedBlocks
  unsigned* counter;  // 1, zero between launches
};
cudaError_t launch_sqnorm(const c64* w, long long n, const RedScratch& rs, double* result, int* nonfinite,
                          cudaStream_t s);
cudaError_t launch_dotc(const c64* a, const c64* b, long long n, const RedScratch& rs, c64* result,
                        cudaStream_t s);
cudaError_t launch_axpy_dotc(c64* w, const c64* v, const c64* h, const c64* vn, long long n, const RedScratch& rs,
                             c64* result, cudaStream_t s);
cudaError_t launch_axpy_sqnorm(c64* w, const c64* v, const c64* h, long long n, const RedScratch& rs,
                               double* result, cudaStream_t s);
cudaError_t launch_div(const c64* in, c64* out, long long n, double d, cudaStream_t s);
cudaError_t launch_update_x(c64* x, const c64* basis, long long ld, const c64* y, int j, long long n,
                            cudaStream_t s);
// whole MGS sequence of one Arnoldi step in one cooperative launch:
// norms[0] = ||w||^2 (if do_pre, + non-finite flag), h_out[0..j], norms[1] = ||w||^2 after
bool mgs_fused_supported(long long n);
// hc_out != null (needs do_pre): the whole Arnoldi step in the launch — the conditional
// second pass into hc_out, norms[2] = final ||w||^2, norms[4] = 1 if reorthogonalised,
// norms[5] = h_{j+1,j} = ||w||, and w normalised by it (if > 0)
cudaError_t launch_mgs_fused(c64* w, const c64* V, long long ld, int j, long long n, c64* h_out, double* norms,
                             int* nonfinite, const RedScratch& rs, bool do_pre, cudaStream_t s,
                             c64* hc_out = nullptr);
// ---- batched (lockstep multi-RHS) vector ops: G right-hand sides at stride ld
constexpr int kBatchBlocks = 64;  // blocks per RHS (upper bound)
struct BatchScratch {
  double* partial_d;  // G * kBatchBlocks
  c64* partial_c;     // G * kBatchBlocks
  unsigned* counter;  // G, zero between launches
};
cudaError_t launch_b_sqnorm(const c64* w, long long ld, long long n, int G, const int* mask, const BatchScratch& bs,
                            double* result, int* nonfinite, cudaStream_t s);
cudaError_t launch_b_dotc(const c64* a, const c64* b, long long ld, long long n, int G, const int* mask,
                          const BatchScratch& bs, c64* result, cudaStream_t s);
cudaError_t launch_b_axpy_dotc(c64* w, const c64* v, const c64* h, const c64* vn, long long ld, long long n, int G,
                               const int* mask, const BatchScratch& bs, c64* result, cudaStream_t s);
cudaError_t launch_b_axpy_sqnorm(c64* w, const c64* v, const c64* h, long long ld, long long n, int G,
                                 const int* mask, const BatchScratch& bs, double* result, cudaStream_t s);
cudaError_t launch_b_div(const c64* in, c64* out, long long ld, long long n, int G, const int* mask, const double* d,
                         cudaStream_t s);
cudaError_t launch_b_update_x(c64* x, const c64* basis, int G, long long ld, const c64* y, int ystride,
                              const int* jr, long long n, const int* mask, cudaStream_t s);
cudaError_t launch_b_residual(const c64* b, const c64* ax, c64* res, long long ld, long long n, int G, const int* mask,
                              const BatchScratch& bs, double* result, int* nonfinite, cudaStream_t s);
cudaError_t launch_b_pack(const c64* src, c64* dst, const int* idx, int count, long long n, bool gather,
                          cudaStream_t s);
// classical Gram-Schmidt passes of the distributed GMRES (krylov.cu):
// partials hold (cols + 1) x kCgsMaxBlocks complex; cols < kCgsMaxCols
constexpr int kCgsMaxBlocks = 4 * kNumSMs;
constexpr int kCgsMaxCols = 1024;
cudaError_t launch_cgs_dots(const c64* V, long long ld, int cols, const c64* w, long long n, c64* partials,
                            unsigned* counter, c64* out, cudaStream_t s);
cudaError_t launch_cgs_update(c64* w, const c64* V, long long ld, int cols, const c64* h, long long n,
                              double* partials, unsigned* counter, double* result, cudaStream_t s);
cudaError_t launch_residual(const c64* b, const c64* ax, c64* r, long long n, const RedScratch& rs,
                            double* result, cudaStream_t s);

// field evaluation (csrc/assembly.cu): out[p] = p_inc[p] + sum over the replicated
// mesh (+ reflection x its mirror) of the representation-formula contributions;
// partial: field_chunks(n * cells) x n_pts scratch
int field_chunks(long long n_total);
cudaError_t launch_field(const double* corners, const int* nv, const double* cen, const double* nrm,
                         const double* diam, const c64* beta, int n, const int counts[3], const double pitch[3],
                         const c64* solution, const double* pts, int n_pts, const c64* p_inc, double k,
                         bool with_image, int hs_axis, double hs_offset, c64 refl, c64* partial, c64* out,
                         cudaStream_t stream);

// x and y lattice DFTs of every z-plane and field in one kernel (csrc/m2l.cu):
// forward moments [iz][iy][ix][E] -> [iz][qy][qx][E]; inverse the reverse with
// the scale; xy_plane_smem bytes of shared memory per CTA
size_t xy_plane_smem(int Mx, int My, int Lx, int Ly, bool inverse);
cudaError_t launch_xy_plane(const c64* in, c64* out, const c64* twx, const c64* twy, int Mx, int My, int Lx, int Ly,
                            int Mz, int E, bool inverse, double scale, cudaStream_t stream);

// P2M (csrc/m2l.cu): mom[(cell * nrhs + r) * b + c] = sum_j V0[c][j] x[r * N + cell * n + j], v0t = V0^T rows
cudaError_t launch_p2m(const c64* v0t, const c64* x, c64* mom, int n, int b, long long N, int nrhs, int cells,
                       cudaStream_t stream);

// device M2L bank (csrc/far_bank.cu): out[s] = [K(delta_s)] + refl K(image_s) P_axis
int far_bank_max_nt();
cudaError_t launch_far_bank(int device, int n_t, double k, int n_blk, const double* delta, const double* image,
                            int parity_axis, c64 refl, c64* out, cudaStream_t stream);

}  // namespace fpbem_cu
