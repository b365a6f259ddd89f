/*
 * fpbem_cuda.h — C-ABI of the B200-native periodic-FMBEM hot path.
 *
 * Drop-in boundary for the reference's operator product and Krylov solver
 * (arXiv 2201.12050 "fpbem", /root/reference/proj):
 *
 *   fpbem_cu_fmm_create   replaces the data hand-off of FmmOperators
 *                         (include/fpbem/fmm.hpp:54-71) into the backend
 *                         built by make_backend (src/scene.cpp:323-327)
 *   fpbem_cu_fmm_apply    replaces FmmOperators::matvec (src/fmm.cpp:246-271)
 *                         i.e. the solver::ApplyFn (include/fpbem/solver.hpp:21)
 *   fpbem_cu_gmres        replaces solver::gmres (src/solver.cpp:21-123,
 *                         include/fpbem/solver.hpp:14-33) with a device-
 *                         resident Krylov basis
 *   fpbem_cu_fmm_bytes    replaces FmmOperators::stored_bytes (src/fmm.cpp:273-279)
 *   fpbem_cu_spectrum     exposes CirculantSpectrum::lambda (include/fpbem/structured.hpp:41)
 *                         when the spectrum was built on the device
 *
 * Plain pointers and sizes only; complex numbers are interleaved (re, im)
 * doubles, layout-identical to std::complex<double> / Eigen::VectorXcd.
 * Vector layout is the reference's: cell-major, x index fastest, then y,
 * then z, n_dof entries per cell (include/fpbem/geometry.hpp:53-62). With
 * nrhs > 1 the right-hand sides are stored one after another (x[r*N + i]).
 *
 * Errors: every int-returning call returns FPBEM_CU_OK (0) or one of the
 * codes below; fpbem_cu_last_error() gives the message of the calling
 * thread's last failure. The C++ shim (include/fpbem_cuda.hpp) maps
 * FPBEM_CU_EDIM to std::invalid_argument and everything else to
 * std::runtime_error, as the reference throws (src/fmm.cpp:250,
 * src/solver.cpp:15).
 */
#ifndef FPBEM_CUDA_H
#define FPBEM_CUDA_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPBEM_CU_OK 0
#define FPBEM_CU_EDIM 1       /* dimension mismatch  -> std::invalid_argument */
#define FPBEM_CU_ENONFINITE 2 /* operator produced NaN/Inf -> runtime_error   */
#define FPBEM_CU_ECUDA 3      /* CUDA runtime failure                         */
#define FPBEM_CU_ENOMEM 4     /* device allocation failed                     */
#define FPBEM_CU_ENCCL 5      /* NCCL failure (multi-GPU)                      */
#define FPBEM_CU_EINVAL 6     /* invalid argument / unsupported option        */

#define FPBEM_CU_PTR_HOST 0   /* x / y are host pointers (copies inside call) */
#define FPBEM_CU_PTR_DEVICE 1 /* x / y are device pointers (stream-ordered)   */

typedef struct {
  double re, im;
} fpbem_c64;

typedef struct fpbem_cu_op fpbem_cu_op;     /* opaque; owns device memory and stream */
typedef struct fpbem_cu_comm fpbem_cu_comm; /* opaque NCCL communicator             */

/* Operator description: FmmOperators' fields (include/fpbem/fmm.hpp:54-71).
 * Host arrays are copied at create; the caller keeps ownership. */
typedef struct {
  int counts[3];                 /* lattice cells per axis (Lattice::counts)              */
  int n_dof;                     /* elements per cell (S block dim)                       */
  int n_coef;                    /* (n_t+1)^2 expansion coefficients                      */
  int n_near;                    /* |S|: stored near offsets                              */
  const int* near_offsets;       /* n_near x 3 (ox,oy,oz) = target - source, in
                                    BlockToeplitzMatrix::offsets order                    */
  const fpbem_c64* near_blocks;  /* n_near x n_dof^2, each column-major (row = target)    */
  const fpbem_c64* u0;           /* L2P: n_dof x n_coef, column-major                      */
  const fpbem_c64* v0;           /* P2M: n_coef x n_dof, column-major                      */
  int fft_sizes[3];              /* circulant embedding lengths; 0 = reference 7-smooth
                                    padding fft_friendly(2M-1) (src/structured.cpp:67-68)  */
  const fpbem_c64* lambda;       /* optional prebuilt spectrum: q x n_coef^2 column-major
                                    blocks, q = (qz*Ly+qy)*Lx+qx (src/structured.cpp:80-86) */
  int n_far;                     /* far offsets (used when lambda == NULL)                */
  const int* far_offsets;        /* n_far x 3                                             */
  const fpbem_c64* far_blocks;   /* n_far x n_coef^2 M2L bank K, column-major; the device
                                    builds the spectrum (src/structured.cpp:63-108)        */
  int mirrored_level;            /* -1: no half-space image pair; else the mirrored level  */
  int max_rhs;                   /* largest nrhs passed to apply/gmres (workspace sizing)  */
  /* half-space image pair (FmmOperators::near_field_image / k_image_spectrum,
   * include/fpbem/fmm.hpp:66-68), used when mirrored_level >= 0. Indices are
   * the reference's BlockHankelMatrix indices: the cell-index SUM in
   * [0, 2M-2] along the mirrored level, offsets target - source elsewhere. */
  int n_hat;                     /* S_hat blocks                                           */
  const int* hat_indices;        /* n_hat x 3                                              */
  const fpbem_c64* hat_blocks;   /* n_hat x n_dof^2, column-major                          */
  int n_far_hat;                 /* K_hat bank (the device builds the spectrum of K_hat P) */
  const int* far_hat_indices;    /* n_far_hat x 3                                          */
  const fpbem_c64* far_hat_blocks; /* n_far_hat x n_coef^2                                 */
  const fpbem_c64* lambda_hat;   /* optional prebuilt spectrum of K_hat P (the reference's
                                    k_image_spectrum, same layout as lambda); else built
                                    from the K_hat bank                                    */
  int blocks_on_device;          /* 1: near_blocks / hat_blocks are device pointers on
                                    `device` (e.g. from fpbem_cu_assemble_near)            */
  int far_on_device;             /* 1: far_blocks / far_hat_blocks are device pointers on
                                    `device` (e.g. from fpbem_cu_m2l_bank)                 */
  int near_path;                 /* FPBEM_CU_NEAR_*: how the Toeplitz near field S p is
                                    applied (same product, different arithmetic order)    */
  int n_sym;                     /* optional (extension): cell symmetries, 0 if none      */
  const int* sym_axes;           /* n_sym axis-sign maps g in 1..7: bit d flips axis d
                                    about the cell centre (mirrors, half-turns, inversion) */
  const int* sym_perms;          /* n_sym x n_dof: element j -> its image under g. Every g
                                    the device verifies (S_{A_g o}[P i, P j] == S_o[i, j]
                                    to 1e-12 max |S|, A_g o = o with the flipped axes
                                    negated) lets the lattice near field store one block
                                    per orbit of Fourier modes                             */
} fpbem_cu_fmm_desc;

#define FPBEM_CU_NEAR_AUTO 0       /* cost model picks (fpbem_cu_fmm_near_path reports it)   */
#define FPBEM_CU_NEAR_DIRECT 1     /* one GEMM per stored offset over its valid targets, as
                                      BlockToeplitzMatrix::matvec (src/assembly.cpp:62-84)  */
#define FPBEM_CU_NEAR_LATTICE 2    /* circulant embedding of the blocks in an (M + max|o|)
                                      lattice, DFT'd once at create; per apply: pruned DFT of
                                      x, one n x n block product per mode, pruned inverse
                                      (no half-space image pair)                            */

/* Unit cell for the device assembly, BIE-oriented (assembly::bie_oriented,
 * src/assembly.cpp:17-21): flat quads, or triangles with corner 3 == corner 2. */
typedef struct {
  int n;                    /* elements                                    */
  const double* corners;    /* n x 4 x 3                                   */
  const int* nv;            /* n: 4 (quad) or 3 (triangle)                 */
  const double* centroid;   /* n x 3                                       */
  const double* normal;     /* n x 3, BIE orientation                      */
  const double* diameter;   /* n                                           */
  const fpbem_c64* beta;    /* n normalised admittances, or NULL (rigid)   */
} fpbem_cu_cell;

/* Near-field blocks of assemble_periodic_fmm on the device (src/fmm.cpp:156-179,
 * src/assembly.cpp:214-239): out[s] = interaction_block(cell, shift(offsets[s]),
 * cell, self = (offset == 0)), n x n column-major, plus
 * hs_reflection * interaction_block(cell, shift, mirror(cell)) when fold != 0
 * (half space parallel to every periodic axis). ptr_kind: FPBEM_CU_PTR_HOST or
 * FPBEM_CU_PTR_DEVICE (out on `device`). */
int fpbem_cu_assemble_near(const fpbem_cu_cell* cell, double k, fpbem_c64 alpha, const double pitch[3],
                           int n_off, const int* offsets, int fold, int hs_axis, double hs_offset,
                           fpbem_c64 hs_reflection, int device, fpbem_c64* out, int ptr_kind);

/* S_hat blocks of a split half space (src/fmm.cpp:204-231): for Hankel index
 * idx, target shift = shift(tgt), source = mirror(cell shifted by shift(src))
 * with tgt/src as the reference picks them, scaled by hs_reflection. */
int fpbem_cu_assemble_hat(const fpbem_cu_cell* cell, double k, fpbem_c64 alpha, const double pitch[3],
                          const int counts[3], int n_hat, const int* hat_indices, int hs_axis,
                          double hs_offset, fpbem_c64 hs_reflection, int device, fpbem_c64* out,
                          int ptr_kind);

/* Pressure at observation points by the representation formula
 * (postproc::evaluate_field, src/postproc.cpp:39-62): for each point x,
 *   out = p_incident + sum_j int_{e_j} [-dG/dn_y p_j + G i k beta_j p_j]
 *         (+ hs_reflection x the same over the mirrored mesh when hs_reflection != 0),
 * over the replicated mesh (cell-major, x fastest) of the BIE-oriented unit
 * cell, with the influence quadrature of src/kernels.cpp:205-212 (order 6,
 * adaptive subdivision near x). solution: N = n x cells pressures;
 * p_incident: n_points values or NULL (0); points: host n_points x 3.
 * ptr_kind applies to solution, p_incident and out. */
int fpbem_cu_evaluate_field(const fpbem_cu_cell* cell, double k, const double pitch[3], const int counts[3],
                            const fpbem_c64* solution, int n_points, const double* points,
                            const fpbem_c64* p_incident, int hs_axis, double hs_offset, fpbem_c64 hs_reflection,
                            int device, fpbem_c64* out, int ptr_kind);

/* M2L translation blocks on the device: TranslationTable::m2l
 * (src/specfun.cpp:332-351) batched over n_blk translation vectors,
 *   out[s] = K(delta[s]) + reflection * K(image_delta[s]) P_axis,
 * each b x b column-major, b = (n_t+1)^2 (n_t <= 15). delta == NULL drops the
 * first term, image_delta == NULL the second; P_axis is the mirror parity map
 * of parity_axis (src/fmm.cpp:108-123). delta, image_delta: host n_blk x 3.
 * The far bank of assemble_periodic_fmm (src/fmm.cpp:180-191) is
 * delta = shift(o); a folded half space adds image_delta = center(o) -
 * mirror(base_center); the split-half-space K_hat bank (src/fmm.cpp:204-242)
 * is image_delta only. Replaces the host loop over far offsets. */
int fpbem_cu_m2l_bank(int n_t, double k, int n_blk, const double* delta, const double* image_delta,
                      int parity_axis, fpbem_c64 reflection, int device, fpbem_c64* out, int ptr_kind);

int fpbem_cu_fmm_create(const fpbem_cu_fmm_desc* desc, int device, fpbem_cu_op** out);
void fpbem_cu_fmm_destroy(fpbem_cu_op* op);

/* y = A x for nrhs right-hand sides. ptr_kind: FPBEM_CU_PTR_HOST (synchronous)
 * or FPBEM_CU_PTR_DEVICE (enqueued on the handle's stream). */
int fpbem_cu_fmm_apply(fpbem_cu_op* op, const fpbem_c64* x, fpbem_c64* y, int nrhs, int ptr_kind);

/* Restarted GMRES(restart) from x0 = 0, independently per right-hand side
 * (src/solver.cpp:21-123: MGS + one conditional reorthogonalisation pass,
 * complex Givens, estimate-based inner exit, true residual per cycle).
 * iterations/converged: nrhs entries. history: per rhs, up to history_cap
 * relative-residual estimates (row r at history + r*history_cap);
 * history_len: nrhs entries (may be NULL). Returns FPBEM_CU_ENONFINITE when
 * the operator produced NaN/Inf (src/solver.cpp:13-17). */
int fpbem_cu_gmres(fpbem_cu_op* op, const fpbem_c64* b, fpbem_c64* x, int nrhs, double tol,
                   int restart, int max_iter, int ptr_kind, int* iterations, int* converged,
                   double* history, int history_cap, int* history_len);

/* The reference's ApplyFn seam (include/fpbem/solver.hpp:21) on the device:
 * GMRES over any operator given as a callback that maps a device vector to
 * a device vector on `stream` (a cudaStream_t). Returns 0 on success.
 * precond (may be NULL) is the optional left preconditioner M^{-1}
 * (GmresOptions::preconditioner, include/fpbem/solver.hpp:27). */
typedef int (*fpbem_cu_apply_fn)(void* ctx, const fpbem_c64* x_dev, fpbem_c64* y_dev, void* stream);
int fpbem_cu_gmres_fn(int device, long long n, fpbem_cu_apply_fn apply, void* apply_ctx,
                      fpbem_cu_apply_fn precond, void* precond_ctx, const fpbem_c64* b, fpbem_c64* x,
                      double tol, int restart, int max_iter, int ptr_kind, int* iterations,
                      int* converged, double* history, int history_cap, int* history_len);

/* Device bytes of the operator data, counted like FmmOperators::stored_bytes
 * (S blocks + spectrum + U0 + V0). */
int fpbem_cu_fmm_bytes(const fpbem_cu_op* op, size_t* bytes);
/* The near-field path in use (FPBEM_CU_NEAR_DIRECT / _LATTICE), its lattice
 * sizes (1,1,1 for direct), the device bytes of its stored block spectrum, the
 * largest number of Fourier modes one stored block serves (1 without verified
 * symmetries), the verified symmetry mask (bit g) and the largest measured
 * deviation max|S_{A_g o}[P i, P j] - S_o[i, j]| / max|S| over the given
 * symmetries (-1 when none were given). */
int fpbem_cu_fmm_near_path(const fpbem_cu_op* op, int* path, int* sizes, size_t* spectrum_bytes, int* modes_per_block,
                           int* symmetry_mask, double* symmetry_dev);

/* Spectrum readback (sizes[3] always; lambda_out may be NULL). */
int fpbem_cu_spectrum(const fpbem_cu_op* op, int* sizes, fpbem_c64* lambda_out);

/* Far-field M2L layout for roofline accounting: *paired = 1 when the spectrum's
 * mirror parity Λ(-q) = D Λ(q) D was verified and each Λ block is streamed once
 * for a mode and its mirror, so an apply reads about half of
 * q b^2 blocks; *paired = 2 when the reflection parity Λ(qx, qy, -qz) = Dz Λ(q) Dz
 * holds as well and the flat stream reads about a quarter of them. */
int fpbem_cu_far_info(const fpbem_cu_op* op, int* sizes, int* paired);

/* Run subsequent device work on an external cudaStream_t (NULL = own stream). */
int fpbem_cu_set_stream(fpbem_cu_op* op, void* stream);

/* The cudaStream_t device work of this handle is ordered on (its own
 * non-blocking stream unless set_stream gave one). Callers that produce inputs
 * or consume outputs on another stream order the two with events around
 * fpbem_cu_fmm_apply(..., FPBEM_CU_PTR_DEVICE). */
int fpbem_cu_get_stream(const fpbem_cu_op* op, void** stream);

/* Per-stage CUDA-event timing of applies (0 = off, 1 = on, 2 = on with
 * P2M + M2L moved from the concurrent aux stream onto the main stream, so each
 * stage is timed alone; the product is unchanged). When on, each apply
 * accumulates milliseconds per stage; fpbem_cu_stage_times copies
 * {near field, near_reduce_l2p (or L2P), p2m, m2l, total, applies,
 * lattice-path mode product} into ms_out[7]
 * and resets the counters. */
int fpbem_cu_enable_stage_timing(fpbem_cu_op* op, int enable);
int fpbem_cu_stage_times(fpbem_cu_op* op, double* ms_out);

/* Slab-distributed product (lattice near field only):
 * rank r of `comm` (NULL = one rank) owns whole planes of cells along the slab
 * axis (the highest lattice axis with more than one cell), rows [lo, hi) of
 * the reference's cell-major vector layout. apply_slab takes x[lo:hi) and
 * returns (A x)[lo:hi); inside, the pruned lattice DFTs below the slab axis run
 * on the rank's planes, one grouped NCCL all-to-all per direction transposes to
 * the rank's columns, where the DFTs along the slab axis, the near-field block
 * products (the rank's share of the stored blocks) and the M2L (the rank's share
 * of Λ) run. fpbem_cu_gmres_dist uses the plan when it is set (slab vectors, no
 * all-gather). Every rank calls set_slabs / apply_slab collectively. */
int fpbem_cu_fmm_set_slabs(fpbem_cu_op* op, fpbem_cu_comm* comm);
int fpbem_cu_fmm_slab_rows(const fpbem_cu_op* op, long long* lo, long long* hi);
int fpbem_cu_fmm_apply_slab(fpbem_cu_op* op, const fpbem_c64* x, fpbem_c64* y, int ptr_kind);
/* The plan of this rank: info[0..7] = rank, ranks, slab axis, planes, stored
 * near-field blocks, near-field modes, far-field (Λ) modes, fused z kernel. */
int fpbem_cu_fmm_slab_info(const fpbem_cu_op* op, long long info[8]);

/* Number of CUDA kernels this handle launched since creation. */
long long fpbem_cu_kernel_launches(const fpbem_cu_op* op);

/* Multi-GPU (one process per GPU). Rank 0 makes the id, the caller
 * broadcasts its 128 bytes (e.g. torch.distributed), every rank inits.
 * With a communicator attached, apply() splits the near-field pairs
 * across ranks and all-reduces the partial products;
 * set_comm measures the far field's cost (fpbem_cu_fmm_far_pairs), averages
 * it over the ranks and gives rank 0 (which runs the far field) that many
 * fewer pairs. */
int fpbem_cu_comm_unique_id(unsigned char id_out[128]);
int fpbem_cu_comm_init(const unsigned char id[128], int nranks, int rank, int device,
                       fpbem_cu_comm** out);
void fpbem_cu_comm_destroy(fpbem_cu_comm* comm);
int fpbem_cu_fmm_set_comm(fpbem_cu_op* op, fpbem_cu_comm* comm);

/* A communicator over a caller-supplied host all-reduce (e.g. a gloo process
 * group, or MPI): allreduce_sum(ctx, buf, count) must replace the host buffer
 * of `count` doubles by its element-wise sum over all ranks and return 0. The
 * library stages device data through pinned host memory; reduce-scatter and
 * all-gather are built from the all-reduce (an all-gather sums zero-filled
 * slabs, which is exact). Same semantics as the NCCL communicator: for hosts
 * whose ranks have no NCCL path between them, and for multi-rank tests. */
typedef int (*fpbem_cu_allreduce_fn)(void* ctx, double* host_buf, size_t count);
int fpbem_cu_comm_from_callback(fpbem_cu_allreduce_fn allreduce_sum, void* ctx, int nranks, int rank,
                                int device, fpbem_cu_comm** out);

/* A simulated communicator: rank `rank` of `nranks`, alone on `device`. Every
 * collective moves only this rank's own block (device to device) and counts
 * the bytes the real collective would send from this rank (ring all-reduce:
 * 2 (P-1)/P of the buffer; reduce-scatter / all-gather: (P-1) slabs;
 * all-to-all: the blocks addressed to other ranks). Results are partial, so
 * it is for timing one rank's share of a multi-GPU product or solve on one
 * GPU (tools/model_scaling.py), never for answers. comm_traffic reads (and
 * with reset != 0 clears) the counters; it fails on a real communicator. */
int fpbem_cu_comm_simulated(int nranks, int rank, int device, fpbem_cu_comm** out);
int fpbem_cu_comm_traffic(fpbem_cu_comm* comm, unsigned long long* bytes_sent, long long* collectives, int reset);

/* Distributed restarted GMRES: the Krylov basis, x and
 * the residual are split over the ranks of the attached communicator in
 * contiguous slabs of whole cells (fpbem_cu_gmres_dist_rows); per Arnoldi
 * step the new basis vector is all-gathered for the product, the ranks'
 * partial products are reduce-scattered back to the slabs, and each
 * Gram-Schmidt pass is classical (one batched all-reduce of the j+1
 * projections and ||w||^2) with the reference's own reorthogonalisation test
 * (second pass iff ||w_post|| < ||w_pre|| / 2, src/solver.cpp:63-69); the
 * Hessenberg / Givens control flow is the reference's, replicated on every
 * rank from all-reduced scalars. Every rank passes the full b and receives
 * the full x (one right-hand side). Without a communicator it runs on one
 * device with the same arithmetic. Arguments and errors as fpbem_cu_gmres. */
int fpbem_cu_gmres_dist(fpbem_cu_op* op, const fpbem_c64* b, fpbem_c64* x, double tol, int restart,
                        int max_iter, int ptr_kind, int* iterations, int* converged, double* history,
                        int history_cap, int* history_len);

/* This rank's slab [lo, hi) of the global rows under fpbem_cu_gmres_dist. */
int fpbem_cu_gmres_dist_rows(const fpbem_cu_op* op, long long* lo, long long* hi);

/* The same partition without a communicator: apply() returns this rank's
 * partial product (its near-field pairs; rank 0 adds the far field). Summing
 * the nranks partial products gives the full product. far_pairs: rank 0's
 * deficit (0 = equal shares; every rank must pass the same value). */
int fpbem_cu_fmm_set_partition(fpbem_cu_op* op, int rank, int nranks, double far_pairs);

/* This handle's current pair range [lo, hi) and rank-0 deficit. */
int fpbem_cu_fmm_partition(const fpbem_cu_op* op, long long* lo, long long* hi, double* far_pairs);

/* The far field's cost (P2M + M2L) in near-field pair equivalents, measured on
 * the handle's device: t_far / t_near(all pairs) x n_pairs. */
int fpbem_cu_fmm_far_pairs(fpbem_cu_op* op, double* far_pairs);

/* The partition rule itself (host only, no GPU): the near-field (offset,
 * target) pairs, in offset-major order, split into nranks contiguous ranges
 * [lo, hi) — every pair costs the same n_dof^2 complex MACs — equal, except
 * that rank 0 takes round(far_pairs) fewer and ranks 1.. share the rest. */
int fpbem_cu_partition_pairs(long long n_pairs, int nranks, int rank, double far_pairs, long long* lo,
                             long long* hi);

const char* fpbem_cu_last_error(void);
const char* fpbem_cu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FPBEM_CUDA_H */
