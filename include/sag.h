/*
 * sag.h -- C-ABI of the B200-native (sm_100a) solve-phase hot path of the
 * monolithic SA-AMG / additive-Vanka Stokes solver (arXiv 2306.06795,
 * reference implementation "stokesamg").
 *
 * Every entry point replaces one reference interface; the citation is given
 * as <reference file>:<line> relative to the reference's proj/core tree.
 * Setup objects (hierarchy, patterns) still come from the reference's own
 * host C++ (build_case / build_monolithic_hierarchy); this library takes the
 * resulting CSR arrays and runs everything from factor_patches down on the GPU.
 *
 * Conventions
 *  - Plain pointers and sizes only. Every `const double*` / `double*` vector
 *    argument may be a HOST pointer (pageable or pinned; copied in/out inside
 *    the call) or a DEVICE pointer of this context's GPU (used in place).
 *  - Every function returns a status (SAG_OK = 0). The codes map 1:1 onto the
 *    reference's exception classes (errors.hpp:8-58); sag_last_error() gives
 *    the message of the calling thread's last failure.
 *  - Calls on one context are serialised on its CUDA stream; results are
 *    complete when a call with host output returns, or after sag_synchronize.
 *  - There is no CPU fallback: without a usable sm_100 device sag_create fails.
 */
#ifndef SAG_H
#define SAG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:8-58) ------------------------------------ */
enum sag_status {
  SAG_OK = 0,
  SAG_ERROR = 1,               /* stokesamg::Error                         */
  SAG_DIMENSION_MISMATCH = 2,  /* stokesamg::DimensionMismatch              */
  SAG_SINGULAR_MATRIX = 3,     /* stokesamg::SingularMatrix                 */
  SAG_SINGULAR_PATCH = 4,      /* stokesamg::SingularPatch                  */
  SAG_CONFIG_ERROR = 5,        /* stokesamg::ConfigError                    */
  SAG_SOLVER_STAGNATION = 6,   /* stokesamg::SolverStagnation               */
  SAG_ZERO_DIAGONAL = 7,       /* stokesamg::ZeroDiagonal (sparse.cpp:211)  */
  SAG_UNSUPPORTED_DISCRETIZATION = 8, /* stokesamg::UnsupportedDiscretization */
  SAG_CUDA_ERROR = 100,        /* device / driver failure (no reference analogue) */
  SAG_INVALID_ARGUMENT = 101   /* null handle / pointer                     */
};

typedef struct sag_ctx sag_ctx;         /* device, stream, workspaces            */
typedef struct sag_matrix sag_matrix;   /* CSR on device (sparse.hpp:11-28)     */
typedef struct sag_patches sag_patches; /* Vanka patch sets (vanka.hpp:11-15)   */
typedef struct sag_vanka sag_vanka;     /* factorization (vanka.hpp:23-40)      */
typedef struct sag_dc sag_dc;           /* DCPreconditioner (preconditioner.hpp:77-100) */

/* Thread-local message of the last failing call on this thread. */
const char* sag_last_error(void);

/* ---- context ------------------------------------------------------------ */
/* Creates a context on CUDA device `device` (fails with SAG_CUDA_ERROR if it
 * is not an sm_100 part). No reference analogue (the reference is host-only). */
int sag_create(int device, sag_ctx** out);
/* The same on a caller-owned CUDA stream (cudaStream_t passed as void*), e.g.
 * a framework's stream: libsag launches on it and never destroys it. */
int sag_create_on_stream(int device, void* stream, sag_ctx** out);
int sag_destroy(sag_ctx* ctx);
int sag_synchronize(sag_ctx* ctx);
/* Device buffers for callers that keep vectors resident (bench, pipelines). */
int sag_alloc(sag_ctx* ctx, size_t bytes, void** dptr);
int sag_free(sag_ctx* ctx, void* dptr);
/* cudaMemcpyDefault semantics, ordered on the context stream, synchronous. */
int sag_memcpy(sag_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Number of kernels this library launched on ctx since creation. */
int sag_launch_count(sag_ctx* ctx, long long* out);
/* CUDA stream of the context (cudaStream_t), for event timing by callers. */
int sag_stream(sag_ctx* ctx, void** stream);

/* ---- sparse (sparse.hpp:11-28, :42, :64-65) ------------------------------ */
/* Uploads a canonical CSR matrix (sorted, duplicate-free rows; int32 indices,
 * fp64 values). Replaces stokesamg::SparseMatrix (sparse.hpp:11-28). */
int sag_matrix_create(sag_ctx* ctx, int nrows, int ncols, long long nnz, const int* row_offsets,
                      const int* col_indices, const double* values, sag_matrix** out);
int sag_matrix_destroy(sag_matrix* m);
int sag_matrix_shape(const sag_matrix* m, int* nrows, int* ncols, long long* nnz);
/* y = m x. Replaces spmv (sparse.hpp:42; sparse.cpp:78-91). */
int sag_spmv(sag_ctx* ctx, const sag_matrix* m, const double* x, double* y);
/* SpMV with one of the fused epilogues the solver uses (device pointers, for
 * per-kernel timing): 0 y = Ax; 1 y = aux - Ax; 2 y += Ax; 3 y = Ax and
 * (y, aux); 4 y = aux - Ax and ||y||. Reductions land in device scratch. */
int sag_spmv_fused(sag_ctx* ctx, const sag_matrix* m, const double* x, double* y,
                   const double* aux, int epilogue);
/* Replaces norm2 / dot (sparse.hpp:64-65; sparse.cpp:217-227). Deterministic
 * fixed-order two-stage reductions. */
int sag_norm2(sag_ctx* ctx, int n, const double* v, double* out);
int sag_dot(sag_ctx* ctx, int n, const double* a, const double* b, double* out);

/* ---- Vanka (vanka.hpp:11-55) --------------------------------------------- */
/* Replaces build_patches (vanka.hpp:20-21; vanka.cpp:11-42): one patch per
 * pressure row, or per consecutive row triple when sv_triples != 0. */
int sag_build_patches(sag_ctx* ctx, const sag_matrix* k, int n_x, int n_y, int n_p,
                      int sv_triples, sag_patches** out);
/* Explicit patch lists (the reference tests build hand-made VankaPatch sets,
 * tests/test_vanka.cpp:98-113). Arrays are host or device, CSR-like. */
int sag_patches_create(sag_ctx* ctx, int npatch, const int* pressure_ptr,
                       const int* pressure_idx, const int* velocity_ptr,
                       const int* velocity_idx, const int* nx, sag_patches** out);
int sag_patches_destroy(sag_patches* p);
/* info = [npatch, total pressure entries, total velocity entries, max nv, max np] */
int sag_patches_info(const sag_patches* p, long long* info);
/* Copies the patch lists out (host or device arrays sized from info). */
int sag_patches_export(sag_ctx* ctx, const sag_patches* p, int* pressure_ptr,
                       int* pressure_idx, int* velocity_ptr, int* velocity_idx, int* nx);

/* Replaces factor_patches (vanka.hpp:42-43; vanka.cpp:64-149): batched
 * block-LU on the device. Fails with SAG_SINGULAR_PATCH like the reference. */
int sag_factor_patches(sag_ctx* ctx, const sag_matrix* k, const sag_patches* p, int n_u,
                       sag_vanka** out);
int sag_vanka_destroy(sag_vanka* f);
/* stats = [a_factor_bytes, aux_bytes, dense_inverse_bytes (vanka.hpp:36-39),
 *          device bytes of the apply representation, npatch, n, n_slots]      */
int sag_vanka_stats(const sag_vanka* f, long long* stats);
/* Apply launch classes (no reference counterpart: the device layout). Class i
 * fills out[4i..4i+3] = [rows per lane R, lanes per patch (32: warp per
 * patch, vanka_patch_kernel<R>; 16 / 8: vanka_subwarp_kernel<LPP>), patches,
 * blob bytes], for i < cap; *nclasses = the number of classes. */
int sag_vanka_classes(const sag_vanka* f, long long* out, int cap, int* nclasses);
/* Factor payload in the reference's layout (vanka.hpp:31-33), concatenated in
 * patch order: u_hat (nv x np), b_hat (np x nv), s_inv (np x np), row-major;
 * weights (length n). Any pointer may be NULL. For parity tests. */
int sag_vanka_export(sag_ctx* ctx, const sag_vanka* f, double* u_hat, double* b_hat,
                     double* s_inv, double* weights);
/* Overrides the PoU weights (vanka.cpp:67-73) with the caller's (length n):
 * a rank that factorizes only its share of the patches of a partitioned
 * operator needs the global multiplicities. */
int sag_vanka_set_weights(sag_ctx* ctx, sag_vanka* f, const double* weights);
/* delta = sum_i V_i^T W K_i^-1 V_i r. Replaces apply_vanka (vanka.hpp:47;
 * vanka.cpp:151-184). */
int sag_apply_vanka(sag_ctx* ctx, const sag_vanka* f, const double* r, double* delta);

/* x += omega * apply_vanka(r) (the update of vanka_relax's stationary mode,
 * vanka.cpp:195), fused into the gather: a partitioned sweep adds its boundary
 * patches' contributions onto the interior ones. */
int sag_apply_vanka_add(sag_ctx* ctx, const sag_vanka* f, const double* r, double* x,
                        double omega);

/* sag_apply_vanka_add fused with the reverse halo of a partitioned sweep:
 * where slot[d] >= 0 (a ghost dof of this rank), the updated x_d -- this
 * rank's complete partial sum there -- is also stored into
 * peers[nbr[d]][slot[d]], a neighbour's receive buffer mapped by
 * sag_ipc_open_handle (NVLink stores, system-scope fence). Device pointers;
 * at most 8 neighbours; dof-ordered result layout (default). */
int sag_apply_vanka_add_push(sag_ctx* ctx, const sag_vanka* f, const double* r, double* x,
                             double omega, const int* slot, const unsigned char* nbr, int npeer,
                             double* const* peers);

/* The hot step as one call: y = K x (spmv, sparse.cpp:78-91) and delta =
 * apply_vanka(x) (vanka.cpp:151-184) on the same input. With host buffers x
 * crosses the host link once and y's copy back overlaps the Vanka sweep (a
 * second stream); results are complete on return. Same results as
 * sag_spmv + sag_apply_vanka. */
int sag_vanka_spmv(sag_ctx* ctx, const sag_vanka* f, const sag_matrix* k, const double* x,
                   double* delta, double* y);
/* Diagnostic (no reference counterpart): the plan of the last pipelined
 * host-buffer step of f (sag_vanka_spmv with pinned host x, delta, y: x
 * arrives in stages and every output range leaves as soon as its inputs
 * arrived). out = [stages (0: no plan), ranges, host->device ranges, SpMV row
 * ranges, gather ranges, patch windows, choice (1 pipelined, -1 plain, 0 not
 * yet timed), ns per plain step, ns per pipelined step]. By default the first
 * call on a plan times both forms of the step and keeps the faster one;
 * SAG_STEP_STAGES=S forces the pipeline with S stages (1: never). */
int sag_vanka_step_plan(const sag_vanka* f, long long* out, int cap);

/* One stage of sag_apply_vanka, for per-kernel timing (device pointers):
 * stage 1 = patch kernel (local solves into the slot buffer),
 * stage 2 = owner-computes gather (slots -> delta). */
int sag_apply_vanka_stage(sag_ctx* ctx, const sag_vanka* f, const double* r, double* delta,
                          int stage);

/* Replaces vanka_relax (vanka.hpp:49-55; vanka.cpp:186-209). */
enum sag_relax_mode { SAG_RELAX_KRYLOV_WRAPPED = 0, SAG_RELAX_STATIONARY = 1 };
int sag_vanka_relax(sag_ctx* ctx, const sag_matrix* k, const sag_vanka* f, double* x,
                    const double* b, int mode, int sweeps, double omega);

/* ---- Krylov (krylov.hpp:17-35) ------------------------------------------- */
typedef struct {
  double tol;       /* relative to ||b|| (krylov.hpp:18) */
  int max_iters;
  int restart;
  double breakdown; /* happy-breakdown threshold (krylov.hpp:21) */
} sag_fgmres_options;

typedef struct {
  int converged;
  int iterations;
  double final_relative_residual;
  int history_len; /* = iterations + 1 (krylov.hpp:26) */
} sag_krylov_report;

/* Preconditioner selector for sag_fgmres (the reference passes a
 * LinearOperator, krylov.hpp:12). */
enum sag_prec_kind {
  SAG_PREC_IDENTITY = 0, /* identity_operator (krylov.cpp:13-15) */
  SAG_PREC_VANKA = 1,    /* prec = const sag_vanka*: apply_vanka  */
  SAG_PREC_JACOBI = 2,   /* prec = const sag_matrix*: z = D^-1 r (amg.cpp:266-269) */
  SAG_PREC_DC = 3,       /* prec = const sag_dc*: DCPreconditioner::apply */
  SAG_PREC_UZAWA = 4     /* prec = const sag_uzawa*: UzawaPreconditioner::apply */
};
/* Replaces fgmres(matrix_operator(a), b, x, prec, opt) (krylov.hpp:33-35;
 * krylov.cpp:17-121). x holds the guess on entry. history may be NULL. */
int sag_fgmres(sag_ctx* ctx, const sag_matrix* a, const double* b, double* x, int prec_kind,
               const void* prec, const sag_fgmres_options* opt, sag_krylov_report* rep,
               double* history, int history_cap);

/* ---- preconditioner (preconditioner.hpp:19-148) --------------------------- */
/* Variant (preconditioner.hpp:14): DC-all / DC-LO / DC-HO and HO-AMG are
 * sag_dc objects; Uzawa is its own object (sag_uzawa_create). */
enum sag_variant { SAG_DC_ALL = 0, SAG_DC_LO = 1, SAG_DC_HO = 2, SAG_HOAMG = 3, SAG_UZAWA = 4 };

typedef struct { /* SolverConfig, preconditioner.hpp:19-36 */
  int variant;
  double eta_u, eta_p, omega0;
  int nu1, nu2, gamma, restart;
  double tol;
  int max_iters;
  int enclosed_flow;
  int allow_sv_hoamg; /* HO-AMG on SV is refused unless set (preconditioner.hpp:31) */
} sag_solver_config;

/* Fills the reference defaults (preconditioner.hpp:20-33). */
int sag_solver_config_default(sag_solver_config* cfg);
/* Replaces SolverConfig::check (preconditioner.cpp:30-38). */
int sag_solver_config_check(const sag_solver_config* cfg);

/* One level of the low-order monolithic hierarchy (amg.hpp:85-90): K and the
 * prolongator to the next level (NULL on the coarsest). */
typedef struct {
  const sag_matrix* k;
  const sag_matrix* p;
  int n_x, n_y, n_p;
} sag_level_desc;

/* With cfg->variant == SAG_HOAMG this is the HoAmgPreconditioner constructor
 * (preconditioner.cpp:155-172): `levels` is the monolithic hierarchy built on
 * the high-order system itself (level 0 == k0), apply = one V-cycle
 * (preconditioner.cpp:174-176). Otherwise it replaces
 * the DCPreconditioner constructor (preconditioner.cpp:90-105) and
 * MonolithicSolver's (preconditioner.cpp:40-55): Vanka factors for K0 and every
 * non-coarsest level, R = P^T, coarse dense LU (with the enclosed-flow pin
 * 1e-12 * norm_inf(K of level 0), preconditioner.cpp:49-53), all on device.
 * TH injection transfer (transfer.cpp:97-125) when sv == 0. For sv != 0 the
 * fine patches are element triples with stationary relaxation, and the
 * transfer needs sag_dc_set_sv_transfer before the first apply. */
int sag_dc_create(sag_ctx* ctx, const sag_matrix* k0, int n_x0, int n_y0, int n_p0, int sv,
                  int nlevels, const sag_level_desc* levels, const sag_solver_config* cfg,
                  sag_dc** out);
int sag_dc_destroy(sag_dc* d);
/* set_parameters (preconditioner.hpp:87) */
int sag_dc_set_parameters(sag_dc* d, double eta_u, double eta_p, double omega0);
/* SV transfer (transfer.cpp:18-53, :82-95): duplication map P^p (n_p0 x n_p1),
 * M_mix (n_p1 x n_p0), Mcg (n_p1 x n_p1) and its scalar SA hierarchy
 * (amg.hpp:68-76): nsl matrices, nsl-1 prolongators. Mass projection solved by
 * device FGMRES(20) to 1e-12 with one scalar V(2,2) cycle as preconditioner. */
int sag_dc_set_sv_transfer(sag_dc* d, const sag_matrix* p_dup, const sag_matrix* m_mix,
                           int nsl, const sag_matrix* const* scalar_levels,
                           const sag_matrix* const* scalar_prolongators);
/* Diagnostic (no reference counterpart): with SAG_PROJ_TRACE=1 at setup the
 * one-launch mass projection records (phase tag, globaltimer ns) pairs of its
 * last run: out[0, 2*8192) for worker CTA 0, out[2*8192, 4*8192) for CTA 0 of
 * the tail cluster; cap = number of 64-bit words of out. */
int sag_dc_proj_trace(sag_ctx* ctx, sag_dc* d, unsigned long long* out, long long cap);
/* Replaces DCPreconditioner::apply (preconditioner.cpp:114-153). */
int sag_dc_apply(sag_ctx* ctx, sag_dc* d, const double* r, double* z);
/* Replaces MonolithicSolver::vcycle (preconditioner.cpp:83-88) on the
 * low-order hierarchy, skip_finest_relax = 0. */
int sag_dc_vcycle(sag_ctx* ctx, sag_dc* d, const double* b, double* x, int nu1, int nu2);
/* counters = [fine_relax_units, level1_relax_units] (preconditioner.hpp:46-48) */
int sag_dc_counters(const sag_dc* d, long long* counters);
/* levels info: out = [nlevels, n0, n_levels rows.., bytes of device factors,
 * launches of the captured apply, then for the SV mass projection: 1 when it
 * runs as one persistent launch, its grid levels, CTAs and worker CTAs] */
int sag_dc_info(const sag_dc* d, long long* out, int cap);

/* Replaces solve_stokes (preconditioner.hpp:147-148; preconditioner.cpp:229-259):
 * outer FGMRES on K0 with the DC preconditioner and the enclosed-flow pressure
 * projection. Solver settings are read from cfg (restart, tol, max_iters,
 * enclosed_flow). x is overwritten (zero initial guess). */
int sag_solve_stokes(sag_ctx* ctx, sag_dc* d, const double* rhs, double* x,
                     const sag_solver_config* cfg, sag_krylov_report* rep, double* history,
                     int history_cap);

/* ---- inexact Uzawa (preconditioner.hpp:118-141) ----------------------------- */
typedef struct sag_uzawa sag_uzawa;
/* A ScalarHierarchy (amg.hpp:64-72) built on the host: nlevels matrices and
 * nlevels - 1 prolongators; R = P^T, Jacobi diagonals and the coarse LU are
 * formed on the device. */
typedef struct {
  int nlevels;
  const sag_matrix* const* a;
  const sag_matrix* const* p;
} sag_scalar_hierarchy;
/* Replaces the UzawaPreconditioner constructor (preconditioner.cpp:178-192):
 * b = B (n_p x n_u), scalar hierarchies of A_x and A_y, and either the Mp
 * hierarchy (TH/ISO; sv_element_areas == NULL) or the SV element areas
 * (n_p / 3 values; hp may be NULL) for the exact element mass inverse. */
int sag_uzawa_create(sag_ctx* ctx, const sag_matrix* b, int n_x, int n_y, int n_p,
                     const sag_scalar_hierarchy* hx, const sag_scalar_hierarchy* hy,
                     const sag_scalar_hierarchy* hp, const double* sv_element_areas,
                     const sag_solver_config* cfg, sag_uzawa** out);
int sag_uzawa_destroy(sag_uzawa* u);
/* Replaces UzawaPreconditioner::apply (preconditioner.cpp:194-218). */
int sag_uzawa_apply(sag_ctx* ctx, sag_uzawa* u, const double* r, double* z);
/* solve_stokes (preconditioner.cpp:229-259) with the Uzawa preconditioner. */
int sag_solve_stokes_uzawa(sag_ctx* ctx, const sag_matrix* k0, sag_uzawa* u, const double* rhs,
                           double* x, const sag_solver_config* cfg, sag_krylov_report* rep,
                           double* history, int history_cap);

/* ---- hierarchy setup products -----------------------------
 * The sparse products of the SA setup on the device, BITWISE the reference's
 * (every entry summed in the reference's order with round-to-nearest ops, the
 * entries that cancel to exactly 0.0 dropped -- the hierarchy's patterns
 * depend on it). New matrices are returned as new handles. */
/* C = A B. Replaces spgemm (sparse.hpp:46; sparse.cpp:113-150). */
int sag_spgemm(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* b, sag_matrix** out);
/* A^T. Replaces transpose (sparse.hpp:44; sparse.cpp:93-111). */
int sag_transpose(sag_ctx* ctx, const sag_matrix* a, sag_matrix** out);
/* P^T K P. Replaces galerkin_triple (sparse.hpp:49; sparse.cpp:152-156). */
int sag_galerkin(sag_ctx* ctx, const sag_matrix* p, const sag_matrix* k, sag_matrix** out);
/* T - omega D^-1 (A T), D = diag(A). Replaces smooth_prolongator
 * (amg.hpp:51; amg.cpp:226-236) given omega = omega_frac / rho, rho from the
 * reference's power_rho_estimate (sparse.cpp:239-261; its mt19937 start
 * vector stays on the host). Fails with SAG_ZERO_DIAGONAL like inv_diagonal. */
int sag_smooth_prolongator(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* t, double omega,
                           sag_matrix** out);
/* Replaces evolution_soc (amg.hpp:24; amg.cpp:45-110) given omega =
 * 4 / (3 rho) from the reference's power_rho_estimate: the symmetrised
 * strength graph (graph_from_adjacency, amg.cpp:13-42) as an n x n CSR whose
 * values are the edge strengths (StrengthGraph offsets / neighbors /
 * weights). Each column's z = (I - omega D^-1 A)^k e_j is accumulated in the
 * reference's order, so the graph is bitwise the reference's. SAG_ERROR if a
 * column's k-step support exceeds 2048 nodes (the caller keeps the host path). */
int sag_evolution_soc(sag_ctx* ctx, const sag_matrix* a, double omega, double theta, int k,
                      sag_matrix** graph);
/* K = [[A, B^T], [B, 0]] from the velocity block A (n_u x n_u) and the
 * divergence B (n_p x n_u). Replaces assemble_saddle_matrix (fem.hpp;
 * fem.cpp:290-306): the blocks never overlap, so K is bitwise the reference's. */
int sag_saddle_matrix(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* b, sag_matrix** out);
/* tentative_prolongator_with_nullvec (amg.cpp:184-205) on the device: T
 * (n x num_aggregates, T_ic = nullvec_i / ||nullvec over aggregate c||, the
 * norms summed in node order), coarse_nullvec = the aggregate norms (host or
 * device, may be NULL). SAG_ERROR for an aggregate with a zero norm. */
int sag_tentative_prolongator(sag_ctx* ctx, int n, int num_aggregates, const int* node_to_agg,
                              const double* nullvec, sag_matrix** t, double* coarse_nullvec);
/* power_rho_estimate (sparse.cpp:239-261) from the caller's normalised start
 * vector x0 (the reference's mt19937 stream / its norm): iters x (y = D^-1 M x
 * on the device, rows summed in order; ||y|| summed sequentially on the host;
 * x = y / ||y||); *rho = the last ||y|| (0 when it vanishes). Bitwise the
 * reference's estimate. */
int sag_power_rho(sag_ctx* ctx, const sag_matrix* m, const double* d_inv, const double* x0,
                  int iters, double* rho);
/* Copies a matrix's CSR arrays out (host or device arrays; any may be NULL). */
int sag_matrix_export(sag_ctx* ctx, const sag_matrix* m, int* row_offsets, int* col_indices,
                      double* values);

/* ---- 3 velocity components (BASELINE config 5) -----------
 * The reference is 2D only. factor_patches / apply_vanka
 * (vanka.cpp:11-184) generalised to K rows [x | y | z | p]: one pressure seed
 * per patch, one LU per velocity component, CTA-per-patch kernels for the
 * 100-250-dof patches of 3D Taylor-Hood. Parity is against oracle.c's
 * 3-component restatement (or_*3). */
typedef struct sag_vanka3 sag_vanka3;
int sag_factor_patches3(sag_ctx* ctx, const sag_matrix* k, int n_x, int n_y, int n_z, int n_p,
                        sag_vanka3** out);
int sag_vanka3_destroy(sag_vanka3* f);
/* stats = [npatch, n, blob bytes, max patch velocity dofs, slots,
 *          a_factor_bytes, aux_bytes] */
int sag_vanka3_stats(const sag_vanka3* f, long long* stats);
int sag_apply_vanka3(sag_ctx* ctx, const sag_vanka3* f, const double* r, double* delta);

/* ---- FEM assembly on the device, bitwise the reference ---
 * A 2D triangle mesh (mesh.hpp:24-43) as plain arrays: vertices (x, y) pairs,
 * triangles (3 vertex ids each, positively oriented), tri_edges[t][k] = edge
 * opposite local vertex k (may be NULL where no P2 space is built),
 * num_edges = size of the lexicographic edge table. Arrays may be host or
 * device memory. */
typedef struct sag_mesh2d {
  int num_vertices, num_triangles, num_edges;
  const double* vertices;
  const int* triangles;
  const int* tri_edges;
} sag_mesh2d;
/* from_triplets (sparse.hpp:37; sparse.cpp:43-66): duplicates summed in the
 * order libstdc++'s std::sort leaves them (reproduced on the device), exact
 * zeros dropped. rows / cols / values: n entries in generation order. */
int sag_from_triplets(sag_ctx* ctx, int nrows, int ncols, long long n, const int* rows,
                      const int* cols, const double* values, sag_matrix** out);
/* perm[i] = the original index of the element std::sort (comparator on the
 * key only) places at position i of the n keys (test hook of the above);
 * *heap_ranges (may be NULL) = ranges that reached introsort's depth limit. */
int sag_sort_permutation(sag_ctx* ctx, long long n, const unsigned long long* keys, int* perm,
                         int* heap_ranges);
/* The P2 element loop of assemble_taylor_hood (sv = 0; fem.cpp:354-389) or
 * assemble_scott_vogelius (sv = 1; fem.cpp:452-498): the full scalar
 * Laplacian a_full (n_s x n_s, n_s = V + E) and divergence b_full (n_p x 2 n_s),
 * the load fx, fy (length n_s; may be NULL) from force_qp = the body force at
 * the 6 quadrature points of each triangle (f_x, f_y pairs, triangle-major;
 * NULL = zero force), and for SV the element mass Mp, the mixed mass M_mix and
 * the element areas (each may be NULL). */
int sag_assemble_p2(sag_ctx* ctx, const sag_mesh2d* mesh, int sv, const double* force_qp,
                    sag_matrix** a_full, sag_matrix** b_full, double* fx, double* fy,
                    sag_matrix** mp, sag_matrix** m_mix, double* areas);
/* assemble_p1_stiffness / assemble_p1_mass (fem.cpp:310-335); either may be NULL. */
int sag_assemble_p1(sag_ctx* ctx, const sag_mesh2d* mesh, sag_matrix** stiffness,
                    sag_matrix** mass);
/* The fine-mesh element loop of assemble_iso (fem.cpp:568-608): a_full
 * (nvf x nvf), b_fine (nvf x 2 nvf) and the load (may be NULL). */
int sag_assemble_iso(sag_ctx* ctx, const sag_mesh2d* fine, const double* force_qp,
                     sag_matrix** a_full, sag_matrix** b_fine, double* fx, double* fy);
/* Dirichlet elimination: reduce_scalar (fem.cpp:207-229) of a_full and
 * reduce_divergence (:233-252) of b_full (columns [x | y], scalar width n_s).
 * old_to_new[n_s] (-1 = constrained), gx / gy[n_s] the Dirichlet values (read
 * at constrained dofs). Outputs a_red, b_red, lift_x / lift_y (kept rows) and
 * rhs_p (b_full rows); the vectors may be NULL. */
int sag_reduce_dirichlet(sag_ctx* ctx, const sag_matrix* a_full, const sag_matrix* b_full,
                         int n_s, const int* old_to_new, const double* gx, const double* gy,
                         sag_matrix** a_red, sag_matrix** b_red, double* lift_x, double* lift_y,
                         double* rhs_p);

/* ---- partitioned solve: multi-GPU behind the C-ABI ----------
 * One process per GPU. A communicator carries the collectives: NCCL (rank 0
 * gets an id from sag_nccl_unique_id and the caller broadcasts it), or the
 * caller's own host-staged transport (sag_comm_ops: gloo, MPI, sockets; every
 * call blocking and made by all ranks in the same order). sag_dist_create
 * plans this rank's share of the row/patch partition from the GLOBAL host
 * CSR arrays every rank passes (K0, the low-order hierarchy and its
 * prolongators as built by build_monolithic_hierarchy, amg.hpp:99), factors
 * its patches and builds the agglomerated coarse levels; vectors are
 * rank-local (sag_dist_local_dofs: local -> global ids, owned flags). The
 * reference has no distributed path; the semantics are solve_stokes'
 * (preconditioner.cpp:229-259) over DCPreconditioner::apply
 * (preconditioner.cpp:114-153) with Taylor-Hood transfers. */
typedef struct sag_csr {
  int nrows, ncols;
  const int* row_offsets;   /* nrows + 1 */
  const int* col_indices;   /* row_offsets[nrows] */
  const double* values;
} sag_csr;
typedef struct sag_comm sag_comm;
typedef struct sag_dist sag_dist;
typedef struct sag_plan sag_plan;
typedef struct sag_comm_ops {
  void* user;
  /* buf (host, n doubles) <- the element-wise sum over all ranks; 0 on success */
  int (*allreduce_sum)(void* user, double* buf, long long n);
  /* send sbuf[i] (scount[i] doubles) to rank to[i] and receive rbuf[j]
   * (rcount[j] doubles) from rank from[j], all at once; 0 on success */
  int (*exchange)(void* user, int nsend, const int* to, const double* const* sbuf,
                  const long long* scount, int nrecv, const int* from, double* const* rbuf,
                  const long long* rcount);
} sag_comm_ops;
int sag_nccl_unique_id(unsigned char* id /* 128 bytes */);
int sag_comm_create_nccl(sag_ctx* ctx, int nranks, int rank, const unsigned char* id,
                         sag_comm** out);
int sag_comm_create_host(int nranks, int rank, const sag_comm_ops* ops, sag_comm** out);
int sag_comm_destroy(sag_comm* comm);
/* buf (device, n doubles) <- the sum over the ranks (blocking) */
int sag_comm_allreduce(sag_ctx* ctx, sag_comm* comm, double* buf, long long n);
/* levels[0..nlevels) / prolongators[0..nlevels-1) / level_nxyz[3 l + {0,1,2}]:
 * the low-order hierarchy (level 0 on the K0 dofs). DC-all / DC-LO / DC-HO,
 * nu1, nu2 <= 1. */
int sag_dist_create(sag_ctx* ctx, sag_comm* comm, const sag_csr* k0, int n_x, int n_y, int n_p,
                    int nlevels, const sag_csr* levels, const sag_csr* prolongators,
                    const int* level_nxyz, const sag_solver_config* cfg, sag_dist** out);
int sag_dist_destroy(sag_dist* d);
/* out = [local dofs, owned, ghosts, neighbours, own K0 patches, level-1 rows,
 * local velocity dofs] */
int sag_dist_info(const sag_dist* d, long long* out);
int sag_dist_local_dofs(const sag_dist* d, long long* l2g, unsigned char* owned);
/* The partitioned hot step on local vectors: delta = apply_vanka(x)
 * (vanka.cpp:151-184), y = K0 x (sparse.cpp:78-91) at the owned dofs. */
int sag_dist_step(sag_ctx* ctx, sag_dist* d, const double* x, double* delta, double* y);
/* solve_stokes over the partition: rhs, x local (owned entries valid); the
 * report and history are the global ones (identical on every rank). */
int sag_dist_solve_stokes(sag_ctx* ctx, sag_dist* d, const double* rhs, double* x,
                          sag_krylov_report* report, double* history, int history_cap);
/* The partition plan alone (host only, no device): for tests and tools.
 * sag_plan_array copies one array out (out may be NULL to query *count). */
enum sag_plan_item {
  SAG_PLAN_INFO = 0,       /* [local dofs, local velocity dofs, patch lo, hi, level-1 rows,
                              forward-send peers, forward-receive peers] (int64) */
  SAG_PLAN_L2G = 1,        /* int64 */
  SAG_PLAN_OWNED = 2,      /* uint8 */
  SAG_PLAN_FWD_SEND = 3,   /* int32 local ids for `peer` */
  SAG_PLAN_FWD_RECV = 4,
  SAG_PLAN_REV_SEND = 5,
  SAG_PLAN_REV_RECV = 6,
  SAG_PLAN_EXT_RP = 7,     /* + 100 for the low-order level 0 instead of K0 */
  SAG_PLAN_EXT_CI = 8,
  SAG_PLAN_EXT_V = 9,
  SAG_PLAN_INT_PVIDX = 10, /* interior patches' velocity lists */
  SAG_PLAN_BND_PVIDX = 11,
  SAG_PLAN_WEIGHTS = 12,
  SAG_PLAN_P_RP = 13,
  SAG_PLAN_P_CI = 14
};
int sag_plan_create(int nranks, int rank, const sag_csr* k0, const sag_csr* l0, const sag_csr* p0,
                    int n_x, int n_y, int n_p, sag_plan** out);
int sag_plan_destroy(sag_plan* plan);
int sag_plan_array(const sag_plan* plan, int which, int peer, void* out, long long* count);

/* ---- partitioned-solve primitives ---------------------------
 * Building blocks for a caller that row-partitions the solve across ranks
 * (one process per GPU, paper_2306_06795_b200/dsolve.py). All pointers are
 * DEVICE pointers and no call synchronises with the host: scalars stay in
 * device memory, so a partial reduction, the caller's all-reduce (NCCL on
 * the same stream) and the axpy that consumes it are stream-ordered.
 * They restate the vector operations of fgmres (krylov.cpp:42-110), norm2 /
 * dot (sparse.cpp:217-227) and project_pressure (preconditioner.cpp:235-240)
 * on a rank's share of the rows. */
/* out[0] = sum_{i: mask[i] != 0} a_i b_i (mask NULL: all i) -- a rank's
 * partial of dot / norm2 over the rows it owns (sparse.cpp:217-227). */
int sag_dot_async(sag_ctx* ctx, int n, const double* a, const double* b,
                  const unsigned char* mask, double* out);
/* y = y + sign * s[0] x  (MGS update w -= h_ij v_i, krylov.cpp:66). */
int sag_axpy_async(sag_ctx* ctx, int n, const double* s, double sign, const double* x, double* y);
/* y = x / d with d = s[0] or sqrt(s[0])  (v = r / ||r||, krylov.cpp:47-48, :71);
 * y = 0 when d == 0 (a zero residual, whose Krylov step the reference skips). */
int sag_div_async(sag_ctx* ctx, int n, const double* x, const double* s, int take_sqrt, double* y);
/* The coefficient y_0 of a one-step FGMRES from a zero guess (vanka_relax with
 * nu = 1, vanka.cpp:199-208 -> krylov.cpp:42-110): from ||r||^2, h_00 and
 * ||w||^2 after the MGS step, the Givens rotation and back substitution;
 * y_0[0] = 0 when r = 0. Device scalars: a relaxation needs no host sync. */
int sag_fgmres1_coef_async(sag_ctx* ctx, const double* ssq_r, const double* h00,
                           const double* ssq_w, double* y0);
/* y = x - sum[0] / count  (pressure-mean projection, preconditioner.cpp:235-240). */
int sag_sub_mean_async(sag_ctx* ctx, int n, const double* x, const double* sum, double count,
                       double* y);
/* y = a x + b y (a == b == 0: y = 0; b == 0: y = a x; b == 1: y += a x,
 * krylov.cpp:108-110). */
int sag_axpby_async(sag_ctx* ctx, int n, double a, const double* x, double b, double* y);
/* Halo pack / unpack: dst[i] = src[idx[i]]; dst[idx[i]] = src[i] or
 * dst[idx[i]] += src[i] (add != 0); idx entries unique. */
int sag_gather_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* dst);
int sag_scatter_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* dst, int add);
/* Peer memory for a partitioned sweep: a rank exports a device buffer
 * (64-byte CUDA IPC handle) and its neighbours map it, so the reverse halo of
 * the Vanka sweep is written straight into the owner's receive buffer over
 * NVLink (sag_gather_async with the peer pointer as destination) instead of
 * a send / receive pair. */
int sag_ipc_get_handle(sag_ctx* ctx, void* dptr, unsigned char* handle);
int sag_ipc_open_handle(sag_ctx* ctx, const unsigned char* handle, void** dptr);
int sag_ipc_close_handle(sag_ctx* ctx, void* dptr);
/* peer_dst[i] = src[idx[i]] into a mapped neighbour buffer (NVLink stores,
 * system-scope fence): the reverse halo's send half. */
int sag_push_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* peer_dst);
/* norm_inf (sparse.cpp:229-237): max absolute row sum (host out). */
int sag_matrix_norm_inf(sag_ctx* ctx, const sag_matrix* m, double* out);
/* Refactors the coarse dense LU with the enclosed-flow pin
 * 1e-12 * level0_norm_inf (preconditioner.cpp:49-53) when the caller's
 * hierarchy starts below the level whose norm the reference uses -- a rank
 * that holds the agglomerated coarse levels of a partitioned hierarchy. */
int sag_dc_set_coarse_pin(sag_ctx* ctx, sag_dc* d, double level0_norm_inf);

#ifdef __cplusplus
}
#endif
#endif /* SAG_H */
