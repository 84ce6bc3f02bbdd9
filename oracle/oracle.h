/* TEST INFRASTRUCTURE ONLY -- the parity checker, never the product path.
 *
 * Plain-C restatement of the reference's solve-phase hot path
 * (stokesamg, /root/reference/proj/core). Each function cites the reference
 * file:line it follows. Loops keep the reference's order of operations and the
 * library is compiled with -ffp-contract=off, so on the same inputs it is
 * bitwise identical to the reference (pinned by tests/test_oracle.py against
 * oracle/_ref and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef SAG_ORACLE_H
#define SAG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference exception classes (errors.hpp:8-58) */
enum {
  OR_OK = 0,
  OR_ERROR = 1,
  OR_DIM = 2,
  OR_SINGULAR_MATRIX = 3,
  OR_SINGULAR_PATCH = 4,
  OR_CONFIG = 5,
  OR_STAGNATION = 6,
};

/* CSR view (sparse.hpp:11-28); arrays are borrowed, never freed here */
typedef struct {
  int nrows, ncols;
  const int* rp;
  const int* ci;
  const double* v;
} or_csr;

/* sparse.cpp:78-91 */
void or_spmv(const or_csr* m, const double* x, double* y);
/* sparse.cpp:217-227 */
double or_norm2(int n, const double* v);
double or_dot(int n, const double* a, const double* b);
/* sparse.cpp:229-237 */
double or_norm_inf(const or_csr* m);
/* sparse.cpp:310-341: in-place packed LU of a row-major n x n matrix */
int or_lu_factor(int n, double* a, int* piv);
/* sparse.cpp:343-361 */
void or_lu_solve(int n, const double* lu, const int* piv, double* b);

/* vanka.hpp:11-15 / vanka.cpp:11-42 */
typedef struct {
  int npatch;
  int *pptr, *pidx; /* pressure rows of patch i: pidx[pptr[i]..pptr[i+1]) */
  int *vptr, *vidx; /* sorted velocity DoFs */
  int* nx;          /* x-component count */
} or_patches;
int or_build_patches(const or_csr* k, int n_x, int n_y, int n_p, int sv_triples,
                     or_patches* out);
void or_patches_free(or_patches* p);

/* vanka.hpp:23-40 */
typedef struct {
  or_patches pat; /* own copy */
  int n;
  int64_t *lu_off, *aux_off; /* per patch offsets into lu[] / uhat[],bhat[] / sinv[] */
  int64_t* s_off;
  double* lu; /* lu_x (nx*nx) then lu_y (ny*ny), row-major */
  int* piv;   /* same layout, per row */
  int64_t* piv_off;
  double *uhat, *bhat, *sinv; /* nv x np, np x nv, np x np row-major */
  double* weights;
  int64_t a_factor_bytes, aux_bytes, dense_inverse_bytes;
} or_vanka;
/* vanka.cpp:64-149 */
int or_factor_patches(const or_csr* k, const or_patches* p, int n_u, or_vanka* out);
void or_vanka_free(or_vanka* f);
/* vanka.cpp:151-184 */
void or_apply_vanka(const or_vanka* f, const double* r, double* delta);

/* The 3-component generalisation (BASELINE config 5, which the reference does
 * not support): K rows [x | y | z | p], one pressure seed per patch,
 * the velocity set split into its x, y, z parts by the block sizes, one LU per
 * component, then vanka.cpp:99-184 with three blocks instead of two. */
typedef struct {
  int npatch;
  int *pptr, *pidx, *vptr, *vidx;
  int* cnt; /* 3 per patch: x, y, z counts */
} or_patches3;
typedef struct {
  or_patches3 pat;
  int n;
  int64_t *lu_off, *piv_off, *aux_off, *s_off;
  double* lu; /* lu_x | lu_y | lu_z, row-major */
  int* piv;
  double *uhat, *bhat, *sinv, *weights;
} or_vanka3;
int or_build_patches3(const or_csr* k, int n_x, int n_y, int n_z, int n_p, or_patches3* out);
void or_patches3_free(or_patches3* p);
int or_factor_patches3(const or_csr* k, const or_patches3* p, or_vanka3* out);
void or_vanka3_free(or_vanka3* f);
void or_apply_vanka3(const or_vanka3* f, const double* r, double* delta);

/* krylov.hpp:12, :17-35 */
typedef void (*or_op)(void* ctx, const double* x, double* y);
typedef struct {
  double tol;
  int max_iters;
  int restart;
  double breakdown;
} or_fgmres_opts;
typedef struct {
  int converged;
  int iterations;
  double final_relative_residual;
  int history_len;
} or_report;
/* krylov.cpp:17-121; hist may be NULL (cap entries are stored) */
int or_fgmres(int n, or_op a, void* actx, const double* b, double* x, or_op prec, void* pctx,
              const or_fgmres_opts* opt, or_report* rep, double* hist, int cap);

/* vanka.cpp:186-209; mode 0 = KrylovWrapped, 1 = Stationary */
int or_vanka_relax(const or_csr* k, const or_vanka* f, double* x, const double* b, int mode,
                   int sweeps, double omega);

/* preconditioner.hpp:53-73: MonolithicSolver on a given hierarchy */
typedef struct {
  int nlevels;
  or_csr* k;     /* nlevels (borrowed arrays) */
  or_csr* p;     /* nlevels-1 (borrowed arrays) */
  int* nxyz;     /* 3 per level */
  or_vanka* vanka; /* nlevels-1, owned */
  int nc;
  double* coarse_lu;
  int* coarse_piv;
} or_mono;
/* preconditioner.cpp:40-55; pin = 1e-12*norm_inf(K of level 0) when enclosed */
int or_mono_setup(or_mono* m, int nlevels, const or_csr* ks, const or_csr* ps, const int* nxyz,
                  int enclosed);
void or_mono_free(or_mono* m);
/* preconditioner.cpp:83-88 (skip_finest_relax = 0) */
int or_vcycle(const or_mono* m, const double* b, double* x, int nu1, int nu2);

/* preconditioner.hpp:19-36 */
typedef struct {
  int variant; /* 0 DCall, 1 DCLO, 2 DCHO */
  double eta_u, eta_p, omega0;
  int nu1, nu2, gamma, restart;
  double tol;
  int max_iters;
  int enclosed_flow;
} or_config;

/* preconditioner.hpp:77-100, TH injection transfer (transfer.cpp:97-125) */
typedef struct {
  or_csr k0;
  int n_x0, n_y0, n_p0;
  int stationary_fine; /* SV */
  or_vanka fine;
  or_mono mono;
  or_config cfg;
} or_dc;
int or_dc_setup(or_dc* d, const or_csr* k0, int n_x0, int n_y0, int n_p0, int sv,
                int nlevels, const or_csr* ks, const or_csr* ps, const int* nxyz,
                const or_config* cfg);
void or_dc_free(or_dc* d);
/* preconditioner.cpp:114-153 */
int or_dc_apply(const or_dc* d, const double* r, double* z);
/* preconditioner.cpp:229-259 */
int or_solve_stokes(const or_dc* d, const double* rhs, double* x, or_report* rep, double* hist,
                    int cap);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
