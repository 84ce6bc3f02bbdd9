// Internal C++ objects behind the C-ABI handles, device-side scalar state of
// the Krylov solvers, and the host-side launchers shared by the .cu files.
#pragma once

#include <atomic>
#include <memory>

#include "common.cuh"

struct sag_ctx {
  sag::Ctx c;
};

namespace sag {

// process-wide serial number of a device matrix: plans cached against an
// operator (the pipelined step) compare it, not the address, so a matrix
// created later at the same address is never mistaken for the planned one
inline unsigned long long next_matrix_uid() {
  static std::atomic<unsigned long long> n{0};
  return ++n;
}

// CSR on device (sparse.hpp:11-28). `group` = lanes per row used by SpMV.
struct Matrix {
  unsigned long long uid = next_matrix_uid();
  Ctx* ctx = nullptr;
  int nrows = 0, ncols = 0;
  long long nnz = 0;
  DevBuf<int> rp, ci;
  DevBuf<double> v;
  int group = 8;
  double norm_inf = -1.0;  // cached (sparse.cpp:229-237)
};
// CSR arrays carry kCsrPad elements of slack (vectorised tail loads stay
// inside the allocation)
constexpr int kCsrPad = 4;

// Vanka patch sets (vanka.hpp:11-15), CSR-like on device.
struct Patches {
  int npatch = 0;
  long long tot_p = 0, tot_v = 0;
  int max_nv = 0, max_np = 0, max_dim = 0;  // max_dim = max over patches of max(nx, ny)
  DevBuf<int> pptr, pidx, vptr, vidx, nx;
};

// Device factorization (vanka.hpp:23-40) in the apply representation: one
// 16-byte-aligned blob per patch
//   header {int nx, ny, np, slot_base}
//   A_x^-1 (nx*nx, column-major) | A_y^-1 (ny*ny, column-major)
//   U_hat  (np rows of nv: [a*nv+i] = u_hat(i,a))
//   B_hat  (np rows of nv: [a*nv+j] = b_hat(a,j))
//   S^-1   (np*np row-major)
//   velocity dofs (nv int32) | pressure dofs (np int32) | pad to 16 B
// plus the PoU weights and the dof -> slot map of the atomic-free
// owner-computes scatter: each dof sums its patch contributions in ascending
// patch order, the order of vanka.cpp:176-181.
struct Vanka {
  int n = 0, npatch = 0;
  DevBuf<unsigned char> blob;
  DevBuf<long long> off;  // npatch + 1, bytes
  int slot_bytes = 0;     // max blob bytes
  // blob size classes (rows per lane R), stored contiguously: patches
  // [k0, k1) of the blob order, max blob bytes of the class
  struct RClass {
    int R, k0, k1;
    long long slot_bytes;
    int lpp;  // lanes per patch: 32, or 16 / 8 for the sub-warp kernel
    long long bytes = 0;  // blob bytes of the class
    int fm = 0, fnp = 0;  // fixed shape (nx = ny = fm, np = fnp; vanka_fixed_kernel), or 0
  };
  std::vector<RClass> rclasses;
  int max_dim = 0, max_nv = 0, max_np = 0;
  long long nslots = 0;
  DevBuf<double> out;     // per-patch local results (nslots)
  DevBuf<double> w;       // PoU weights (n)
  bool w_ext = false;     // w set by sag_vanka_set_weights (else 1/multiplicity on the fly)
  DevBuf<int> dof_ptr;    // n + 1
  DevBuf<int> dof_slot;   // nslots
  // dof-ordered results (seq): each blob also carries, after its dof indices,
  // the position of each local result in the dof-sorted order (dof, then
  // patch), so the patch kernel writes there and the gather reads every
  // dof's contributions as one contiguous run -- no dof_slot indirection
  bool seq = false;
  long long a_factor_bytes = 0, aux_bytes = 0, dense_inverse_bytes = 0;
  long long blob_bytes = 0;
  bool sym = false;  // A^-1 blocks stored as packed symmetrised upper triangles
  // paired blobs (every patch of a level, or none): np <= 4 pressure seeds
  // and m + np <= 64 (m = max(nx, ny)); pair_rows = max(m + np) sets the
  // kernel's rows per lane. They store (A_x, A_y), (U_x, U_y), (B_x, B_y) interleaved
  // element by element, the smaller component zero-padded to m, so the apply
  // loads both components with one 16-byte shared-memory access
  bool pairs = false;
  int pair_rows = 0;
  // per-patch payload bases and shapes (host copies, for export)
  std::vector<long long> h_dbase, h_ibase;
  std::vector<int> h_nx, h_nv, h_np;
  std::vector<unsigned char> h_nob;  // per patch: blob without b_hat (fixed-shape class)
  int n_u = 0;                       // velocity block size given to factor_patches
  std::vector<int> h_order;          // blob position -> patch id
  // pipelined host-buffer step (sag_vanka_spmv), planned per operator on first use
  mutable std::shared_ptr<struct StepPlan> step_plan;

};

// Krylov scalar state in device memory (one per FGMRES instance); mirrors the
// host scalars of krylov.cpp:17-121.
// Per-patch rule for the paired blob layout (factor, apply and export agree).
// m rows + np b_hat rows, one or two per lane (the R <= 2 kernels)
__host__ __device__ inline bool vanka_paired(bool pairs, int nx, int ny, int np) {
  const int m = nx > ny ? nx : ny;
  return pairs && np >= 1 && np <= 4 && m + np <= 64;
}
// doubles of a paired blob of padded size m with np pressure seeds:
// A pairs (m x m packed) | U pairs [a][i] | B pairs [a][j] | S^-1 (np x np)
__host__ __device__ inline long long vanka_paired_doubles(int m, int np) {
  return (long long)m * (m + 1) + 4LL * np * m + (long long)np * np;
}

struct KState {
  double ref, tol, bd;
  double beta, rnorm, wnorm;
  int m, stop, breakdown, jeff, iterations, hist_len, hist_cap, converged;
  // followed by h[(m+1)*m], cs[m], sn[m], g[m+1], y[m], hist[hist_cap]
};
__host__ __device__ inline size_t kstate_bytes(int m, int hist_cap) {
  return sizeof(KState) +
         sizeof(double) * ((size_t)(m + 1) * m + m + m + (m + 1) + m + hist_cap);
}
__host__ __device__ inline double* ks_h(KState* s) { return reinterpret_cast<double*>(s + 1); }
__host__ __device__ inline double* ks_cs(KState* s) { return ks_h(s) + (size_t)(s->m + 1) * s->m; }
__host__ __device__ inline double* ks_sn(KState* s) { return ks_cs(s) + s->m; }
__host__ __device__ inline double* ks_g(KState* s) { return ks_sn(s) + s->m; }
__host__ __device__ inline double* ks_y(KState* s) { return ks_g(s) + s->m + 1; }
__host__ __device__ inline double* ks_hist(KState* s) { return ks_y(s) + s->m; }

// What the last block of a reducing kernel does with the total.
enum FinKind {
  FIN_NONE = 0,
  FIN_STORE,      // *out = tot
  FIN_SQRT,       // *out = sqrt(tot)
  FIN_MEAN,       // *out = tot / i
  FIN_REF,        // st->ref = sqrt(tot) > 0 ? sqrt(tot) : 1           (krylov.cpp:23-24)
  FIN_BETA,       // (re)start: beta = rnorm = sqrt(tot); g = beta e_0;   (krylov.cpp:44-53)
  FIN_H,          // h[i*m+j] = tot                                       (krylov.cpp:64-65)
  FIN_ARNOLDI,    // wnorm = sqrt(tot); Givens; residual estimate        (krylov.cpp:68-100)
  FIN_FINAL,      // *out = sqrt(tot) / st->ref                           (krylov.cpp:116-118)
};
struct Fin {
  int kind = FIN_NONE;
  KState* st = nullptr;
  int i = 0, j = 0;
  double* out = nullptr;
  double tol = 0.0;  // FIN_BETA with bit 4: (re)initialise st (m = j, tol, bd = 1e-30)
};

__device__ void apply_fin(const Fin& f, double tot);

// SpMV epilogues: y_i from the row sum s_i
enum class Epi {
  Store,      // y = s
  Resid,      // y = b - s
  ResidEta,   // y = eta_(u|p) * (b - s)     (residual + apply_eta_weighting, transfer.cpp:127-135)
  Add,        // y += s                      (x += P xc, preconditioner.cpp:75-76)
  StoreDot,   // y = s, reduce y * dotv      (w = A z_j fused with h_0j, krylov.cpp:61-64)
  ResidSsq,   // y = b - s, reduce y^2       (residual + norm2, krylov.cpp:44-46)
};

struct SpmvArgs {
  const double* b = nullptr;
  const double* dotv = nullptr;
  double eta_u = 1.0, eta_p = 1.0;
  int n_u = 0;
  Fin fin;
  const int* gate = nullptr;  // skip the whole launch when *gate != 0
};

void launch_spmv(Ctx& c, const Matrix& m, const double* x, double* y, Epi e,
                 const SpmvArgs& a = SpmvArgs());
void compute_norm_inf(Ctx& c, Matrix& m);
// y[r0, r1) = (K x)[r0, r1)  (Store)
void launch_spmv_rows(Ctx& c, const Matrix& m, int r0, int r1, const double* x, double* y);

// deterministic BLAS-1 (reductions finish through Fin)
void launch_dot(Ctx& c, int n, const double* a, const double* b, const Fin& fin,
                const int* gate = nullptr);
void launch_ssq(Ctx& c, int n, const double* a, const Fin& fin, const int* gate = nullptr);
void launch_sum(Ctx& c, int n, const double* a, const Fin& fin);
// y = x / *s (skipped when *gate or *gate2)
void launch_div(Ctx& c, int n, const double* x, const double* s, double* y, const int* gate,
                const int* gate2 = nullptr);
// w -= (*h) * vprev; reduce w . vnext (vprev may be null)        (krylov.cpp:63-67)
void launch_mgs(Ctx& c, int n, double* w, const double* vprev, const double* h,
                const double* vnext, const Fin& fin, const int* gate);
// w -= (*h) * v; reduce w . w
void launch_mgs_last(Ctx& c, int n, double* w, const double* v, const double* h, const Fin& fin,
                     const int* gate, bool write_w = true);
// r = eta .* (b - y_0 w): residual after a one-step relaxation x = y_0 z_0
// whose w = K z_0 is kept (K x by linearity, no SpMV)
void launch_lin_resid(Ctx& c, int n, int n_u, double eta_u, double eta_p, const double* b,
                      const double* w, const KState* st, double* r);
// y = back-substitution of the jeff x jeff Hessenberg system (krylov.cpp:102-107)
void launch_backsub(Ctx& c, KState* st);
// x += sum_{i<jeff} y_i Z_i   (krylov.cpp:108-110 then vanka.cpp:208);
// store = true: x = sum (x was zero)
void launch_update(Ctx& c, int n, double* x, const double* Z, size_t zstride, KState* st,
                   bool store = false);
// z = dinv * r
void launch_mul(Ctx& c, int n, const double* a, const double* b, double* y);
// ||a||^2 applied to two finishers (one pass)
void launch_ssq2(Ctx& c, int n, const double* a, const Fin& f1, const Fin& f2);
// y = x / *s, z = d .* y (skipped when *gate)
void launch_div_mul(Ctx& c, int n, const double* x, const double* s, double* y, const double* d,
                    double* z, const int* gate);
// launch_backsub + launch_update in one launch when the restart length m is
// at most kUpdBsMax (else the two launches)
constexpr int kUpdBsMax = 4;
void launch_update_bs(Ctx& c, int n, double* x, const double* Z, size_t zstride, KState* st,
                      int m, bool store = false);
// dinv_i = 1 / a_ii; returns false (via *bad) if a diagonal entry is missing/zero
void launch_inv_diag(Ctx& c, const Matrix& m, double* dinv, int* bad);

// The small levels of a scalar V(2,2) cycle (amg.cpp:258-296) in ONE launch:
// a thread-block cluster whose CTAs own contiguous row chunks of every level.
// All level vectors live in the CTAs' shared memory (SpMV gathers read the
// other CTAs' chunks over DSMEM), cluster barriers separate the phases, and
// the Krylov scalars of every Jacobi-FGMRES(2) smoother are computed
// redundantly (identically) in each CTA from DSMEM-gathered partial sums.
// Replaces ~30 dependent small launches per level; levels run from L[0]
// (b0 given, x0 out, global memory) down to the coarse L[nlev-1].
// A few row (or dof) ranges handled by one launch: virtual index v in
// [vstart[k], vstart[k + 1]) is row row0[k] + v - vstart[k].
constexpr int kMaxRowRanges = 12;
struct RowRanges {
  int n = 0;
  int vstart[kMaxRowRanges + 1] = {0};
  int row0[kMaxRowRanges] = {0};
  __host__ __device__ int total() const { return vstart[n]; }
  __device__ __forceinline__ int row(int v) const {
    int k = 0;
#pragma unroll
    for (int i = 1; i < kMaxRowRanges; ++i)
      if (i < n && v >= vstart[i]) k = i;
    return row0[k] + v - vstart[k];
  }
  bool push(int a, int b) {  // host: append rows [a, b); false when full
    if (n >= kMaxRowRanges) return false;
    row0[n] = a;
    vstart[n + 1] = vstart[n] + (b - a);
    ++n;
    return true;
  }
};
// y[rows] = (A x)[rows] for the rows of R, on stream st
void launch_spmv_ranges(Ctx& c, const Matrix& m, const RowRanges& R, const double* x, double* y,
                        cudaStream_t st);

// Sliced ELLPACK copy of a CSR matrix for the persistent small-level kernels.
// G = 2^g lanes share a row (g from the mean row length); a slice is 32 / G
// consecutive rows; entry k of row r (rho = r % (32 / G)) is word
// sptr[r / (32 / G)] + 32 (k / G) + rho G + k % G, so each step of a warp
// reads 32 consecutive entries and no row pointer is needed per row. Rows are
// padded to the slice's longest row with (value 0, the row's last column:
// the gather stays unconditional and local). A row's sum is the shuffle tree
// over its G lanes of the lanes' sums in ascending k.
struct SellView {
  const int* sptr = nullptr;  // nslices + 1 entry offsets (multiples of 32)
  const int* ci = nullptr;
  const double* v = nullptr;
  int g = 0;                  // log2 lanes per row
};
struct Sell {
  DevBuf<int> sptr, ci;
  DevBuf<double> v;
  long long entries = 0;
  int g = 0;
  SellView view() const { return SellView{sptr.p, ci.p, v.p, g}; }
};
void build_sell(Ctx& c, const Matrix& m, Sell& out);

constexpr int kTailMaxLev = 6;
constexpr int kTailVecs = 9;  // b x r rs w v0 v1 z0 z1 per level
struct TailLevel {
  int n = 0, chunk = 0, off = 0;  // rows, rows per CTA, shared-memory offset (doubles)
  const int *arp = nullptr, *aci = nullptr;
  const double* av = nullptr;     // A_l
  const int *rrp = nullptr, *rci = nullptr;
  const double* rv = nullptr;     // R_l = P_l^T (not on the coarse level)
  const int *prp = nullptr, *pci = nullptr;
  const double* pv = nullptr;     // P_l
  const double* dinv = nullptr;
};
struct TailParams {
  int nlev = 0, cs = 0;           // levels (the last is the coarse one), CTAs per cluster
  size_t smem = 0;                // dynamic shared memory per CTA
  TailLevel L[kTailMaxLev];
  const double* cinv = nullptr;   // n x n row-major inverse of the coarse level
  const double* b0 = nullptr;     // per launch: right-hand side of L[0]
  double* x0 = nullptr;           // per launch: result on L[0]
};
// The SV pressure mass projection p_cg = Mcg^-1 (M_mix p_dg)
// (transfer.cpp:18-37: FGMRES(20) to 1e-12, scalar V(2,2) preconditioner,
// amg.cpp:258-296) as ONE persistent launch. The grid is a set of clusters:
// cluster 0 runs the small levels exactly as scalar_tail_kernel does; the
// CTAs of the other clusters ("workers") own contiguous row chunks of the
// large ("grid") levels, whose gathered vectors live in global memory (L2
// resident) and whose pointwise vectors live in the owner's shared memory.
// A gathered vector's producer and consumers are separated by a grid-wide
// barrier (release fence + one atomic per CTA). A reduction needs no barrier:
// every worker publishes its partial as two 8-byte {half of the value, phase
// number} words (each an atomic store, so data and flag arrive together) and
// every CTA polls all workers' words and sums them in worker order, so every
// CTA holds the same Krylov scalars (KState in shared memory, updated by
// apply_fin) and takes the same branches.
constexpr int kProjMaxGl = 3;        // grid levels
constexpr int kProjMaxRestart = 20;
struct ProjLevel {
  int n = 0, chunk = 0;           // rows, rows per worker (a multiple of 32)
  SellView a;                     // A_l
  SellView rt;                    // R_l = P_l^T (rows of level l + 1)
  SellView p;                     // P_l
  const double* dinv = nullptr;
  int nc = 0, cchunk = 0;         // rows of level l + 1, per worker
  double *b = nullptr, *x = nullptr;  // level vectors (level 0: set per Arnoldi step)
  double *r = nullptr, *z0 = nullptr, *z1 = nullptr;
};
struct ProjParams {
  int ngl = 0, grid = 0, workers = 0;
  size_t smem = 0;
  ProjLevel G[kProjMaxGl];
  TailParams tail;                // levels ngl..; b0 / x0 are global work vectors
  int n = 0;                      // rows of level 0 (Mcg)
  SellView mm;                    // M_mix (n rows)
  const double* p_dg = nullptr;   // per launch: input
  double* x = nullptr;            // per launch: result p_cg (n)
  double *rhs = nullptr, *V = nullptr, *Z = nullptr;  // n, (restart + 1) n, restart n
  KState* st = nullptr;           // outer KState (header + arrays written back at the end)
  int restart = 20, max_iters = 200;
  double tol = 1e-12, bd = 1e-30;
  unsigned* bar = nullptr;        // grid barrier counter; zeroed with the slots at launch
  unsigned long long* ll = nullptr;  // reduction slots [2][workers][2][2]: {value half, phase}
  size_t sync_bytes = 0;          // bytes from bar to zero at launch
  int* fail = nullptr;            // set when the solve did not converge
  // diagnostic (SAG_PROJ_TRACE): (phase tag, globaltimer ns) pairs of worker
  // 0 [0, 2 cap) and of tail CTA 0 [2 cap, 4 cap)
  unsigned long long* trace = nullptr;
  int trace_cap = 0;
};
// grid, chunks and shared memory for p (levels and tail set); false when the
// device cannot hold the grid levels' chunks or co-schedule the clusters
bool sv_project_plan(Ctx& c, ProjParams& p);
void launch_sv_project(Ctx& c, const ProjParams& p);

// cluster size, row chunks and shared-memory layout for p.L[0..nlev) (n set);
// false when no resident cluster can hold the levels
bool scalar_tail_plan(Ctx& c, TailParams& p);
void launch_scalar_tail(Ctx& c, const TailParams& p);
// KState (re)initialisation for a new solve: ref/tol/bd/m/iterations
void launch_kinit(Ctx& c, KState* st, int m, double tol, double bd, int hist_cap,
                  bool keep_ref);
void launch_copy(Ctx& c, int n, const double* x, double* y);
void launch_zero(Ctx& c, int n, double* y);
// partitioned-solve primitives on device scalars (sag_core.cu)
void launch_fin_from(Ctx& c, const Fin& f, const double* tot);  // apply_fin(f, *tot)
// *out = sum over i with mask[i] (all i when mask is null) of a_i b_i
void launch_dot_mask(Ctx& c, int n, const double* a, const double* b, const unsigned char* mask,
                     double* out);
void launch_axpy_dev(Ctx& c, int n, const double* s, double sign, const double* x, double* y);
void launch_div_dev(Ctx& c, int n, const double* x, const double* s, int take_sqrt, double* y);
void launch_fgmres1_coef(Ctx& c, const double* ssq_r, const double* h00, const double* ssq_w,
                         double* y0);
void launch_sub_mean(Ctx& c, int n, const double* x, const double* sum, double count, double* y);
void launch_axpby(Ctx& c, int n, double a, const double* x, double b, double* y);
void launch_gather_idx(Ctx& c, int n, const int* idx, const double* src, double* dst);
void launch_scatter_idx(Ctx& c, int n, const int* idx, const double* src, double* dst, int add);
// y = x with the pressure block shifted by -(*mean)   (preconditioner.cpp:235-240)
void launch_project(Ctx& c, int n, int n_u, const double* x, const double* mean, double* y);
// y = eta_u * x (i < n_u), eta_p * x (i >= n_u)   (transfer.cpp:127-135)
void launch_eta(Ctx& c, int n, int n_u, double eta_u, double eta_p, const double* x, double* y);
// x += y
void launch_add(Ctx& c, int n, double* x, const double* y);
// x += omega * d
void launch_axpy(Ctx& c, int n, double* x, double omega, const double* d);

// Vanka: delta = apply_vanka(r) (vanka.cpp:151-184). With `div`, r is read as
// r / *div (v_0 = r / ||r||, krylov.cpp:47). With `xadd`, the gather adds
// omega*delta into xadd instead of storing delta (vanka.cpp:195).
void vanka_apply(Ctx& c, const Vanka& f, const double* r, double* delta,
                 const int* gate = nullptr);
void vanka_apply_stage(Ctx& c, const Vanka& f, const double* r, double* delta, int stage);
void vanka_apply_stationary(Ctx& c, const Vanka& f, const double* r, double* x, double omega);
// the gather stage for dofs [d0, d1) only (delta = the unweighted-sum store)
void vanka_gather_range(Ctx& c, const Vanka& f, int d0, int d1, double* delta);
std::unique_ptr<Patches> build_patches_dev(Ctx& c, const Matrix& k, int n_x, int n_y, int n_p,
                                           bool sv_triples);
std::unique_ptr<Patches> patches_from_lists(Ctx& c, int npatch, const int* pptr,
                                            const int* pidx, const int* vptr, const int* vidx,
                                            const int* nx);
std::unique_ptr<Vanka> factor_patches_dev(Ctx& c, const Matrix& k, const Patches& p, int n_u);
// the reference's factor layout, for parity tests (vanka.hpp:31-33)
void vanka_export(Ctx& c, const Vanka& f, double* uhat, double* bhat, double* sinv,
                  double* weights);

// transpose on device (sparse.cpp:93-111): rows of the result in ascending order
std::unique_ptr<Matrix> transpose_dev(Ctx& c, const Matrix& a);
std::unique_ptr<Matrix> matrix_upload(Ctx& c, int nrows, int ncols, long long nnz, const int* rp,
                                      const int* ci, const double* v);
// setup products, bitwise the reference's (sag_setup.cu)
std::unique_ptr<Matrix> spgemm_dev(Ctx& c, const Matrix& a, const Matrix& b);
std::unique_ptr<Matrix> smooth_prolongator_dev(Ctx& c, const Matrix& a, const Matrix& t,
                                               double omega);

}  // namespace sag

struct sag_matrix {
  sag::Matrix m;
};
struct sag_patches {
  sag::Patches p;
};
struct sag_vanka {
  sag::Vanka f;
  sag::Ctx* c = nullptr;  // the context whose stream the factorization's kernels run on
};
