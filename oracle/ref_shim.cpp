// TEST INFRASTRUCTURE ONLY -- the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference library (stokesamg, compiled
// from /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).
// It lets the Python test-suite and bench.py's cpu_baseline leg drive the
// reference's own code path: case construction (experiments.cpp:215-235),
// spmv (sparse.cpp:78-91), build_patches/factor_patches/apply_vanka/vanka_relax
// (vanka.cpp:11-209), fgmres (krylov.cpp:17-121), DCPreconditioner::apply
// (preconditioner.cpp:114-153) and solve_stokes (preconditioner.cpp:229-259).
// Nothing in here re-implements reference arithmetic; it only marshals arrays.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "stokesamg/errors.hpp"
#include "stokesamg/experiments.hpp"

using namespace stokesamg;

namespace {

thread_local std::string g_err;

struct H {
  virtual ~H() = default;
};
struct MatH : H {
  SparseMatrix m;
};
struct CaseH : H {
  AssembledCase c;
};
struct VankaH : H {
  std::vector<VankaPatch> patches;
  VankaFactorization own;
  const VankaFactorization* f = nullptr;  // &own, or borrowed from a DC handle
  int n = 0;
};
struct DcH : H {
  SolverConfig cfg;
  std::unique_ptr<DCPreconditioner> prec;
  int n_p1 = 0;
};

enum : int {
  OK = 0,
  E_ERROR = 1,
  E_DIM = 2,
  E_SINGULAR_MATRIX = 3,
  E_SINGULAR_PATCH = 4,
  E_CONFIG = 5,
  E_STAGNATION = 6,
  E_ZERO_DIAG = 7,
  E_UNSUPPORTED = 8,
  E_OTHER = 99,
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return OK;
  } catch (const DimensionMismatch& e) {
    g_err = e.what();
    return E_DIM;
  } catch (const SingularMatrix& e) {
    g_err = e.what();
    return E_SINGULAR_MATRIX;
  } catch (const SingularPatch& e) {
    g_err = e.what();
    return E_SINGULAR_PATCH;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return E_CONFIG;
  } catch (const SolverStagnation& e) {
    g_err = e.what();
    return E_STAGNATION;
  } catch (const ZeroDiagonal& e) {
    g_err = e.what();
    return E_ZERO_DIAG;
  } catch (const UnsupportedDiscretization& e) {
    g_err = e.what();
    return E_UNSUPPORTED;
  } catch (const Error& e) {
    g_err = e.what();
    return E_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_OTHER;
  }
}

SparseMatrix csr_in(int nr, int nc, long long nnz, const int* rp, const int* ci, const double* v) {
  SparseMatrix m(nr, nc);
  m.row_offsets.assign(rp, rp + nr + 1);
  m.col_indices.assign(ci, ci + nnz);
  m.values.assign(v, v + nnz);
  return m;
}

void csr_out(const SparseMatrix& m, int* rp, int* ci, double* v) {
  std::memcpy(rp, m.row_offsets.data(), sizeof(int) * (m.nrows + 1));
  std::memcpy(ci, m.col_indices.data(), sizeof(int) * m.col_indices.size());
  std::memcpy(v, m.values.data(), sizeof(double) * m.values.size());
}

MatH* new_mat(SparseMatrix m) {
  auto* h = new MatH;
  h->m = std::move(m);
  return h;
}

struct RefFgmresOpts {
  double tol;
  int max_iters;
  int restart;
  double breakdown;
};
struct RefReport {
  int converged;
  int iterations;
  double final_relative_residual;
  int history_len;
};
struct RefConfig {
  int variant;
  double eta_u, eta_p, omega0;
  int nu1, nu2, gamma, restart;
  double tol;
  int max_iters;
  int enclosed_flow;
  int coarse_size;
};

void report_out(const KrylovReport& r, RefReport* rep, double* hist, int cap) {
  if (rep) {
    rep->converged = r.converged ? 1 : 0;
    rep->iterations = r.iterations;
    rep->final_relative_residual = r.final_relative_residual;
    rep->history_len = static_cast<int>(r.residual_history.size());
  }
  if (hist)
    for (int i = 0; i < cap && i < static_cast<int>(r.residual_history.size()); ++i)
      hist[i] = r.residual_history[i];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* h) { delete static_cast<H*>(h); }

// ----------------------------------------------------------------- matrices
void* ref_mat_new(int nr, int nc, long long nnz, const int* rp, const int* ci, const double* v) {
  return new_mat(csr_in(nr, nc, nnz, rp, ci, v));
}

void* ref_mat_from_triplets(int nr, int nc, long long nt, const int* r, const int* c,
                            const double* v) {
  std::vector<Triplet> t(nt);
  for (long long i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
  MatH* out = nullptr;
  if (guard([&] { out = new_mat(from_triplets(nr, nc, std::move(t))); }) != OK) return nullptr;
  return out;
}

int ref_mat_shape(void* h, int* nr, int* nc, long long* nnz) {
  const auto& m = static_cast<MatH*>(h)->m;
  *nr = m.nrows;
  *nc = m.ncols;
  *nnz = m.nnz();
  return OK;
}

int ref_mat_copy(void* h, int* rp, int* ci, double* v) {
  csr_out(static_cast<MatH*>(h)->m, rp, ci, v);
  return OK;
}

int ref_spmv(void* h, const double* x, double* y) {
  const auto& m = static_cast<MatH*>(h)->m;
  return guard([&] {
    std::vector<double> xv(x, x + m.ncols);
    auto yv = spmv(m, xv);
    std::memcpy(y, yv.data(), sizeof(double) * yv.size());
  });
}

double ref_norm_inf(void* h) { return norm_inf(static_cast<MatH*>(h)->m); }

void* ref_transpose(void* h) { return new_mat(transpose(static_cast<MatH*>(h)->m)); }

// dense LU (sparse.cpp:310-369) on a row-major n x n matrix
int ref_dense_lu_solve(int n, const double* a, const double* b, double* x) {
  return guard([&] {
    DenseMatrix d(n, n);
    std::memcpy(d.values.data(), a, sizeof(double) * n * n);
    auto f = dense_lu_factor(d);
    std::vector<double> bv(b, b + n);
    auto xv = dense_lu_solve(f, bv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

// -------------------------------------------------------------------- cases
// build_case (experiments.cpp:215-235) for the named problem/discretization.
void* ref_case_build(const char* problem, int sv, const char* mesh_kind, int n,
                     const char* mesh_path, int refinement) {
  CaseH* out = nullptr;
  int rc = guard([&] {
    ExperimentSpec s;
    s.problem = problem;
    s.disc = sv ? Discretization::SV : Discretization::TH;
    s.mesh.kind = mesh_kind;
    s.mesh.n = n;
    if (mesh_path) s.mesh.path = mesh_path;
    auto* h = new CaseH;
    h->c = build_case(s, refinement);
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// A TH case on an n x n structured mesh with optional coordinate jitter (the
// reference tests' jittered meshes, tests/acceptance.cpp:29-39), selectable
// boundary tagging (0 = all Dirichlet, 1 = Neumann right side as in
// tests/test_preconditioner.cpp:12-14) and forcing (0 zero, 1 constant (1,0.3)
// as in tests/test_preconditioner.cpp:220-223, 2 = "forced" experiments.cpp:73-79).
void* ref_case_custom_th(int n, int tagger, double jitter, int force) {
  CaseH* out = nullptr;
  int rc = guard([&] {
    EdgeTagger tg = [tagger](double x, double) {
      if (tagger == 1 && x > 1 - 1e-12) return BoundaryTag::Neumann;
      return BoundaryTag::DirichletZero;
    };
    auto m = structured_tri_mesh(n, n, RectDomain{0, 0, 1, 1}, tg);
    if (jitter != 0.0) {
      for (int i = 0; i < m.num_vertices(); ++i) {
        auto& v = m.vertices[i];
        if (v[0] > 1e-12 && v[0] < 1 - 1e-12 && v[1] > 1e-12 && v[1] < 1 - 1e-12) {
          v[0] += jitter * std::sin(3.1 * i);
          v[1] += jitter * std::cos(2.7 * i);
        }
      }
    }
    ProblemData prob = zero_problem();
    if (force == 1) prob.force = [](double, double) { return std::array<double, 2>{1.0, 0.3}; };
    if (force == 2)
      prob.force = [](double x, double y) {
        return std::array<double, 2>{std::sin(3.0 * y) + 1.0, std::cos(2.0 * x)};
      };
    prob.check_compatibility = false;
    auto* h = new CaseH;
    h->c.enclosed = (tagger == 0);
    h->c.mesh = m;
    h->c.sys0 = assemble_taylor_hood(m, prob);
    auto [mf, qmap] = quadrisect(m);
    h->c.sys1 = assemble_iso(m, mf, qmap, prob);
    h->c.transfer = build_th_transfer(h->c.sys0, h->c.sys1);
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// BASELINE config 4 through the reference: mesh JSON read by read_mesh
// (mesh.cpp:230-289), every boundary edge DirichletZero, body force
// f = (sin(k1 x), cos(k2 y)), enclosed (all-Dirichlet) TH + ISO + transfer.
void* ref_case_mesh_forced(const char* path, double k1, double k2) {
  CaseH* out = nullptr;
  int rc = guard([&] {
    ProblemData prob = zero_problem();
    prob.force = [k1, k2](double x, double y) {
      return std::array<double, 2>{std::sin(k1 * x), std::cos(k2 * y)};
    };
    prob.check_compatibility = false;
    auto* h = new CaseH;
    h->c.enclosed = true;
    h->c.mesh = read_mesh(path);
    for (auto& be : h->c.mesh.boundary_edges) be.tag = BoundaryTag::DirichletZero;
    h->c.sys0 = assemble_taylor_hood(h->c.mesh, prob);
    auto [mf, qmap] = quadrisect(h->c.mesh);
    h->c.sys1 = assemble_iso(h->c.mesh, mf, qmap, prob);
    h->c.transfer = build_th_transfer(h->c.sys0, h->c.sys1);
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// out = [n_x0, n_y0, n_p0, n_x1, n_y1, n_p1, enclosed, sv]
int ref_case_info(void* h, int* out) {
  const auto& c = static_cast<CaseH*>(h)->c;
  out[0] = c.sys0.n_x;
  out[1] = c.sys0.n_y;
  out[2] = c.sys0.n_p;
  out[3] = c.sys1.n_x;
  out[4] = c.sys1.n_y;
  out[5] = c.sys1.n_p;
  out[6] = c.enclosed ? 1 : 0;
  out[7] = c.sys0.disc == Discretization::SV ? 1 : 0;
  return OK;
}

int ref_case_rhs(void* h, double* rhs) {
  const auto& r = static_cast<CaseH*>(h)->c.sys0.rhs;
  std::memcpy(rhs, r.data(), sizeof(double) * r.size());
  return OK;
}

void* ref_case_k0(void* h) { return new_mat(assemble_saddle_matrix(static_cast<CaseH*>(h)->c.sys0)); }
void* ref_case_k1(void* h) { return new_mat(assemble_saddle_matrix(static_cast<CaseH*>(h)->c.sys1)); }

// SV transfer pieces (transfer.cpp:45-53, :82-95): which = 0 p0_pressure
// (dg x cg duplication), 1 Mp_cg, 2 M_mix.
void* ref_case_sv_matrix(void* h, int which) {
  const auto& c = static_cast<CaseH*>(h)->c;
  if (which == 0) return new_mat(c.transfer.p0_pressure);
  if (which == 1) return new_mat(c.sys0.Mp_cg);
  return new_mat(c.sys0.M_mix);
}

int ref_transfer_restrict(void* h, const double* r0, double* r1) {
  const auto& t = static_cast<CaseH*>(h)->c.transfer;
  return guard([&] {
    std::vector<double> v(r0, r0 + t.n_u0 + t.n_p0);
    auto o = t.restrict_(v);
    std::memcpy(r1, o.data(), sizeof(double) * o.size());
  });
}

int ref_transfer_prolong(void* h, const double* x1, double* x0) {
  const auto& t = static_cast<CaseH*>(h)->c.transfer;
  return guard([&] {
    std::vector<double> v(x1, x1 + t.n_u1 + t.n_p1);
    auto o = t.prolong(v);
    std::memcpy(x0, o.data(), sizeof(double) * o.size());
  });
}

// -------------------------------------------------------------------- vanka
void* ref_vanka_build(void* kh, int n_x, int n_y, int n_p, int sv_triples) {
  const auto& k = static_cast<MatH*>(kh)->m;
  VankaH* out = nullptr;
  int rc = guard([&] {
    auto* h = new VankaH;
    h->patches = build_patches(k, n_x, n_y, n_p, sv_triples != 0);
    h->own = factor_patches(k, h->patches, n_x + n_y);
    h->f = &h->own;
    h->n = k.nrows;
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// Only build_patches (vanka.cpp:11-42), no factorization.
void* ref_build_patches(void* kh, int n_x, int n_y, int n_p, int sv_triples) {
  const auto& k = static_cast<MatH*>(kh)->m;
  VankaH* out = nullptr;
  int rc = guard([&] {
    auto* h = new VankaH;
    h->patches = build_patches(k, n_x, n_y, n_p, sv_triples != 0);
    h->n = k.nrows;
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// factor_patches on explicitly given patch lists (the reference tests build
// hand-made patches, tests/test_vanka.cpp:98-113).
void* ref_vanka_from_lists(void* kh, int npatch, const int* pptr, const int* pidx,
                           const int* vptr, const int* vidx, const int* nx, int n_u) {
  const auto& k = static_cast<MatH*>(kh)->m;
  VankaH* out = nullptr;
  int rc = guard([&] {
    auto* h = new VankaH;
    h->patches.resize(npatch);
    for (int i = 0; i < npatch; ++i) {
      h->patches[i].pressure.assign(pidx + pptr[i], pidx + pptr[i + 1]);
      h->patches[i].velocity.assign(vidx + vptr[i], vidx + vptr[i + 1]);
      h->patches[i].nx = nx[i];
    }
    h->own = factor_patches(k, h->patches, n_u);
    h->f = &h->own;
    h->n = k.nrows;
    out = h;
  });
  return rc == OK ? out : nullptr;
}

// out = [npatch, total pressure entries, total velocity entries,
//        a_factor_bytes, aux_bytes, dense_inverse_bytes, n]
int ref_vanka_info(void* h, long long* out) {
  auto* v = static_cast<VankaH*>(h);
  long long tp = 0, tv = 0;
  const int np = v->f ? static_cast<int>(v->f->patches.size()) : static_cast<int>(v->patches.size());
  for (int i = 0; i < np; ++i) {
    if (v->f) {
      tp += v->f->patches[i].pressure.size();
      tv += v->f->patches[i].velocity.size();
    } else {
      tp += v->patches[i].pressure.size();
      tv += v->patches[i].velocity.size();
    }
  }
  out[0] = np;
  out[1] = tp;
  out[2] = tv;
  out[3] = v->f ? static_cast<long long>(v->f->a_factor_bytes) : 0;
  out[4] = v->f ? static_cast<long long>(v->f->aux_bytes) : 0;
  out[5] = v->f ? static_cast<long long>(v->f->dense_inverse_bytes) : 0;
  out[6] = v->n;
  return OK;
}

int ref_vanka_patches(void* h, int* pptr, int* pidx, int* vptr, int* vidx, int* nx) {
  auto* v = static_cast<VankaH*>(h);
  const bool fac = v->f != nullptr;
  const int np = fac ? static_cast<int>(v->f->patches.size()) : static_cast<int>(v->patches.size());
  pptr[0] = vptr[0] = 0;
  for (int i = 0; i < np; ++i) {
    const auto& pres = fac ? v->f->patches[i].pressure : v->patches[i].pressure;
    const auto& vel = fac ? v->f->patches[i].velocity : v->patches[i].velocity;
    std::memcpy(pidx + pptr[i], pres.data(), sizeof(int) * pres.size());
    std::memcpy(vidx + vptr[i], vel.data(), sizeof(int) * vel.size());
    pptr[i + 1] = pptr[i] + static_cast<int>(pres.size());
    vptr[i + 1] = vptr[i] + static_cast<int>(vel.size());
    nx[i] = fac ? v->f->patches[i].nx : v->patches[i].nx;
  }
  return OK;
}

// Per-patch factor payload, concatenated in patch order, each DenseMatrix
// row-major as stored by the reference: u_hat (nv x np), b_hat (np x nv),
// s_inv (np x np); plus the PoU weights (length n).
int ref_vanka_factors(void* h, double* uhat, double* bhat, double* sinv, double* weights) {
  auto* v = static_cast<VankaH*>(h);
  size_t ou = 0, ob = 0, os = 0;
  for (const auto& p : v->f->patches) {
    std::memcpy(uhat + ou, p.u_hat.values.data(), sizeof(double) * p.u_hat.values.size());
    std::memcpy(bhat + ob, p.b_hat.values.data(), sizeof(double) * p.b_hat.values.size());
    std::memcpy(sinv + os, p.s_inv.values.data(), sizeof(double) * p.s_inv.values.size());
    ou += p.u_hat.values.size();
    ob += p.b_hat.values.size();
    os += p.s_inv.values.size();
  }
  std::memcpy(weights, v->f->weights.data(), sizeof(double) * v->f->weights.size());
  return OK;
}

// Packed LU factors (nx*nx then ny*ny per patch, row-major) and pivots.
int ref_vanka_lu(void* h, double* lu, int* piv) {
  auto* v = static_cast<VankaH*>(h);
  size_t o = 0, q = 0;
  for (const auto& p : v->f->patches) {
    for (const LUFactors* f : {&p.lu_x, &p.lu_y}) {
      std::memcpy(lu + o, f->lu.values.data(), sizeof(double) * f->lu.values.size());
      std::memcpy(piv + q, f->pivot.data(), sizeof(int) * f->pivot.size());
      o += f->lu.values.size();
      q += f->pivot.size();
    }
  }
  return OK;
}

int ref_apply_vanka(void* h, const double* r, double* delta) {
  auto* v = static_cast<VankaH*>(h);
  return guard([&] {
    std::vector<double> rv(r, r + v->n);
    auto d = apply_vanka(*v->f, rv);
    std::memcpy(delta, d.data(), sizeof(double) * d.size());
  });
}

int ref_vanka_relax(void* kh, void* h, double* x, const double* b, int mode, int sweeps,
                    double omega) {
  const auto& k = static_cast<MatH*>(kh)->m;
  auto* v = static_cast<VankaH*>(h);
  return guard([&] {
    std::vector<double> xv(x, x + k.nrows), bv(b, b + k.nrows);
    vanka_relax(k, *v->f, xv, bv, mode == 0 ? RelaxMode::KrylovWrapped : RelaxMode::Stationary,
                sweeps, omega);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
  });
}

// ------------------------------------------------------------------- krylov
// prec_kind: 0 identity, 1 vanka (prec = VankaH), 2 Jacobi (prec = MatH whose
// inverse diagonal is used), 3 DC preconditioner (prec = DcH, raw apply).
int ref_fgmres(void* ah, const double* b, double* x, int prec_kind, void* prec,
               const RefFgmresOpts* o, RefReport* rep, double* hist, int cap) {
  const auto& a = static_cast<MatH*>(ah)->m;
  return guard([&] {
    FgmresOptions opt;
    opt.tol = o->tol;
    opt.max_iters = o->max_iters;
    opt.restart = o->restart;
    opt.breakdown = o->breakdown;
    std::vector<double> bv(b, b + a.nrows), xv(x, x + a.nrows);
    LinearOperator p = identity_operator();
    std::vector<double> dinv;
    if (prec_kind == 1) {
      auto* v = static_cast<VankaH*>(prec);
      p = [v](const std::vector<double>& r, std::vector<double>& z) { z = apply_vanka(*v->f, r); };
    } else if (prec_kind == 2) {
      dinv = inv_diagonal(static_cast<MatH*>(prec)->m);
      p = [&dinv](const std::vector<double>& r, std::vector<double>& z) {
        z.resize(r.size());
        for (size_t i = 0; i < r.size(); ++i) z[i] = dinv[i] * r[i];
      };
    } else if (prec_kind == 3) {
      auto* d = static_cast<DcH*>(prec);
      p = [d](const std::vector<double>& r, std::vector<double>& z) { z = d->prec->apply(r); };
    }
    auto r = fgmres(matrix_operator(a), bv, xv, p, opt);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    report_out(r, rep, hist, cap);
  });
}

// ----------------------------------------------------------- preconditioner
static SolverConfig config_in(const RefConfig* c) {
  SolverConfig s;
  s.variant = static_cast<Variant>(c->variant);
  s.eta_u = c->eta_u;
  s.eta_p = c->eta_p;
  s.omega0 = c->omega0;
  s.nu1 = c->nu1;
  s.nu2 = c->nu2;
  s.gamma = c->gamma;
  s.restart = c->restart;
  s.tol = c->tol;
  s.max_iters = c->max_iters;
  s.enclosed_flow = c->enclosed_flow != 0;
  if (c->coarse_size > 0) s.amg.coarse_size = c->coarse_size;
  return s;
}

void* ref_dc_new(void* ch, const RefConfig* c) {
  const auto& cs = static_cast<CaseH*>(ch)->c;
  DcH* out = nullptr;
  int rc = guard([&] {
    auto* h = new DcH;
    h->cfg = config_in(c);
    h->prec = std::make_unique<DCPreconditioner>(cs.sys0, cs.sys1, cs.transfer, h->cfg);
    h->n_p1 = cs.sys1.n_p;
    out = h;
  });
  return rc == OK ? out : nullptr;
}

int ref_dc_set_parameters(void* h, double eta_u, double eta_p, double omega0) {
  auto* d = static_cast<DcH*>(h);
  return guard([&] {
    d->prec->set_parameters(eta_u, eta_p, omega0);
    d->cfg.eta_u = eta_u;
    d->cfg.eta_p = eta_p;
    d->cfg.omega0 = omega0;
  });
}

int ref_dc_nlevels(void* h) { return static_cast<DcH*>(h)->prec->low_order().hierarchy().num_levels(); }

// level l of the low-order hierarchy: out = [n_x, n_y, n_p, has_p]; K and P as
// new matrix handles (P null on the coarsest level).
int ref_dc_level(void* h, int l, int* out, void** k, void** p) {
  const auto& lev = static_cast<DcH*>(h)->prec->low_order().hierarchy().levels.at(l);
  out[0] = lev.n_x;
  out[1] = lev.n_y;
  out[2] = lev.n_p;
  const int nl = static_cast<DcH*>(h)->prec->low_order().hierarchy().num_levels();
  out[3] = l + 1 < nl ? 1 : 0;
  if (k) *k = new_mat(lev.k);
  if (p) *p = out[3] ? new_mat(lev.p) : nullptr;
  return OK;
}

void* ref_dc_k0(void* h) { return new_mat(static_cast<DcH*>(h)->prec->k0()); }

// Borrowed view of level l's Vanka factorization (valid while the DC lives).
void* ref_dc_level_vanka(void* h, int l) {
  auto* d = static_cast<DcH*>(h);
  const auto& fs = d->prec->low_order().factorizations();
  auto* v = new VankaH;
  v->f = &fs.at(l);
  v->n = static_cast<int>(v->f->weights.size());
  return v;
}

int ref_dc_apply(void* h, const double* r, double* z) {
  auto* d = static_cast<DcH*>(h);
  return guard([&] {
    const int n = d->prec->size();
    std::vector<double> rv(r, r + n);
    auto zv = d->prec->apply(rv);
    std::memcpy(z, zv.data(), sizeof(double) * n);
  });
}

int ref_dc_vcycle(void* h, const double* b, double* x, int nu1, int nu2) {
  auto* d = static_cast<DcH*>(h);
  return guard([&] {
    const auto& mono = d->prec->low_order();
    const int n = mono.hierarchy().levels.front().total();
    std::vector<double> bv(b, b + n);
    auto xv = mono.vcycle(bv, nu1, nu2, false, nullptr);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

int ref_dc_counters(void* h, long long* out) {
  auto* d = static_cast<DcH*>(h);
  out[0] = d->prec->fine_relax_units;
  out[1] = d->prec->level1_relax_units;
  return OK;
}

// Any preconditioner variant through the reference's own classes, as
// experiments.cpp:124-140 makes them (HOAMG, Uzawa on sys0; DC variants).
struct PrecH : H {
  SolverConfig cfg;
  std::unique_ptr<StokesPreconditioner> prec;
  SparseMatrix k0;
};

void* ref_prec_new(void* ch, const RefConfig* c) {
  const auto& cs = static_cast<CaseH*>(ch)->c;
  PrecH* out = nullptr;
  int rc = guard([&] {
    auto* h = new PrecH;
    h->cfg = config_in(c);
    if (h->cfg.variant == Variant::HOAMG)
      h->prec = std::make_unique<HoAmgPreconditioner>(cs.sys0, h->cfg);
    else if (h->cfg.variant == Variant::Uzawa)
      h->prec = std::make_unique<UzawaPreconditioner>(cs.sys0, h->cfg);
    else
      h->prec = std::make_unique<DCPreconditioner>(cs.sys0, cs.sys1, cs.transfer, h->cfg);
    h->k0 = assemble_saddle_matrix(cs.sys0);
    out = h;
  });
  return rc == OK ? out : nullptr;
}

int ref_prec_apply(void* h, const double* r, double* z) {
  auto* d = static_cast<PrecH*>(h);
  return guard([&] {
    const int n = d->prec->size();
    std::vector<double> rv(r, r + n);
    auto zv = d->prec->apply(rv);
    std::memcpy(z, zv.data(), sizeof(double) * n);
  });
}

int ref_prec_solve(void* h, const double* rhs, double* x, RefReport* rep, double* hist, int cap) {
  auto* d = static_cast<PrecH*>(h);
  return guard([&] {
    const int n = d->prec->size();
    std::vector<double> rv(rhs, rhs + n);
    auto res = solve_stokes(d->k0, rv, *d->prec, d->cfg);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    report_out(res.report, rep, hist, cap);
  });
}

int ref_solve_stokes(void* h, const double* rhs, double* x, RefReport* rep, double* hist,
                     int cap) {
  auto* d = static_cast<DcH*>(h);
  return guard([&] {
    const int n = d->prec->size();
    std::vector<double> rv(rhs, rhs + n);
    auto res = solve_stokes(d->prec->k0(), rv, *d->prec, d->cfg);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    report_out(res.report, rep, hist, cap);
  });
}

// std::sort's permutation under from_triplets' comparator (sparse.cpp:44-46)
// on the reference's own Triplet: keys = row << 32 | col, the value carries
// the original index. The device reproduces this (sag_sort_permutation).
int ref_sort_permutation(long long n, const unsigned long long* keys, int* perm) {
  return guard([&] {
    std::vector<Triplet> t(n);
    for (long long i = 0; i < n; ++i)
      t[i] = {static_cast<int>(keys[i] >> 32), static_cast<int>(keys[i] & 0xffffffffu),
              static_cast<double>(i)};
    std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    for (long long i = 0; i < n; ++i) perm[i] = static_cast<int>(t[i].value);
  });
}

// McIlroy's adversary ("A killer adversary for quicksort", 1999) against
// std::sort: keys that drive libstdc++'s introsort towards its depth limit
// (the heap-sort fallback); gas elements left at the end share one key.
int ref_antiqsort_keys(int n, unsigned long long* keys) {
  return guard([&] {
    std::vector<int> val(n, n), ptr(n);
    int nsolid = 0, candidate = 0;
    const int gas = n;
    for (int i = 0; i < n; ++i) ptr[i] = i;
    auto cmp = [&](int x, int y) {
      if (val[x] == gas && val[y] == gas) {
        if (x == candidate) val[x] = nsolid++;
        else val[y] = nsolid++;
      }
      if (val[x] == gas) candidate = x;
      else if (val[y] == gas) candidate = y;
      return val[x] < val[y];
    };
    std::sort(ptr.begin(), ptr.end(), cmp);
    for (int i = 0; i < n; ++i) keys[i] = static_cast<unsigned long long>(val[i]);
  });
}

}  // extern "C"
