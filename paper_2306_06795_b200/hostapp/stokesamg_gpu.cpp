// Drop-in adapter: reference C++ solver API on top of libsag's C-ABI, and the
// host-application entry points (sagh_*) the Python harness uses to obtain
// reference-built cases (build_case, assemble_saddle_matrix,
// build_monolithic_hierarchy -- the setup north_star keeps in the reference's
// host C++).
#include "stokesamg_gpu.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <utility>

#include "stokesamg/experiments.hpp"

namespace stokesamg::gpu {

void check(int s) {
  if (s == SAG_OK) return;
  const std::string msg = sag_last_error();
  switch (s) {
    case SAG_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case SAG_SINGULAR_MATRIX: throw SingularMatrix(msg);
    case SAG_SINGULAR_PATCH: throw SingularPatch(msg);
    case SAG_CONFIG_ERROR: throw ConfigError(msg);
    case SAG_SOLVER_STAGNATION: throw SolverStagnation(msg);
    case SAG_ZERO_DIAGONAL: throw ZeroDiagonal(msg);
    case SAG_UNSUPPORTED_DISCRETIZATION: throw UnsupportedDiscretization(msg);
    default: throw Error(msg);
  }
}

Device::Device(int ordinal) { check(sag_create(ordinal, &ctx_)); }
Device::~Device() { sag_destroy(ctx_); }

DeviceMatrix::DeviceMatrix(Device& dev, const SparseMatrix& m) : nrows_(m.nrows), ncols_(m.ncols) {
  check(sag_matrix_create(dev.handle(), m.nrows, m.ncols, m.nnz(), m.row_offsets.data(),
                          m.col_indices.data(), m.values.data(), &h_));
}
DeviceMatrix::~DeviceMatrix() { sag_matrix_destroy(h_); }

std::vector<double> spmv(Device& dev, const DeviceMatrix& m, const std::vector<double>& x) {
  if (static_cast<int>(x.size()) != m.ncols())
    throw DimensionMismatch("spmv: vector length does not match column count");
  std::vector<double> y(m.nrows());
  check(sag_spmv(dev.handle(), m.handle(), x.data(), y.data()));
  return y;
}

VankaFactorization::VankaFactorization(Device& dev, const DeviceMatrix& k, int n_x, int n_y,
                                       int n_p, bool sv_triples) {
  sag_patches* p = nullptr;
  check(sag_build_patches(dev.handle(), k.handle(), n_x, n_y, n_p, sv_triples ? 1 : 0, &p));
  const int rc = sag_factor_patches(dev.handle(), k.handle(), p, n_x + n_y, &f_);
  sag_patches_destroy(p);
  check(rc);
  long long s[7];
  check(sag_vanka_stats(f_, s));
  a_factor_bytes = s[0];
  aux_bytes = s[1];
  dense_inverse_bytes = s[2];
}
VankaFactorization::~VankaFactorization() { sag_vanka_destroy(f_); }

std::vector<double> apply_vanka(Device& dev, const VankaFactorization& f,
                                const std::vector<double>& r) {
  std::vector<double> d(r.size());
  check(sag_apply_vanka(dev.handle(), f.handle(), r.data(), d.data()));
  return d;
}

static sag_solver_config to_c(const SolverConfig& c) {
  sag_solver_config s;
  switch (c.variant) {
    case Variant::DCLO: s.variant = SAG_DC_LO; break;
    case Variant::DCHO: s.variant = SAG_DC_HO; break;
    case Variant::HOAMG: s.variant = SAG_HOAMG; break;
    case Variant::Uzawa: s.variant = SAG_UZAWA; break;
    default: s.variant = SAG_DC_ALL; break;
  }
  s.eta_u = c.eta_u;
  s.eta_p = c.eta_p;
  s.omega0 = c.omega0;
  s.nu1 = c.nu1;
  s.nu2 = c.nu2;
  s.gamma = c.gamma;
  s.restart = c.restart;
  s.tol = c.tol;
  s.max_iters = c.max_iters;
  s.enclosed_flow = c.enclosed_flow ? 1 : 0;
  s.allow_sv_hoamg = c.allow_sv_hoamg ? 1 : 0;
  return s;
}

DCPreconditioner::DCPreconditioner(Device& dev, const SaddleSystem& sys0, const SaddleSystem& sys1,
                                   TransferPair transfer, SolverConfig cfg)
    : dev_(dev), cfg_(std::move(cfg)) {
  if (cfg_.validate) cfg_.check();
  if (cfg_.variant != Variant::DCall && cfg_.variant != Variant::DCLO &&
      cfg_.variant != Variant::DCHO)
    throw ConfigError("gpu::DCPreconditioner: variant must be a DC variant");
  k0_ = assemble_saddle_matrix(sys0);
  n_p0_ = sys0.n_p;
  if (transfer.n_u0 != sys0.n_u() || transfer.n_p0 != n_p0_)
    throw DimensionMismatch("DCPreconditioner: transfer does not match the high-order system");
  h_ = build_monolithic_hierarchy(dev, sys1, cfg_.amg);  // device setup, bitwise the reference's
  const bool sv = sys0.disc == Discretization::SV;
  mats_.push_back(std::make_unique<DeviceMatrix>(dev, k0_));
  const sag_matrix* k0h = mats_.back()->handle();
  std::vector<sag_level_desc> lv(h_.num_levels());
  for (int l = 0; l < h_.num_levels(); ++l) {
    const auto& L = h_.levels[l];
    mats_.push_back(std::make_unique<DeviceMatrix>(dev, L.k));
    lv[l].k = mats_.back()->handle();
    lv[l].p = nullptr;
    if (l + 1 < h_.num_levels()) {
      mats_.push_back(std::make_unique<DeviceMatrix>(dev, L.p));
      lv[l].p = mats_.back()->handle();
    }
    lv[l].n_x = L.n_x;
    lv[l].n_y = L.n_y;
    lv[l].n_p = L.n_p;
  }
  const sag_solver_config c = to_c(cfg_);
  check(sag_dc_create(dev.handle(), k0h, sys0.n_x, sys0.n_y, sys0.n_p, sv ? 1 : 0,
                      h_.num_levels(), lv.data(), &c, &dc_));
  if (sv) {
    // SvPressureRestrict's own hierarchy (transfer.cpp:18-23), rebuilt by the
    // reference's build_scalar_hierarchy with the default AmgConfig
    ScalarHierarchy sh = build_scalar_hierarchy(dev, sys0.Mp_cg, AmgConfig{});
    mats_.push_back(std::make_unique<DeviceMatrix>(dev, transfer.p0_pressure));
    const sag_matrix* pdup = mats_.back()->handle();
    mats_.push_back(std::make_unique<DeviceMatrix>(dev, sys0.M_mix));
    const sag_matrix* mmix = mats_.back()->handle();
    std::vector<const sag_matrix*> A, P;
    for (const auto& m : sh.matrices) {
      mats_.push_back(std::make_unique<DeviceMatrix>(dev, m));
      A.push_back(mats_.back()->handle());
    }
    for (const auto& m : sh.prolongators) {
      mats_.push_back(std::make_unique<DeviceMatrix>(dev, m));
      P.push_back(mats_.back()->handle());
    }
    check(sag_dc_set_sv_transfer(dc_, pdup, mmix, static_cast<int>(A.size()), A.data(),
                                 P.data()));
  }
}

DCPreconditioner::~DCPreconditioner() { sag_dc_destroy(dc_); }

std::vector<double> DCPreconditioner::apply(const std::vector<double>& r) const {
  if (static_cast<int>(r.size()) != size())
    throw DimensionMismatch("DCPreconditioner::apply: size mismatch");
  std::vector<double> z(r.size());
  check(sag_dc_apply(dev_.handle(), dc_, r.data(), z.data()));
  long long cnt[2];
  check(sag_dc_counters(dc_, cnt));
  fine_relax_units = cnt[0];
  level1_relax_units = cnt[1];
  return z;
}

void DCPreconditioner::set_parameters(double eta_u, double eta_p, double omega0) {
  cfg_.eta_u = eta_u;
  cfg_.eta_p = eta_p;
  cfg_.omega0 = omega0;
  if (cfg_.validate) cfg_.check();
  check(sag_dc_set_parameters(dc_, eta_u, eta_p, omega0));
}

namespace {
SolveResult report_in(std::vector<double> x, const sag_krylov_report& rep,
                      const std::vector<double>& hist) {
  SolveResult res;
  res.x = std::move(x);
  res.report.converged = rep.converged != 0;
  res.report.iterations = rep.iterations;
  res.report.final_relative_residual = rep.final_relative_residual;
  res.report.residual_history.assign(
      hist.begin(), hist.begin() + std::min<size_t>(rep.history_len, hist.size()));
  return res;
}

SolveResult solve_dc(const SparseMatrix& k0, const std::vector<double>& rhs, Device& dev,
                     sag_dc* dc, int n, const SolverConfig& cfg) {
  if (cfg.validate) cfg.check();
  if (k0.nrows != n || static_cast<int>(rhs.size()) != n)
    throw DimensionMismatch("solve_stokes: size mismatch");
  std::vector<double> x(rhs.size(), 0.0);
  const sag_solver_config c = to_c(cfg);
  sag_krylov_report rep{};
  std::vector<double> hist(cfg.max_iters + 2);
  check(sag_solve_stokes(dev.handle(), dc, rhs.data(), x.data(), &c, &rep, hist.data(),
                         static_cast<int>(hist.size())));
  return report_in(std::move(x), rep, hist);
}

// a ScalarHierarchy uploaded level by level
struct ScalarUpload {
  std::vector<const sag_matrix*> a, p;
  sag_scalar_hierarchy desc{};
};
ScalarUpload upload_scalar(Device& dev, const ScalarHierarchy& h,
                           std::vector<std::unique_ptr<DeviceMatrix>>& keep) {
  ScalarUpload u;
  for (const auto& m : h.matrices) {
    keep.push_back(std::make_unique<DeviceMatrix>(dev, m));
    u.a.push_back(keep.back()->handle());
  }
  for (const auto& m : h.prolongators) {
    keep.push_back(std::make_unique<DeviceMatrix>(dev, m));
    u.p.push_back(keep.back()->handle());
  }
  u.desc.nlevels = static_cast<int>(u.a.size());
  u.desc.a = u.a.data();
  u.desc.p = u.p.empty() ? nullptr : u.p.data();
  return u;
}
}  // namespace

SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const DCPreconditioner& prec, const SolverConfig& cfg) {
  return solve_dc(k0, rhs, prec.device(), prec.handle(), prec.size(), cfg);
}

HoAmgPreconditioner::HoAmgPreconditioner(Device& dev, const SaddleSystem& sys0, SolverConfig cfg)
    : dev_(dev), cfg_(std::move(cfg)) {
  if (cfg_.validate) cfg_.check();
  const bool sv = sys0.disc == Discretization::SV;
  if (sv && !cfg_.allow_sv_hoamg)
    throw UnsupportedDiscretization(
        "HO-AMG on Scott-Vogelius is refused by default (known poorly convergent); set the "
        "override to force it");
  n_ = sys0.total_dofs();
  n_p_ = sys0.n_p;
  if (sv) {
    // the dg pressure space guides coarsening with its mass matrix
    // (preconditioner.cpp:163-168)
    SaddleSystem tmp = sys0;
    tmp.Ap = sys0.Mp;
    h_ = build_monolithic_hierarchy(dev, tmp, cfg_.amg);
  } else {
    h_ = build_monolithic_hierarchy(dev, sys0, cfg_.amg);
  }
  std::vector<sag_level_desc> lv(h_.num_levels());
  for (int l = 0; l < h_.num_levels(); ++l) {
    const auto& L = h_.levels[l];
    mats_.push_back(std::make_unique<DeviceMatrix>(dev, L.k));
    lv[l].k = mats_.back()->handle();
    lv[l].p = nullptr;
    if (l + 1 < h_.num_levels()) {
      mats_.push_back(std::make_unique<DeviceMatrix>(dev, L.p));
      lv[l].p = mats_.back()->handle();
    }
    lv[l].n_x = L.n_x;
    lv[l].n_y = L.n_y;
    lv[l].n_p = L.n_p;
  }
  sag_solver_config c = to_c(cfg_);
  c.variant = SAG_HOAMG;
  const auto& L0 = h_.levels.front();
  check(sag_dc_create(dev.handle(), lv[0].k, L0.n_x, L0.n_y, L0.n_p, sv ? 1 : 0, h_.num_levels(),
                      lv.data(), &c, &dc_));
}

HoAmgPreconditioner::~HoAmgPreconditioner() { sag_dc_destroy(dc_); }

std::vector<double> HoAmgPreconditioner::apply(const std::vector<double>& r) const {
  if (static_cast<int>(r.size()) != size())
    throw DimensionMismatch("HoAmgPreconditioner::apply: size mismatch");
  std::vector<double> z(r.size());
  check(sag_dc_apply(dev_.handle(), dc_, r.data(), z.data()));
  long long cnt[2];
  check(sag_dc_counters(dc_, cnt));
  fine_relax_units = cnt[0];
  return z;
}

SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const HoAmgPreconditioner& prec, const SolverConfig& cfg) {
  return solve_dc(k0, rhs, prec.device(), prec.handle(), prec.size(), cfg);
}

UzawaPreconditioner::UzawaPreconditioner(Device& dev, const SaddleSystem& sys, SolverConfig cfg)
    : dev_(dev), cfg_(std::move(cfg)) {
  if (cfg_.validate) cfg_.check();
  const int n_x = sys.n_x;
  n_u_ = sys.n_u();
  n_p_ = sys.n_p;
  ScalarHierarchy hx =
      build_scalar_hierarchy(dev, extract_block(sys.A, 0, n_x, 0, n_x), cfg_.amg);
  ScalarHierarchy hy =
      build_scalar_hierarchy(dev, extract_block(sys.A, n_x, n_u_, n_x, n_u_), cfg_.amg);
  mats_.push_back(std::make_unique<DeviceMatrix>(dev, sys.B));
  const sag_matrix* b = mats_.back()->handle();
  ScalarUpload ux = upload_scalar(dev, hx, mats_), uy = upload_scalar(dev, hy, mats_);
  const sag_solver_config c = to_c(cfg_);
  if (sys.disc == Discretization::SV) {
    check(sag_uzawa_create(dev.handle(), b, n_x, n_u_ - n_x, n_p_, &ux.desc, &uy.desc, nullptr,
                           sys.sv_element_areas.data(), &c, &u_));
  } else {
    ScalarHierarchy hp = build_scalar_hierarchy(dev, sys.Mp, cfg_.amg);
    ScalarUpload up = upload_scalar(dev, hp, mats_);
    check(sag_uzawa_create(dev.handle(), b, n_x, n_u_ - n_x, n_p_, &ux.desc, &uy.desc, &up.desc,
                           nullptr, &c, &u_));
  }
}

UzawaPreconditioner::~UzawaPreconditioner() { sag_uzawa_destroy(u_); }

std::vector<double> UzawaPreconditioner::apply(const std::vector<double>& r) const {
  if (static_cast<int>(r.size()) != size())
    throw DimensionMismatch("UzawaPreconditioner::apply: size mismatch");
  std::vector<double> z(r.size());
  check(sag_uzawa_apply(dev_.handle(), u_, r.data(), z.data()));
  return z;
}

SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const UzawaPreconditioner& prec, const SolverConfig& cfg) {
  if (cfg.validate) cfg.check();
  if (k0.nrows != prec.size() || static_cast<int>(rhs.size()) != prec.size())
    throw DimensionMismatch("solve_stokes: size mismatch");
  DeviceMatrix k(prec.device(), k0);
  std::vector<double> x(rhs.size(), 0.0);
  const sag_solver_config c = to_c(cfg);
  sag_krylov_report rep{};
  std::vector<double> hist(cfg.max_iters + 2);
  check(sag_solve_stokes_uzawa(prec.device().handle(), k.handle(), prec.handle(), rhs.data(),
                               x.data(), &c, &rep, hist.data(), static_cast<int>(hist.size())));
  return report_in(std::move(x), rep, hist);
}

// ---- hierarchy setup with device products (amg.cpp:300-360) ---------------
namespace {
struct DevM {  // owned device matrix handle
  sag_matrix* h = nullptr;
  DevM() = default;
  explicit DevM(sag_matrix* m) : h(m) {}
  DevM(Device& dev, const SparseMatrix& m) {
    check(sag_matrix_create(dev.handle(), m.nrows, m.ncols, m.nnz(), m.row_offsets.data(),
                            m.col_indices.data(), m.values.data(), &h));
  }
  DevM(const DevM&) = delete;
  DevM& operator=(const DevM&) = delete;
  DevM(DevM&& o) noexcept : h(o.h) { o.h = nullptr; }
  DevM& operator=(DevM&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~DevM() {
    if (h) sag_matrix_destroy(h);
  }
};

SparseMatrix to_host(Device& dev, const DevM& m) {
  int nr = 0, nc = 0;
  long long nnz = 0;
  check(sag_matrix_shape(m.h, &nr, &nc, &nnz));
  SparseMatrix out(nr, nc);
  out.col_indices.resize(nnz);
  out.values.resize(nnz);
  check(sag_matrix_export(dev.handle(), m.h, out.row_offsets.data(), out.col_indices.data(),
                          out.values.data()));
  return out;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

// One coarsening step of a scalar block (amg.cpp:219-236, :317-329), the
// setup timers and the strength-graph counters shared by both builders.
struct DeviceSetup {
  Device& dev;
  const AmgConfig& cfg;
  double t_host = 0.0, t_dev = 0.0;
  int soc_dev = 0, soc_host = 0;
  template <class F>
  void host(F&& f) {
    const auto t0 = std::chrono::steady_clock::now();
    f();
    t_host += seconds_since(t0);
  }
  template <class F>
  void device(F&& f) {
    const auto t0 = std::chrono::steady_clock::now();
    f();
    t_dev += seconds_since(t0);
  }
  struct Step {
    SparseMatrix p;
    DevM dp;
    std::vector<double> coarse_null;
  };
  // SoC -> aggregate -> tentative -> smoothed prolongator; stagnated when
  // the aggregation keeps more than 90% of the nodes (amg.cpp:216-219)
  Step coarsen(const SparseMatrix& a, const DevM& da, const std::vector<double>& nullvec,
               bool& stagnated) {
    Step s;
    Aggregation agg;
    double omega = 0.0;
    bool stop = false;
    // rho(D^-1 A): evolution_soc (amg.cpp:47-49) and smooth_prolongator
    // (amg.cpp:227-229) estimate it identically -- once here: the start
    // vector is the reference's mt19937 stream (host), the iterations'
    // products on the device, their sequential norms on the host
    double rho = 0.0;
    std::vector<double> dinv, x0;
    host([&] {
      dinv = inv_diagonal(a);
      std::mt19937 rng(1234);  // power_rho_estimate's default seed (sparse.hpp:70-71)
      std::uniform_real_distribution<double> dist(-1.0, 1.0);
      x0.resize(a.nrows);
      for (double& v : x0) v = dist(rng);
      const double nx = norm2(x0);
      if (nx == 0.0 || a.nrows == 0) x0.clear();
      for (double& v : x0) v /= nx;
    });
    device([&] {
      if (!x0.empty()) check(sag_power_rho(dev.handle(), da.h, dinv.data(), x0.data(), 10, &rho));
    });
    StrengthGraph g;
    bool soc_on_device = false;
    if (cfg.use_evolution_soc) {
      device([&] {
        sag_matrix* gh = nullptr;
        if (sag_evolution_soc(dev.handle(), da.h, 4.0 / (3.0 * rho), cfg.theta, cfg.soc_k,
                              &gh) == SAG_OK) {
          DevM gm(gh);
          const SparseMatrix gc = to_host(dev, gm);
          g.n = gc.nrows;
          g.offsets = gc.row_offsets;
          g.neighbors = gc.col_indices;
          g.weights = gc.values;
          soc_on_device = true;
          ++soc_dev;
        }
      });
    }
    host([&] {
      if (!soc_on_device) {  // symmetric measure, or a support too large for the device table
        g = cfg.use_evolution_soc ? evolution_soc(a, cfg.theta, cfg.soc_k)
                                  : symmetric_soc(a, cfg.sym_theta);
        ++soc_host;
      }
      agg = aggregate(g);
      if (agg.num_aggregates > 0.9 * a.nrows) {
        stop = true;
        return;
      }
      omega = cfg.omega_frac / rho;
    });
    if (stop) {
      stagnated = true;
      return s;
    }
    device([&] {
      // tentative_prolongator_with_nullvec (amg.cpp:184-205) on the device
      DevM dt;
      s.coarse_null.resize(agg.num_aggregates);
      gpu::check(sag_tentative_prolongator(dev.handle(), static_cast<int>(agg.node_to_agg.size()),
                                           agg.num_aggregates, agg.node_to_agg.data(),
                                           nullvec.data(), &dt.h, s.coarse_null.data()));
      check(sag_smooth_prolongator(dev.handle(), da.h, dt.h, omega, &s.dp.h));
      s.p = to_host(dev, s.dp);
    });
    return s;
  }
  // P^T K P on the device; the result kept on the device and copied out
  DevM galerkin(const DevM& p, const DevM& k, SparseMatrix& out) {
    DevM r;
    device([&] {
      check(sag_galerkin(dev.handle(), p.h, k.h, &r.h));
      out = to_host(dev, r);
    });
    return r;
  }
  void report(double* times) const {
    if (!times) return;
    times[0] = t_host;
    times[1] = t_dev;
    times[2] = soc_dev;
    times[3] = soc_host;
  }
};

MonolithicHierarchy build_monolithic_hierarchy(Device& dev, const SaddleSystem& sys,
                                               const AmgConfig& cfg, double* times) {
  if (sys.Ap.nrows != sys.n_p)
    throw DimensionMismatch(
        "build_monolithic_hierarchy: pressure auxiliary operator does not match the pressure "
        "space");
  DeviceSetup S{dev, cfg};
  MonolithicHierarchy h;
  MonolithicLevel l0;
  SparseMatrix ax, ay, ap;
  S.host([&] {
    l0.n_x = sys.n_x;
    l0.n_y = sys.n_y;
    l0.n_p = sys.n_p;
    ax = extract_block(sys.A, 0, sys.n_x, 0, sys.n_x);
    ay = extract_block(sys.A, sys.n_x, sys.n_x + sys.n_y, sys.n_x, sys.n_x + sys.n_y);
    ap = sys.Ap;
  });
  DevM kcur, dax, day, dap;
  S.device([&] {
    // assemble_saddle_matrix (fem.cpp:290-306) on the device
    DevM da(dev, sys.A), db(dev, sys.B);
    check(sag_saddle_matrix(dev.handle(), da.h, db.h, &kcur.h));
    l0.k = to_host(dev, kcur);
    dax = DevM(dev, ax);
    day = DevM(dev, ay);
    dap = DevM(dev, ap);
  });
  h.levels.push_back(std::move(l0));
  std::vector<double> null_x(ax.nrows, 1.0), null_y(ay.nrows, 1.0), null_p(ap.nrows, 1.0);
  using Step = DeviceSetup::Step;
  while (h.num_levels() < cfg.max_levels) {
    MonolithicLevel& cur = h.levels.back();
    if (cur.total() <= cfg.coarse_size) break;
    bool stagnated = false;
    Step sx = S.coarsen(ax, dax, null_x, stagnated);
    Step sy = stagnated ? Step{} : S.coarsen(ay, day, null_y, stagnated);
    Step sp = stagnated ? Step{} : S.coarsen(ap, dap, null_p, stagnated);
    if (stagnated) {
      h.truncated = true;
      break;
    }
    S.host([&] { cur.p = block_diag({&sx.p, &sy.p, &sp.p}); });
    MonolithicLevel next;
    DevM dP;
    S.device([&] { dP = DevM(dev, cur.p); });
    kcur = S.galerkin(dP, kcur, next.k);
    dax = S.galerkin(sx.dp, dax, ax);
    day = S.galerkin(sy.dp, day, ay);
    dap = S.galerkin(sp.dp, dap, ap);
    next.n_x = sx.p.ncols;
    next.n_y = sy.p.ncols;
    next.n_p = sp.p.ncols;
    null_x = std::move(sx.coarse_null);
    null_y = std::move(sy.coarse_null);
    null_p = std::move(sp.coarse_null);
    h.levels.push_back(std::move(next));
  }
  S.report(times);
  return h;
}

ScalarHierarchy build_scalar_hierarchy(Device& dev, const SparseMatrix& a, const AmgConfig& cfg,
                                       double* times) {
  DeviceSetup S{dev, cfg};
  ScalarHierarchy h;
  h.matrices.push_back(a);
  std::vector<double> nullvec(a.nrows, 1.0);
  DevM dcur;
  S.device([&] { dcur = DevM(dev, a); });
  while (h.levels() < cfg.max_levels) {
    const SparseMatrix& cur = h.matrices.back();
    if (cur.nrows <= cfg.coarse_size) break;
    bool stagnated = false;
    DeviceSetup::Step st = S.coarsen(cur, dcur, nullvec, stagnated);
    if (stagnated) {
      h.truncated = true;
      break;
    }
    SparseMatrix coarse;
    dcur = S.galerkin(st.dp, dcur, coarse);
    h.prolongators.push_back(std::move(st.p));
    h.matrices.push_back(std::move(coarse));
    nullvec = std::move(st.coarse_null);
  }
  S.host([&] {
    for (size_t l = 0; l + 1 < h.matrices.size(); ++l)
      h.d_inv.push_back(inv_diagonal(h.matrices[l]));
    h.coarse_lu = dense_lu_factor(to_dense(h.matrices.back()));
  });
  S.report(times);
  return h;
}

// ---- multi-GPU: the partitioned solve -----------------------
Communicator::NcclId Communicator::nccl_unique_id() {
  NcclId id{};
  check(sag_nccl_unique_id(id.data()));
  return id;
}

Communicator::Communicator(Device& dev, int nranks, int rank, const NcclId& id)
    : size_(nranks), rank_(rank) {
  check(sag_comm_create_nccl(dev.handle(), nranks, rank, id.data(), &comm_));
}

Communicator::Communicator(int nranks, int rank, const sag_comm_ops& ops)
    : size_(nranks), rank_(rank) {
  check(sag_comm_create_host(nranks, rank, &ops, &comm_));
}

Communicator::~Communicator() { sag_comm_destroy(comm_); }

namespace {
sag_csr csr_view(const SparseMatrix& m) {
  return sag_csr{m.nrows, m.ncols, m.row_offsets.data(), m.col_indices.data(), m.values.data()};
}
}  // namespace

DistDCPreconditioner::DistDCPreconditioner(Device& dev, Communicator& comm,
                                           const SaddleSystem& sys0, const SaddleSystem& sys1,
                                           TransferPair transfer, SolverConfig cfg)
    : dev_(dev), comm_(comm), cfg_(std::move(cfg)) {
  if (cfg_.validate) cfg_.check();
  if (sys0.disc == Discretization::SV)
    throw UnsupportedDiscretization("gpu::DistDCPreconditioner: Taylor-Hood systems only");
  if (transfer.n_u0 != sys0.n_u() || transfer.n_p0 != sys0.n_p)
    throw DimensionMismatch("DCPreconditioner: transfer does not match the high-order system");
  k0_ = assemble_saddle_matrix(dev, sys0);
  h_ = build_monolithic_hierarchy(dev, sys1, cfg_.amg);
  const int nl = h_.num_levels();
  std::vector<sag_csr> lv(nl), pv(std::max(nl - 1, 1));
  std::vector<int> nxyz(3 * nl);
  for (int l = 0; l < nl; ++l) {
    lv[l] = csr_view(h_.levels[l].k);
    if (l + 1 < nl) pv[l] = csr_view(h_.levels[l].p);
    nxyz[3 * l] = h_.levels[l].n_x;
    nxyz[3 * l + 1] = h_.levels[l].n_y;
    nxyz[3 * l + 2] = h_.levels[l].n_p;
  }
  const sag_csr k = csr_view(k0_);
  const sag_solver_config c = to_c(cfg_);
  check(sag_dist_create(dev.handle(), comm.handle(), &k, sys0.n_x, sys0.n_y, sys0.n_p, nl,
                        lv.data(), pv.data(), nxyz.data(), &c, &d_));
  long long info[7];
  check(sag_dist_info(d_, info));
  l2g_.resize(info[0]);
  owned_.resize(info[0]);
  check(sag_dist_local_dofs(d_, l2g_.data(), owned_.data()));
}

DistDCPreconditioner::~DistDCPreconditioner() { sag_dist_destroy(d_); }

SolveResult DistDCPreconditioner::solve(const std::vector<double>& rhs) const {
  if ((int)rhs.size() != k0_.nrows) throw DimensionMismatch("solve_stokes: rhs length");
  const size_t nl = l2g_.size();
  std::vector<double> b(nl), x(nl);
  for (size_t i = 0; i < nl; ++i) b[i] = rhs[l2g_[i]];
  sag_krylov_report rep{};
  std::vector<double> hist(cfg_.max_iters + 2);
  check(sag_dist_solve_stokes(dev_.handle(), d_, b.data(), x.data(), &rep, hist.data(),
                              (int)hist.size()));
  // the global solution: owned entries, summed over the ranks (one all-reduce)
  std::vector<double> xg(rhs.size(), 0.0);
  for (size_t i = 0; i < nl; ++i)
    if (owned_[i]) xg[l2g_[i]] = x[i];
  if (comm_.size() > 1) {
    sag_ctx* ctx = dev_.handle();
    void* dbuf = nullptr;
    check(sag_alloc(ctx, 8 * xg.size(), &dbuf));
    check(sag_memcpy(ctx, dbuf, xg.data(), 8 * xg.size()));
    const int st = sag_comm_allreduce(ctx, comm_.handle(), static_cast<double*>(dbuf),
                                      (long long)xg.size());
    if (st == SAG_OK) check(sag_memcpy(ctx, xg.data(), dbuf, 8 * xg.size()));
    sag_free(ctx, dbuf);
    check(st);
  }
  SolveResult out;
  out.x = std::move(xg);
  out.report.converged = rep.converged != 0;
  out.report.iterations = rep.iterations;
  out.report.final_relative_residual = rep.final_relative_residual;
  out.report.residual_history.assign(hist.begin(),
                                     hist.begin() + std::min<int>(rep.history_len, hist.size()));
  return out;
}

// ---- FEM assembly on the device --------------------------
// The host keeps the mesh, the user's callbacks (Dirichlet values, body force,
// Neumann data) and the boundary bookkeeping; the element loops, every
// from_triplets and the Dirichlet elimination run in libsag (sag_fem.cu),
// bitwise the reference's.
namespace {

// tri_quadrature (fem.cpp:21-36) and line_quadrature (:41-50)
struct QuadPt {
  std::array<double, 3> l;
  double w;
};
const std::array<QuadPt, 6>& quad6() {
  static const double a1 = 0.445948490915965, w1 = 0.223381589678011;
  static const double a2 = 0.091576213509771, w2 = 0.109951743655322;
  static const std::array<QuadPt, 6> q = {{{{a1, a1, 1 - 2 * a1}, w1},
                                           {{a1, 1 - 2 * a1, a1}, w1},
                                           {{1 - 2 * a1, a1, a1}, w1},
                                           {{a2, a2, 1 - 2 * a2}, w2},
                                           {{a2, 1 - 2 * a2, a2}, w2},
                                           {{1 - 2 * a2, a2, a2}, w2}}};
  return q;
}
struct LinePt {
  double s, w;
};
const std::array<LinePt, 3>& quad_line() {
  static const double c = std::sqrt(3.0 / 5.0);
  static const std::array<LinePt, 3> q = {
      {{0.5 * (1 - c), 5.0 / 18.0}, {0.5, 8.0 / 18.0}, {0.5 * (1 + c), 5.0 / 18.0}}};
  return q;
}

// the mesh as plain arrays for the C-ABI
struct MeshView {
  std::vector<double> v;
  std::vector<int> t, te;
  sag_mesh2d m{};
  explicit MeshView(const SimplicialMesh2D& mesh, bool edges) {
    v.resize(2 * mesh.vertices.size());
    for (size_t i = 0; i < mesh.vertices.size(); ++i) {
      v[2 * i] = mesh.vertices[i][0];
      v[2 * i + 1] = mesh.vertices[i][1];
    }
    t.resize(3 * mesh.triangles.size());
    for (size_t i = 0; i < mesh.triangles.size(); ++i)
      for (int k = 0; k < 3; ++k) t[3 * i + k] = mesh.triangles[i][k];
    if (edges) {
      te.resize(3 * mesh.tri_edges.size());
      for (size_t i = 0; i < mesh.tri_edges.size(); ++i)
        for (int k = 0; k < 3; ++k) te[3 * i + k] = mesh.tri_edges[i][k];
    }
    m.num_vertices = mesh.num_vertices();
    m.num_triangles = mesh.num_triangles();
    m.num_edges = mesh.num_edges();
    m.vertices = v.data();
    m.triangles = t.data();
    m.tri_edges = edges ? te.data() : nullptr;
  }
};

// The body force at every quadrature point (point_at, fem.cpp:73-76), the
// user's callback evaluated here on the host; empty when it vanishes
// everywhere (the element loop then adds nothing, fem.cpp:382).
std::vector<double> force_at_quadrature(const SimplicialMesh2D& m, const ProblemData& prob) {
  std::vector<double> f(12 * (size_t)m.num_triangles());
  bool any = false;
  for (int t = 0; t < m.num_triangles(); ++t) {
    const auto& c0 = m.vertices[m.triangles[t][0]];
    const auto& c1 = m.vertices[m.triangles[t][1]];
    const auto& c2 = m.vertices[m.triangles[t][2]];
    for (int q = 0; q < 6; ++q) {
      const auto& l = quad6()[q].l;
      const double x = l[0] * c0[0] + l[1] * c1[0] + l[2] * c2[0];
      const double y = l[0] * c0[1] + l[1] * c1[1] + l[2] * c2[1];
      const auto v = prob.force(x, y);
      f[12 * (size_t)t + 2 * q] = v[0];
      f[12 * (size_t)t + 2 * q + 1] = v[1];
      any = any || v[0] != 0.0 || v[1] != 0.0;
    }
  }
  if (!any) f.clear();
  return f;
}

// p2_dirichlet_values / p1_dirichlet_values (fem.cpp:120-146)
std::map<int, std::array<double, 2>> dirichlet_values(const SimplicialMesh2D& m,
                                                      const ProblemData& prob, bool p2) {
  std::map<int, std::array<double, 2>> vals;
  for (const auto& be : m.boundary_edges) {
    if (be.tag == BoundaryTag::Neumann) continue;
    const auto& pa = m.vertices[be.a];
    const auto& pb = m.vertices[be.b];
    vals[be.a] = prob.dirichlet(be.tag, pa[0], pa[1]);
    vals[be.b] = prob.dirichlet(be.tag, pb[0], pb[1]);
    if (p2)
      vals[m.num_vertices() + m.edge_index(be.a, be.b)] =
          prob.dirichlet(be.tag, 0.5 * (pa[0] + pb[0]), 0.5 * (pa[1] + pb[1]));
  }
  return vals;
}

// check_compatibility (fem.cpp:148-196): the enclosed-flow net boundary flux.
// A boundary edge has exactly one incident triangle, found here through an
// edge map instead of a scan over all triangles (same triangle, same flux).
void compatibility(const SimplicialMesh2D& m, const ProblemData& prob) {
  if (!prob.check_compatibility) return;
  for (const auto& be : m.boundary_edges)
    if (be.tag == BoundaryTag::Neumann) return;
  std::map<std::array<int, 2>, int> opposite;  // boundary edge -> third vertex
  for (const auto& be : m.boundary_edges)
    opposite[{std::min(be.a, be.b), std::max(be.a, be.b)}] = -1;
  for (int t = 0; t < m.num_triangles(); ++t)
    for (int k = 0; k < 3; ++k) {
      const int a = m.triangles[t][(k + 1) % 3], b = m.triangles[t][(k + 2) % 3];
      auto it = opposite.find({std::min(a, b), std::max(a, b)});
      if (it != opposite.end() && it->second < 0) it->second = m.triangles[t][k];
    }
  double flux = 0.0, scale = 0.0;
  for (const auto& be : m.boundary_edges) {
    const auto& pa = m.vertices[be.a];
    const auto& pb = m.vertices[be.b];
    const double tx = pb[0] - pa[0], ty = pb[1] - pa[1];
    const double len = std::hypot(tx, ty);
    scale += len;
    std::array<double, 2> n{ty / len, -tx / len};
    const int other = opposite[{std::min(be.a, be.b), std::max(be.a, be.b)}];
    if (other >= 0) {
      const auto& po = m.vertices[other];
      const double dx = po[0] - 0.5 * (pa[0] + pb[0]);
      const double dy = po[1] - 0.5 * (pa[1] + pb[1]);
      if (n[0] * dx + n[1] * dy > 0) {
        n[0] = -n[0];
        n[1] = -n[1];
      }
    }
    for (const auto& q : quad_line()) {
      const auto g = prob.dirichlet(be.tag, pa[0] + q.s * tx, pa[1] + q.s * ty);
      flux += q.w * len * (g[0] * n[0] + g[1] * n[1]);
    }
  }
  if (std::abs(flux) > 1e-10 * std::max(scale, 1.0))
    throw CompatibilityError("enclosed flow with nonzero net boundary flux");
}

// Neumann edge loads (fem.cpp:391-414 P2, :610-627 ISO), after the element loop
void neumann_loads(const SimplicialMesh2D& m, const ProblemData& prob, bool p2,
                   std::vector<double>& fx, std::vector<double>& fy) {
  if (!prob.neumann) return;
  for (const auto& be : m.boundary_edges) {
    if (be.tag != BoundaryTag::Neumann) continue;
    const auto& pa = m.vertices[be.a];
    const auto& pb = m.vertices[be.b];
    const double len = std::hypot(pb[0] - pa[0], pb[1] - pa[1]);
    const int mid = p2 ? m.num_vertices() + m.edge_index(be.a, be.b) : -1;
    for (const auto& q : quad_line()) {
      const double x = pa[0] + q.s * (pb[0] - pa[0]);
      const double y = pa[1] + q.s * (pb[1] - pa[1]);
      const auto gn = (*prob.neumann)(x, y);
      const double w = q.w * len;
      if (p2) {
        const double na = (1 - q.s) * (1 - 2 * q.s);
        const double nb = q.s * (2 * q.s - 1);
        const double nm = 4 * q.s * (1 - q.s);
        fx[be.a] += w * na * gn[0];
        fy[be.a] += w * na * gn[1];
        fx[be.b] += w * nb * gn[0];
        fy[be.b] += w * nb * gn[1];
        fx[mid] += w * nm * gn[0];
        fy[mid] += w * nm * gn[1];
      } else {
        fx[be.a] += w * (1 - q.s) * gn[0];
        fy[be.a] += w * (1 - q.s) * gn[1];
        fx[be.b] += w * q.s * gn[0];
        fy[be.b] += w * q.s * gn[1];
      }
    }
  }
}

// make_reduction (fem.cpp:198-205) + the device elimination (reduce_scalar,
// reduce_divergence) + the system's remaining fields (fem.cpp:420-449)
void finish_system(Device& dev, SaddleSystem& sys, const DevM& a_full, const DevM& b_full,
                   int n_s, const std::map<int, std::array<double, 2>>& vals,
                   const std::vector<double>& fx, const std::vector<double>& fy) {
  std::vector<int> o2n(n_s, -1), kept;
  std::vector<double> gx(n_s, 0.0), gy(n_s, 0.0);
  for (int i = 0; i < n_s; ++i) {
    auto it = vals.find(i);
    if (it == vals.end()) {
      o2n[i] = static_cast<int>(kept.size());
      kept.push_back(i);
    } else {
      gx[i] = it->second[0];
      gy[i] = it->second[1];
    }
  }
  const int ns_red = static_cast<int>(kept.size());
  int nbr = 0, nbc = 0;
  long long nbz = 0;
  check(sag_matrix_shape(b_full.h, &nbr, &nbc, &nbz));
  std::vector<double> lift_x(ns_red), lift_y(ns_red), rhs_p(nbr);
  DevM a_red, b_red;
  check(sag_reduce_dirichlet(dev.handle(), a_full.h, b_full.h, n_s, o2n.data(), gx.data(),
                             gy.data(), &a_red.h, &b_red.h, lift_x.data(), lift_y.data(),
                             rhs_p.data()));
  sys.n_x = sys.n_y = ns_red;
  sys.n_p = nbr;
  SparseMatrix ar = to_host(dev, a_red);
  sys.B = to_host(dev, b_red);
  sys.A = block_diag({&ar, &ar});
  sys.rhs.assign(sys.total_dofs(), 0.0);
  for (int i = 0; i < ns_red; ++i) {
    sys.rhs[i] = fx[kept[i]] - lift_x[i];
    sys.rhs[ns_red + i] = fy[kept[i]] - lift_y[i];
  }
  for (int i = 0; i < nbr; ++i) sys.rhs[2 * ns_red + i] = rhs_p[i];
  for (const auto& [dof, g] : vals) {
    sys.bc.constrained.push_back(dof);
    sys.bc.values_x.push_back(g[0]);
    sys.bc.values_y.push_back(g[1]);
  }
  sys.velocity_coords.clear();
  sys.velocity_coords.reserve(ns_red);
}

std::vector<std::array<double, 2>> p2_coords(const SimplicialMesh2D& m) {  // fem.cpp:110-118
  std::vector<std::array<double, 2>> c = m.vertices;
  c.reserve(m.num_vertices() + m.num_edges());
  for (const auto& e : m.edges)
    c.push_back({0.5 * (m.vertices[e[0]][0] + m.vertices[e[1]][0]),
                 0.5 * (m.vertices[e[0]][1] + m.vertices[e[1]][1])});
  return c;
}

void p1_operators(Device& dev, const SimplicialMesh2D& m, SparseMatrix* ap, SparseMatrix* mp) {
  MeshView mv(m, false);
  DevM s, ms;
  check(sag_assemble_p1(dev.handle(), &mv.m, ap ? &s.h : nullptr, mp ? &ms.h : nullptr));
  if (ap) *ap = to_host(dev, s);
  if (mp) *mp = to_host(dev, ms);
}

SaddleSystem assemble_p2(Device& dev, const SimplicialMesh2D& m, const ProblemData& prob,
                         bool sv) {
  const int nv = m.num_vertices(), nt = m.num_triangles();
  const int n_s = nv + m.num_edges();
  MeshView mv(m, true);
  const std::vector<double> fq = force_at_quadrature(m, prob);
  std::vector<double> fx(n_s), fy(n_s), areas(sv ? nt : 0);
  DevM a_full, b_full, mp, mix;
  check(sag_assemble_p2(dev.handle(), &mv.m, sv ? 1 : 0, fq.empty() ? nullptr : fq.data(),
                        &a_full.h, &b_full.h, fx.data(), fy.data(), sv ? &mp.h : nullptr,
                        sv ? &mix.h : nullptr, sv ? areas.data() : nullptr));
  neumann_loads(m, prob, true, fx, fy);
  const auto vals = dirichlet_values(m, prob, true);
  SaddleSystem sys;
  sys.disc = sv ? Discretization::SV : Discretization::TH;
  finish_system(dev, sys, a_full, b_full, n_s, vals, fx, fy);
  const auto coords = p2_coords(m);
  for (int i = 0; i < n_s; ++i)
    if (!vals.count(i)) sys.velocity_coords.push_back(coords[i]);
  if (sv) {
    p1_operators(dev, m, &sys.Ap, &sys.Mp_cg);
    sys.Mp = to_host(dev, mp);
    sys.M_mix = to_host(dev, mix);
    sys.sv_element_areas = std::move(areas);
    sys.pressure_coords.reserve(3 * (size_t)nt);
    sys.sv_pressure_vertices.reserve(nt);
    for (int t = 0; t < nt; ++t) {
      sys.sv_pressure_vertices.push_back(m.triangles[t]);
      for (int k = 0; k < 3; ++k) sys.pressure_coords.push_back(m.vertices[m.triangles[t][k]]);
    }
  } else {
    p1_operators(dev, m, &sys.Ap, &sys.Mp);
    sys.pressure_coords = m.vertices;
  }
  return sys;
}

}  // namespace

SaddleSystem assemble_taylor_hood(Device& dev, const SimplicialMesh2D& m,
                                  const ProblemData& prob) {
  if (m.boundary_edges.empty()) throw UntaggedBoundary("assemble_taylor_hood: no boundary tags");
  compatibility(m, prob);
  return assemble_p2(dev, m, prob, false);
}

SaddleSystem assemble_scott_vogelius(Device& dev, const SimplicialMesh2D& m,
                                     const ProblemData& prob, bool force_unrefined) {
  if (!m.barycentric && !force_unrefined)
    throw StabilityWarning("assemble_scott_vogelius: mesh is not barycentrically refined");
  if (m.boundary_edges.empty()) throw UntaggedBoundary("assemble_scott_vogelius: no boundary tags");
  compatibility(m, prob);
  return assemble_p2(dev, m, prob, true);
}

SaddleSystem assemble_iso(Device& dev, const SimplicialMesh2D& m, const SimplicialMesh2D& m_fine,
                          const RefinementMap& map, const ProblemData& prob) {
  if (m_fine.num_vertices() != m.num_vertices() + m.num_edges() ||
      m_fine.num_triangles() != 4 * m.num_triangles())
    throw DimensionMismatch("assemble_iso: fine mesh is not a quadrisection of the coarse mesh");
  compatibility(m, prob);
  const int nvf = m_fine.num_vertices(), nvc = m.num_vertices();
  MeshView mv(m_fine, false);
  const std::vector<double> fq = force_at_quadrature(m_fine, prob);
  std::vector<double> fx(nvf), fy(nvf);
  DevM a_full, b_fine;
  check(sag_assemble_iso(dev.handle(), &mv.m, fq.empty() ? nullptr : fq.data(), &a_full.h,
                         &b_fine.h, fx.data(), fy.data()));
  neumann_loads(m_fine, prob, false, fx, fy);
  // p1_interpolation (fem.cpp:337-352): one or two entries per fine vertex,
  // already in CSR order; b_coarse_p = transpose(E) b_fine on the device
  if (static_cast<int>(map.vertex_origin.size()) != nvf)
    throw DimensionMismatch("p1_interpolation: refinement map does not match fine mesh");
  SparseMatrix e(nvf, nvc);
  for (int i = 0; i < nvf; ++i) {
    const auto& org = map.vertex_origin[i];
    if (const auto* cv = std::get_if<CoarseVertex>(&org)) {
      e.col_indices.push_back(cv->index);
      e.values.push_back(1.0);
    } else if (const auto* em = std::get_if<EdgeMidpoint>(&org)) {
      const int lo = std::min(em->a, em->b), hi = std::max(em->a, em->b);
      e.col_indices.push_back(lo);
      e.values.push_back(0.5);
      e.col_indices.push_back(hi);
      e.values.push_back(0.5);
    } else {
      throw DimensionMismatch("p1_interpolation: barycentric lineage not supported here");
    }
    e.row_offsets[i + 1] = static_cast<int>(e.col_indices.size());
  }
  DevM de(dev, e), et, bcp;
  check(sag_transpose(dev.handle(), de.h, &et.h));
  check(sag_spgemm(dev.handle(), et.h, b_fine.h, &bcp.h));
  const auto vals = dirichlet_values(m_fine, prob, false);
  SaddleSystem sys;
  sys.disc = Discretization::ISO;
  finish_system(dev, sys, a_full, bcp, nvf, vals, fx, fy);
  sys.n_p = nvc;
  for (int i = 0; i < nvf; ++i)
    if (!vals.count(i)) sys.velocity_coords.push_back(m_fine.vertices[i]);
  p1_operators(dev, m, &sys.Ap, &sys.Mp);
  sys.pressure_coords = m.vertices;
  return sys;
}

SparseMatrix assemble_saddle_matrix(Device& dev, const SaddleSystem& sys) {
  DevM a(dev, sys.A), b(dev, sys.B), k;
  check(sag_saddle_matrix(dev.handle(), a.h, b.h, &k.h));
  return to_host(dev, k);
}

AssembledCase build_case(Device& dev, const SimplicialMesh2D& base, const ProblemData& prob,
                         Discretization disc, bool enclosed) {
  AssembledCase c;
  c.enclosed = enclosed;
  if (disc == Discretization::SV) {
    auto [mb, bmap] = barycentric_refine(base);
    c.mesh = std::move(mb);
    c.sys0 = assemble_scott_vogelius(dev, c.mesh, prob);
    auto [mf, qmap] = quadrisect(c.mesh);
    c.sys1 = assemble_iso(dev, c.mesh, mf, qmap, prob);
    c.transfer = build_sv_transfer(c.sys0, c.sys1);
  } else {
    c.mesh = base;
    c.sys0 = assemble_taylor_hood(dev, c.mesh, prob);
    auto [mf, qmap] = quadrisect(c.mesh);
    c.sys1 = assemble_iso(dev, c.mesh, mf, qmap, prob);
    c.transfer = build_th_transfer(c.sys0, c.sys1);
  }
  return c;
}

}  // namespace stokesamg::gpu

// ======================================================================
// Host-application entry points for the Python harness (bench.py): the
// reference's setup produces the inputs of the GPU path.
// ======================================================================
using namespace stokesamg;

namespace {
thread_local std::string g_err;

struct HostCase {
  AssembledCase c;
  ProblemData prob;  // the case's problem data (device assembly input)
  SparseMatrix k0;
  AmgConfig amg;
  MonolithicHierarchy h;
  ScalarHierarchy sh;  // SV only
  // HO-AMG / Uzawa inputs (sagh_case_build_extra)
  MonolithicHierarchy ho;
  ScalarHierarchy ux, uy, ump;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

const SparseMatrix* pick(const HostCase& hc, int which) {
  if (which == 0) return &hc.k0;
  if (which >= 1 && which < 1000) {
    const int l = (which - 1) / 2;
    if (l >= hc.h.num_levels()) return nullptr;
    if ((which - 1) % 2 == 0) return &hc.h.levels[l].k;
    return l + 1 < hc.h.num_levels() ? &hc.h.levels[l].p : nullptr;
  }
  if (which == 1000) return &hc.c.transfer.p0_pressure;
  if (which == 1001) return &hc.c.sys0.M_mix;
  if (which >= 2000 && which < 3000) {  // HO-AMG hierarchy: 2000 + 2l K, 2001 + 2l P
    const int l = (which - 2000) / 2;
    if (l >= hc.ho.num_levels()) return nullptr;
    if ((which - 2000) % 2 == 0) return &hc.ho.levels[l].k;
    return l + 1 < hc.ho.num_levels() ? &hc.ho.levels[l].p : nullptr;
  }
  if (which == 3000) return &hc.c.sys0.B;
  if (which > 3000 && which < 4000) {  // Uzawa: 3100/3200/3300 + 2s A_s, + 2s + 1 P_s
    const int f = (which - 3000) / 100, k = (which - 3000) % 100, s = k / 2;
    const ScalarHierarchy* sh = f == 1 ? &hc.ux : f == 2 ? &hc.uy : f == 3 ? &hc.ump : nullptr;
    if (!sh) return nullptr;
    if (k % 2 == 0) return s < sh->levels() ? &sh->matrices[s] : nullptr;
    return s + 1 < sh->levels() ? &sh->prolongators[s] : nullptr;
  }
  const int s = (which - 1002) / 2;
  if ((which - 1002) % 2 == 0) return s < hc.sh.levels() ? &hc.sh.matrices[s] : nullptr;
  return s + 1 < hc.sh.levels() ? &hc.sh.prolongators[s] : nullptr;
}

// problem_data_for (experiments.cpp:56-84): the problem data build_case uses
ProblemData problem_for(const std::string& problem) {
  if (problem == "bfs") return bfs_problem();
  if (problem == "channel") return channel_problem();
  if (problem == "manufactured") return manufactured_unit_square().problem;
  if (problem == "cavity") {
    ProblemData p = zero_problem();
    p.dirichlet = [](BoundaryTag, double, double y) {
      return std::array<double, 2>{y > 1 - 1e-12 ? 1.0 : 0.0, 0.0};
    };
    p.check_compatibility = false;
    return p;
  }
  if (problem == "forced") {
    ProblemData p = zero_problem();
    p.force = [](double x, double y) {
      return std::array<double, 2>{std::sin(3.0 * y) + 1.0, std::cos(2.0 * x)};
    };
    return p;
  }
  throw ConfigError("experiment spec: unknown problem: " + problem);
}

// f = (sin(k1 x), cos(k2 y)) body force, all-Dirichlet zero (BASELINE config 4)
ProblemData forced_problem(double k1, double k2) {
  ProblemData prob = zero_problem();
  prob.force = [k1, k2](double x, double y) {
    return std::array<double, 2>{std::sin(k1 * x), std::cos(k2 * y)};
  };
  prob.check_compatibility = false;
  return prob;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

bool same(const SparseMatrix& a, const SparseMatrix& b) {
  return a.nrows == b.nrows && a.ncols == b.ncols && a.row_offsets == b.row_offsets &&
         a.col_indices == b.col_indices &&
         a.values.size() == b.values.size() &&
         (a.values.empty() ||
          std::memcmp(a.values.data(), b.values.data(), 8 * a.values.size()) == 0);
}
bool same(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 8 * a.size()) == 0);
}
// every field of two saddle systems, bitwise; bit i set = field i differs
int system_diff(const SaddleSystem& a, const SaddleSystem& b) {
  int d = 0;
  if (!same(a.A, b.A)) d |= 1;
  if (!same(a.B, b.B)) d |= 2;
  if (!same(a.Ap, b.Ap)) d |= 4;
  if (!same(a.Mp, b.Mp)) d |= 8;
  if (!same(a.rhs, b.rhs)) d |= 16;
  if (a.n_x != b.n_x || a.n_y != b.n_y || a.n_p != b.n_p || a.disc != b.disc) d |= 32;
  if (a.velocity_coords != b.velocity_coords || a.pressure_coords != b.pressure_coords) d |= 64;
  if (a.bc.constrained != b.bc.constrained || !same(a.bc.values_x, b.bc.values_x) ||
      !same(a.bc.values_y, b.bc.values_y))
    d |= 128;
  if (!same(a.Mp_cg, b.Mp_cg) || !same(a.M_mix, b.M_mix) ||
      !same(a.sv_element_areas, b.sv_element_areas) ||
      a.sv_pressure_vertices != b.sv_pressure_vertices)
    d |= 256;
  return d;
}

AssembledCase mesh_case(const char* path, double k1, double k2) {
  ProblemData prob = forced_problem(k1, k2);
  AssembledCase c;
  c.enclosed = true;
  c.mesh = read_mesh(path);
  for (auto& be : c.mesh.boundary_edges) be.tag = BoundaryTag::DirichletZero;
  c.sys0 = assemble_taylor_hood(c.mesh, prob);
  auto [mf, qmap] = quadrisect(c.mesh);
  c.sys1 = assemble_iso(c.mesh, mf, qmap, prob);
  c.transfer = build_th_transfer(c.sys0, c.sys1);
  return c;
}
}  // namespace

extern "C" {

const char* sagh_last_error() { return g_err.c_str(); }
int sagh_case_solve_variant(void* h, int device, int variant, int nu, int restart, double tol,
                            int max_iters, double eta_u, double eta_p, double omega0, double* x,
                            int* rep, double* res);

// problem/sv/mesh_kind/n as ExperimentSpec (experiments.hpp:24-38); mesh_kind
// "file" reads mesh_path; "file_forced" builds BASELINE config 4 from
// mesh_path with force wavenumbers (k1, k2). coarse_size <= 0 keeps the
// reference default (amg.hpp:58).
void* sagh_case_build(const char* problem, int sv, const char* mesh_kind, int n,
                      const char* mesh_path, int coarse_size, double k1, double k2) {
  HostCase* out = nullptr;
  guarded([&] {
    auto hc = std::make_unique<HostCase>();
    if (std::string(mesh_kind) == "file_forced") {
      hc->c = mesh_case(mesh_path, k1, k2);
      hc->prob = forced_problem(k1, k2);
    } else {
      hc->prob = problem_for(problem);
      ExperimentSpec s;
      s.problem = problem;
      s.disc = sv ? Discretization::SV : Discretization::TH;
      s.mesh.kind = mesh_kind;
      s.mesh.n = n;
      if (mesh_path) s.mesh.path = mesh_path;
      hc->c = build_case(s, 0);
    }
    AmgConfig amg;
    if (coarse_size > 0) amg.coarse_size = coarse_size;
    hc->amg = amg;
    hc->k0 = assemble_saddle_matrix(hc->c.sys0);
    hc->h = build_monolithic_hierarchy(hc->c.sys1, amg);
    if (hc->c.sys0.disc == Discretization::SV)
      hc->sh = build_scalar_hierarchy(hc->c.sys0.Mp_cg, AmgConfig{});
    out = hc.release();
  });
  return out;
}

void sagh_case_free(void* h) { delete static_cast<HostCase*>(h); }

// The case's systems assembled again on the device (gpu::assemble_*, from the
// same high-order mesh and problem data) and compared with the reference's
// bitwise. out = [sys0 diff bits, sys1 diff bits, K0 equal, device
// assembly s (sys0 + quadrisect + sys1 + K0), reference assembly s (the same
// calls, only when time_reference), sys0 s, sys1 s, K0 s]
int sagh_case_assembly_gpu(void* h, int device, int time_reference, double* out) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    gpu::Device dev(device);
    const bool sv = hc.c.sys0.disc == Discretization::SV;
    auto t0 = std::chrono::steady_clock::now();
    SaddleSystem s0 = sv ? gpu::assemble_scott_vogelius(dev, hc.c.mesh, hc.prob)
                         : gpu::assemble_taylor_hood(dev, hc.c.mesh, hc.prob);
    const double t_s0 = seconds_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    auto [mf, qmap] = quadrisect(hc.c.mesh);
    SaddleSystem s1 = gpu::assemble_iso(dev, hc.c.mesh, mf, qmap, hc.prob);
    const double t_s1 = seconds_since(t1);
    auto t2 = std::chrono::steady_clock::now();
    SparseMatrix k0 = gpu::assemble_saddle_matrix(dev, s0);
    const double t_k0 = seconds_since(t2);
    const double t_dev = seconds_since(t0);
    double t_ref = -1.0;
    if (time_reference) {
      auto r0 = std::chrono::steady_clock::now();
      SaddleSystem a = sv ? assemble_scott_vogelius(hc.c.mesh, hc.prob)
                          : assemble_taylor_hood(hc.c.mesh, hc.prob);
      auto [mf2, qmap2] = quadrisect(hc.c.mesh);
      SaddleSystem b = assemble_iso(hc.c.mesh, mf2, qmap2, hc.prob);
      SparseMatrix k = assemble_saddle_matrix(a);
      t_ref = seconds_since(r0);
    }
    out[0] = system_diff(s0, hc.c.sys0);
    out[1] = system_diff(s1, hc.c.sys1);
    out[2] = same(k0, hc.k0) ? 1.0 : 0.0;
    out[3] = t_dev;
    out[4] = t_ref;
    out[5] = t_s0;
    out[6] = t_s1;
    out[7] = t_k0;
  });
}

// gpu::DistDCPreconditioner at one rank (NCCL communicator of size 1): the C++
// multi-GPU drop-in end to end. rep = [converged, iterations]
int sagh_case_solve_dist(void* h, int device, double* x, int* rep, double* res) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    gpu::Device dev(device);
    gpu::Communicator comm(dev, 1, 0, gpu::Communicator::NcclId{});
    SolverConfig cfg;
    cfg.variant = Variant::DCall;
    cfg.nu1 = cfg.nu2 = 1;
    cfg.restart = 30;
    cfg.tol = 1e-8;
    cfg.max_iters = 500;
    cfg.enclosed_flow = hc.c.enclosed;
    gpu::DistDCPreconditioner prec(dev, comm, hc.c.sys0, hc.c.sys1, hc.c.transfer, cfg);
    const SolveResult r = prec.solve(hc.c.sys0.rhs);
    std::copy(r.x.begin(), r.x.end(), x);
    rep[0] = r.report.converged ? 1 : 0;
    rep[1] = r.report.iterations;
    *res = r.report.final_relative_residual;
  });
}

// std::sort's permutation of n keys on the device (sag_sort_permutation)
int sagh_sort_permutation(int device, long long n, const unsigned long long* keys, int* perm,
                          int* heap_ranges) {
  return guarded([&] {
    gpu::Device dev(device);
    gpu::check(sag_sort_permutation(dev.handle(), n, keys, perm, heap_ranges));
  });
}

// build_scalar_hierarchy by the reference and on the device for the case's
// scalar operators -- A_x of the high-order system (Uzawa) and the pressure
// auxiliary operator (TH: Mp; SV: the continuous mass matrix of the pressure
// projection) -- compared bitwise: out = [equal (1/0), operators compared,
// levels of the last, strength graphs on the device]
int sagh_case_scalar_hierarchy_gpu(void* h, int device, double* out) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    const SaddleSystem& s0 = hc.c.sys0;
    std::vector<SparseMatrix> ops;
    ops.push_back(extract_block(s0.A, 0, s0.n_x, 0, s0.n_x));
    ops.push_back(s0.disc == Discretization::SV ? s0.Mp_cg : s0.Mp);
    gpu::Device dev(device);
    auto same = [](const SparseMatrix& a, const SparseMatrix& b) {
      return a.nrows == b.nrows && a.ncols == b.ncols && a.row_offsets == b.row_offsets &&
             a.col_indices == b.col_indices && a.values.size() == b.values.size() &&
             std::memcmp(a.values.data(), b.values.data(), sizeof(double) * a.values.size()) == 0;
    };
    bool eq = true;
    int levels = 0;
    double soc = 0.0;
    for (const auto& a : ops) {
      const ScalarHierarchy ref = build_scalar_hierarchy(a, AmgConfig{});
      double parts[4] = {0, 0, 0, 0};
      const ScalarHierarchy got = gpu::build_scalar_hierarchy(dev, a, AmgConfig{}, parts);
      soc += parts[2];
      eq = eq && ref.levels() == got.levels() && ref.truncated == got.truncated &&
           ref.coarse_lu.lu.values == got.coarse_lu.lu.values && ref.coarse_lu.pivot == got.coarse_lu.pivot;
      for (int l = 0; eq && l < ref.levels(); ++l) {
        eq = same(ref.matrices[l], got.matrices[l]) &&
             (l + 1 == ref.levels() || same(ref.prolongators[l], got.prolongators[l]));
        if (eq && l + 1 < ref.levels()) eq = ref.d_inv[l] == got.d_inv[l];
      }
      levels = got.levels();
    }
    out[0] = eq ? 1.0 : 0.0;
    out[1] = (double)ops.size();
    out[2] = levels;
    out[3] = soc;
  });
}

// The case's low-order hierarchy built again by the reference (host) and by
// gpu::build_monolithic_hierarchy (device products), compared bitwise:
// out = [reference s, device-assisted total s, its host part s, its device
// part s, levels equal (1/0), levels, strength graphs built on the device,
// on the host]
int sagh_case_hierarchy_gpu(void* h, int device, double* out) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    auto t0 = std::chrono::steady_clock::now();
    const MonolithicHierarchy ref = build_monolithic_hierarchy(hc.c.sys1, hc.amg);
    const double t_ref = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    gpu::Device dev(device);
    double parts[4] = {0.0, 0.0, 0.0, 0.0};
    t0 = std::chrono::steady_clock::now();
    const MonolithicHierarchy got = gpu::build_monolithic_hierarchy(dev, hc.c.sys1, hc.amg, parts);
    const double t_gpu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    auto same = [](const SparseMatrix& a, const SparseMatrix& b) {
      return a.nrows == b.nrows && a.ncols == b.ncols && a.row_offsets == b.row_offsets &&
             a.col_indices == b.col_indices &&
             std::memcmp(a.values.data(), b.values.data(), sizeof(double) * a.values.size()) == 0 &&
             a.values.size() == b.values.size();
    };
    bool eq = ref.num_levels() == got.num_levels() && ref.truncated == got.truncated;
    for (int l = 0; eq && l < ref.num_levels(); ++l) {
      const auto &a = ref.levels[l], &b = got.levels[l];
      eq = a.n_x == b.n_x && a.n_y == b.n_y && a.n_p == b.n_p && same(a.k, b.k) &&
           (l + 1 == ref.num_levels() || same(a.p, b.p));
    }
    out[0] = t_ref;
    out[1] = t_gpu;
    out[2] = parts[0];
    out[3] = parts[1];
    out[4] = eq ? 1.0 : 0.0;
    out[5] = got.num_levels();
    out[6] = parts[2];
    out[7] = parts[3];
  });
}

// The reference's setup for the other preconditioners of this case, with the
// default AmgConfig: what = 1 -> HoAmgPreconditioner's hierarchy
// (preconditioner.cpp:155-172), what = 2 -> UzawaPreconditioner's scalar
// hierarchies (preconditioner.cpp:178-192).
int sagh_case_build_extra(void* h, int what) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    const SaddleSystem& s0 = hc.c.sys0;
    if (what == 1) {
      if (s0.disc == Discretization::SV) {
        SaddleSystem tmp = s0;
        tmp.Ap = s0.Mp;
        hc.ho = build_monolithic_hierarchy(tmp, AmgConfig{});
      } else {
        hc.ho = build_monolithic_hierarchy(s0, AmgConfig{});
      }
    } else if (what == 2) {
      hc.ux = build_scalar_hierarchy(extract_block(s0.A, 0, s0.n_x, 0, s0.n_x), AmgConfig{});
      hc.uy = build_scalar_hierarchy(extract_block(s0.A, s0.n_x, s0.n_u(), s0.n_x, s0.n_u()),
                                     AmgConfig{});
      if (s0.disc != Discretization::SV) hc.ump = build_scalar_hierarchy(s0.Mp, AmgConfig{});
    } else {
      throw ConfigError("sagh_case_build_extra: what must be 1 or 2");
    }
  });
}

// out = [HO levels, A_x levels, A_y levels, Mp levels, SV element count]
int sagh_case_info_extra(void* h, long long* out) {
  const auto& hc = *static_cast<HostCase*>(h);
  out[0] = hc.ho.num_levels();
  out[1] = hc.ux.levels();
  out[2] = hc.uy.levels();
  out[3] = hc.ump.levels();
  out[4] = static_cast<long long>(hc.c.sys0.sv_element_areas.size());
  return 0;
}

int sagh_case_ho_level(void* h, int l, int* nxyz) {
  const auto& lev = static_cast<HostCase*>(h)->ho.levels.at(l);
  nxyz[0] = lev.n_x;
  nxyz[1] = lev.n_y;
  nxyz[2] = lev.n_p;
  return 0;
}

int sagh_case_sv_areas(void* h, double* out) {
  const auto& a = static_cast<HostCase*>(h)->c.sys0.sv_element_areas;
  std::memcpy(out, a.data(), sizeof(double) * a.size());
  return 0;
}

// out = [n_x0, n_y0, n_p0, nlevels, enclosed, sv, scalar levels]
int sagh_case_info(void* h, long long* out) {
  const auto& hc = *static_cast<HostCase*>(h);
  out[0] = hc.c.sys0.n_x;
  out[1] = hc.c.sys0.n_y;
  out[2] = hc.c.sys0.n_p;
  out[3] = hc.h.num_levels();
  out[4] = hc.c.enclosed ? 1 : 0;
  out[5] = hc.c.sys0.disc == Discretization::SV ? 1 : 0;
  out[6] = hc.sh.levels();
  return 0;
}

int sagh_case_level(void* h, int l, int* nxyz) {
  const auto& lev = static_cast<HostCase*>(h)->h.levels.at(l);
  nxyz[0] = lev.n_x;
  nxyz[1] = lev.n_y;
  nxyz[2] = lev.n_p;
  return 0;
}

int sagh_case_matrix_shape(void* h, int which, int* nr, int* nc, long long* nnz) {
  const SparseMatrix* m = pick(*static_cast<HostCase*>(h), which);
  if (!m) {
    g_err = "sagh_case_matrix_shape: no such matrix";
    return 2;
  }
  *nr = m->nrows;
  *nc = m->ncols;
  *nnz = m->nnz();
  return 0;
}

int sagh_case_matrix_copy(void* h, int which, int* rp, int* ci, double* v) {
  const SparseMatrix* m = pick(*static_cast<HostCase*>(h), which);
  if (!m) {
    g_err = "sagh_case_matrix_copy: no such matrix";
    return 2;
  }
  std::memcpy(rp, m->row_offsets.data(), sizeof(int) * (m->nrows + 1));
  std::memcpy(ci, m->col_indices.data(), sizeof(int) * m->nnz());
  std::memcpy(v, m->values.data(), sizeof(double) * m->nnz());
  return 0;
}

int sagh_case_rhs(void* h, double* rhs) {
  const auto& r = static_cast<HostCase*>(h)->c.sys0.rhs;
  std::memcpy(rhs, r.data(), sizeof(double) * r.size());
  return 0;
}

// Drop-in end to end through the C++ adapter: gpu::DCPreconditioner +
// gpu::solve_stokes on this case. rep = [converged, iterations], res = final
// relative residual.
int sagh_case_solve(void* h, int device, int nu, int restart, double tol, int max_iters,
                    double eta_u, double eta_p, double omega0, double* x, int* rep, double* res) {
  return sagh_case_solve_variant(h, device, 0, nu, restart, tol, max_iters, eta_u, eta_p, omega0,
                                 x, rep, res);
}

// as sagh_case_solve with the preconditioner variant (preconditioner.hpp:14):
// 0-2 gpu::DCPreconditioner, 3 gpu::HoAmgPreconditioner, 4 gpu::UzawaPreconditioner
int sagh_case_solve_variant(void* h, int device, int variant, int nu, int restart, double tol,
                            int max_iters, double eta_u, double eta_p, double omega0, double* x,
                            int* rep, double* res) {
  return guarded([&] {
    auto& hc = *static_cast<HostCase*>(h);
    gpu::Device dev(device);
    SolverConfig cfg;
    cfg.variant = static_cast<Variant>(variant);
    cfg.nu1 = cfg.nu2 = nu;
    cfg.restart = restart;
    cfg.tol = tol;
    cfg.max_iters = max_iters;
    cfg.eta_u = eta_u;
    cfg.eta_p = eta_p;
    cfg.omega0 = omega0;
    cfg.enclosed_flow = hc.c.enclosed;
    SolveResult r;
    if (variant == 3) {
      gpu::HoAmgPreconditioner prec(dev, hc.c.sys0, cfg);
      r = gpu::solve_stokes(hc.k0, hc.c.sys0.rhs, prec, cfg);
    } else if (variant == 4) {
      gpu::UzawaPreconditioner prec(dev, hc.c.sys0, cfg);
      r = gpu::solve_stokes(hc.k0, hc.c.sys0.rhs, prec, cfg);
    } else {
      gpu::DCPreconditioner prec(dev, hc.c.sys0, hc.c.sys1, hc.c.transfer, cfg);
      r = gpu::solve_stokes(prec.k0(), hc.c.sys0.rhs, prec, cfg);
    }
    std::memcpy(x, r.x.data(), sizeof(double) * r.x.size());
    rep[0] = r.report.converged ? 1 : 0;
    rep[1] = r.report.iterations;
    *res = r.report.final_relative_residual;
  });
}

}  // extern "C"
