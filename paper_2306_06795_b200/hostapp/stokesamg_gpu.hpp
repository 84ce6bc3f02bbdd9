// stokesamg_gpu.hpp -- drop-in GPU solve phase for the reference C++ API
// (stokesamg, proj/core/include/stokesamg). A stokesamg user keeps building
// meshes, systems and hierarchies with the reference library and swaps
//
//     stokesamg::DCPreconditioner  ->  stokesamg::gpu::DCPreconditioner
//     stokesamg::solve_stokes      ->  stokesamg::gpu::solve_stokes
//
// Everything from factor_patches down (Vanka factorization and sweeps, SpMV,
// V-cycle transfers, FGMRES vector work) then runs in libsag's sm_100a
// kernels through the C-ABI in include/sag.h. Errors surface as the
// reference's own exception classes (errors.hpp:8-58).
#pragma once

#include <array>
#include <memory>
#include <vector>

#include "sag.h"
#include "stokesamg/errors.hpp"
#include "stokesamg/experiments.hpp"
#include "stokesamg/fem.hpp"
#include "stokesamg/mesh.hpp"
#include "stokesamg/preconditioner.hpp"
#include "stokesamg/transfer.hpp"

namespace stokesamg::gpu {

// Throws the stokesamg exception matching a libsag status code.
void check(int status);

// One CUDA device + stream (sag_ctx).
class Device {
 public:
  explicit Device(int ordinal = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  sag_ctx* handle() const { return ctx_; }

 private:
  sag_ctx* ctx_ = nullptr;
};

// Device copy of a stokesamg::SparseMatrix (sparse.hpp:11-28).
class DeviceMatrix {
 public:
  DeviceMatrix(Device& dev, const SparseMatrix& m);
  ~DeviceMatrix();
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;
  sag_matrix* handle() const { return h_; }
  int nrows() const { return nrows_; }
  int ncols() const { return ncols_; }

 private:
  sag_matrix* h_ = nullptr;
  int nrows_ = 0, ncols_ = 0;
};

// spmv (sparse.hpp:42) on the device.
std::vector<double> spmv(Device& dev, const DeviceMatrix& m, const std::vector<double>& x);

// factor_patches (vanka.hpp:42-43) on the device; apply_vanka (vanka.hpp:47).
class VankaFactorization {
 public:
  VankaFactorization(Device& dev, const DeviceMatrix& k, int n_x, int n_y, int n_p,
                     bool sv_triples = false);
  ~VankaFactorization();
  VankaFactorization(const VankaFactorization&) = delete;
  VankaFactorization& operator=(const VankaFactorization&) = delete;
  sag_vanka* handle() const { return f_; }
  size_t a_factor_bytes = 0, aux_bytes = 0, dense_inverse_bytes = 0;

 private:
  sag_vanka* f_ = nullptr;
};
std::vector<double> apply_vanka(Device& dev, const VankaFactorization& f,
                                const std::vector<double>& r);

// DCPreconditioner (preconditioner.hpp:77-100) with the same constructor
// arguments as the reference. The low-order hierarchy is built by the
// reference's build_monolithic_hierarchy on the host (setup, discrete and
// rounding-sensitive: SURVEY.md H1), then uploaded once.
class DCPreconditioner : public StokesPreconditioner {
 public:
  DCPreconditioner(Device& dev, const SaddleSystem& sys0, const SaddleSystem& sys1,
                   TransferPair transfer, SolverConfig cfg);
  ~DCPreconditioner() override;

  std::vector<double> apply(const std::vector<double>& r) const override;
  int size() const override { return k0_.nrows; }
  int pressure_size() const override { return n_p0_; }
  void set_parameters(double eta_u, double eta_p, double omega0);
  const SolverConfig& config() const { return cfg_; }
  const SparseMatrix& k0() const { return k0_; }
  const MonolithicHierarchy& hierarchy() const { return h_; }
  sag_dc* handle() const { return dc_; }
  Device& device() const { return dev_; }

 private:
  Device& dev_;
  SolverConfig cfg_;
  SparseMatrix k0_;
  int n_p0_ = 0;
  MonolithicHierarchy h_;
  std::vector<std::unique_ptr<DeviceMatrix>> mats_;
  sag_dc* dc_ = nullptr;
};

// HoAmgPreconditioner (preconditioner.hpp:103-118): the monolithic hierarchy
// built by the reference on the high-order system itself, one V-cycle per
// apply on the device (a sag_dc in HO-AMG mode).
class HoAmgPreconditioner : public StokesPreconditioner {
 public:
  HoAmgPreconditioner(Device& dev, const SaddleSystem& sys0, SolverConfig cfg);
  ~HoAmgPreconditioner() override;

  std::vector<double> apply(const std::vector<double>& r) const override;
  int size() const override { return n_; }
  int pressure_size() const override { return n_p_; }
  const MonolithicHierarchy& hierarchy() const { return h_; }
  sag_dc* handle() const { return dc_; }
  Device& device() const { return dev_; }

 private:
  Device& dev_;
  SolverConfig cfg_;
  int n_ = 0, n_p_ = 0;
  MonolithicHierarchy h_;
  std::vector<std::unique_ptr<DeviceMatrix>> mats_;
  sag_dc* dc_ = nullptr;
};

// UzawaPreconditioner (preconditioner.hpp:118-141): scalar hierarchies of
// A_x, A_y (and Mp for TH/ISO) built by the reference on the host, all
// V-cycles and the SV exact element mass inverse on the device.
class UzawaPreconditioner : public StokesPreconditioner {
 public:
  UzawaPreconditioner(Device& dev, const SaddleSystem& sys, SolverConfig cfg);
  ~UzawaPreconditioner() override;

  std::vector<double> apply(const std::vector<double>& r) const override;
  int size() const override { return n_u_ + n_p_; }
  int pressure_size() const override { return n_p_; }
  sag_uzawa* handle() const { return u_; }
  Device& device() const { return dev_; }

 private:
  Device& dev_;
  SolverConfig cfg_;
  int n_u_ = 0, n_p_ = 0;
  std::vector<std::unique_ptr<DeviceMatrix>> mats_;
  sag_uzawa* u_ = nullptr;
};

// solve_stokes (preconditioner.hpp:147-148): the outer FGMRES with all
// vectors resident on the device.
SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const DCPreconditioner& prec, const SolverConfig& cfg);
SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const HoAmgPreconditioner& prec, const SolverConfig& cfg);
SolveResult solve_stokes(const SparseMatrix& k0, const std::vector<double>& rhs,
                         const UzawaPreconditioner& prec, const SolverConfig& cfg);

// build_monolithic_hierarchy (amg.hpp:99; amg.cpp:300-360) with the setup's
// strength graphs (sag_evolution_soc) and sparse products on the device --
// smooth_prolongator's A T product, scaling and T - omega D^-1 A T
// (sag_smooth_prolongator) and every Galerkin product P^T K P (sag_galerkin)
// -- bitwise the reference's hierarchy. The greedy aggregation (sequential
// by definition, amg.cpp:113-160), tentative prolongators and the spectral
// radius estimates (mt19937 start vector) stay the reference's host code.
// times (may be null) = [host part s, device part s, strength graphs built
// on the device, on the host].
MonolithicHierarchy build_monolithic_hierarchy(Device& dev, const SaddleSystem& sys,
                                               const AmgConfig& cfg, double* times = nullptr);
// build_scalar_hierarchy (amg.hpp:74; amg.cpp:200-256) likewise: the scalar SA
// hierarchies of the Uzawa preconditioner and the SV mass projection.
ScalarHierarchy build_scalar_hierarchy(Device& dev, const SparseMatrix& a, const AmgConfig& cfg,
                                       double* times = nullptr);

// ---- multi-GPU: the partitioned solve ----------------------
// One process per GPU. The communicator carries the collectives: NCCL (rank
// 0 calls nccl_unique_id() and the caller broadcasts the id -- MPI_Bcast, a
// file, a socket) or the caller's own host-staged transport (sag_comm_ops).
class Communicator {
 public:
  using NcclId = std::array<unsigned char, 128>;
  static NcclId nccl_unique_id();
  Communicator(Device& dev, int nranks, int rank, const NcclId& id);
  Communicator(int nranks, int rank, const sag_comm_ops& ops);
  ~Communicator();
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  sag_comm* handle() const { return comm_; }
  int size() const { return size_; }
  int rank() const { return rank_; }

 private:
  sag_comm* comm_ = nullptr;
  int size_ = 1, rank_ = 0;
};

// DCPreconditioner + solve_stokes over a row/patch partition of K0 across the
// communicator's ranks (Taylor-Hood; DC-all / DC-LO / DC-HO, nu <= 1): the
// same constructor arguments as DCPreconditioner (every rank passes the
// whole systems), the hierarchy built as DCPreconditioner builds it, then
// libsag plans this rank's share (sag_dist_create). solve() takes the global
// rhs and returns the global solution (owned entries summed over the ranks
// by one all-reduce), the report identical on every rank.
class DistDCPreconditioner {
 public:
  DistDCPreconditioner(Device& dev, Communicator& comm, const SaddleSystem& sys0,
                       const SaddleSystem& sys1, TransferPair transfer, SolverConfig cfg);
  ~DistDCPreconditioner();
  DistDCPreconditioner(const DistDCPreconditioner&) = delete;
  DistDCPreconditioner& operator=(const DistDCPreconditioner&) = delete;
  SolveResult solve(const std::vector<double>& rhs) const;
  const std::vector<long long>& local_to_global() const { return l2g_; }
  const std::vector<unsigned char>& owned() const { return owned_; }
  const SparseMatrix& k0() const { return k0_; }
  sag_dist* handle() const { return d_; }

 private:
  Device& dev_;
  Communicator& comm_;
  SolverConfig cfg_;
  SparseMatrix k0_;
  MonolithicHierarchy h_;
  std::vector<long long> l2g_;
  std::vector<unsigned char> owned_;
  sag_dist* d_ = nullptr;
};

// FEM assembly with the element loops, every from_triplets (sparse.cpp:43-66)
// and the Dirichlet elimination (fem.cpp:207-266) on the device, bitwise the
// reference's systems (same signatures as fem.hpp:70-78 plus the device):
// the host keeps the mesh, the user's callbacks and the boundary bookkeeping.
SaddleSystem assemble_taylor_hood(Device& dev, const SimplicialMesh2D& m, const ProblemData& prob);
SaddleSystem assemble_scott_vogelius(Device& dev, const SimplicialMesh2D& m_bary,
                                     const ProblemData& prob, bool force_unrefined = false);
SaddleSystem assemble_iso(Device& dev, const SimplicialMesh2D& m, const SimplicialMesh2D& m_fine,
                          const RefinementMap& map, const ProblemData& prob);
// assemble_saddle_matrix (fem.hpp:70; fem.cpp:290-306) on the device.
SparseMatrix assemble_saddle_matrix(Device& dev, const SaddleSystem& sys);
// build_case (experiments.cpp:215-235) from the base mesh and problem data
// the caller built with the reference (base_mesh, problem_data_for), with
// the assembly above.
AssembledCase build_case(Device& dev, const SimplicialMesh2D& base, const ProblemData& prob,
                         Discretization disc, bool enclosed);

}  // namespace stokesamg::gpu
