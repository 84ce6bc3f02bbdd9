// libsag solver module: device-resident FGMRES (krylov.cpp:17-121),
// Krylov-wrapped / stationary Vanka relaxation (vanka.cpp:186-209), coarse
// dense solve, the monolithic V-cycle (preconditioner.cpp:40-88), the
// defect-correction preconditioner (preconditioner.cpp:90-153) and
// solve_stokes (preconditioner.cpp:229-259), plus their C-ABI.
//
// All vectors and all Krylov scalars (Hessenberg matrix, Givens rotations,
// residual estimates) stay on the device; a preconditioner application is a
// fixed sequence of kernel launches with no host synchronisation (captured
// once into a CUDA graph). The outer solve reads one small status record per
// Arnoldi step to decide convergence, as krylov.cpp:95-97 does.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <vector>

#include "dist_plan.hpp"
#include "internal.cuh"

namespace sag {

// ================================================================ Krylov ==

struct Krylov {
  int n = 0, m = 0, hist_cap = 0;
  DevBuf<double> V, Z, w, r;
  DevBuf<unsigned char> stbuf;
  KState* st = nullptr;
  void init(int n_, int m_, int hist_cap_) {
    n = n_;
    m = std::max(m_, 1);
    hist_cap = hist_cap_;
    V.alloc((size_t)(m + 1) * n);
    Z.alloc((size_t)m * n);
    w.alloc(n);
    r.alloc(n);
    stbuf.alloc(kstate_bytes(m, hist_cap));
    SAG_CUDA(cudaMemset(stbuf.p, 0, stbuf.n));
    st = reinterpret_cast<KState*>(stbuf.p);
  }
  double* v(int i) { return V.p + (size_t)i * n; }
  double* z(int i) { return Z.p + (size_t)i * n; }
  // device address of h[i*mm + j] for restart length mm (address arithmetic only)
  double* h(int mm, int i, int j) { return ks_h(st) + (size_t)i * mm + j; }
  const int* stop() { return &st->stop; }
  const int* breakdown() { return &st->breakdown; }
  const double* beta() { return &st->beta; }
  const double* wnorm() { return &st->wnorm; }
};

// Arnoldi step j with z_j already in K.z(j) (krylov.cpp:61-100):
//   w = A z_j fused with h_0j = (w, v_0)
//   MGS: w -= h_(i-1)j v_(i-1) fused with h_ij = (w, v_i), i = 1..j
//   w -= h_jj v_j fused with ||w||^2 -> Givens + residual estimate (finisher)
//   v_(j+1) = w / ||w|| unless breakdown
// last: final step of a fixed-length inner solve -- v_(j+1) is never used, so
// it is not formed and w keeps A z_j (reused by lin_resid for nu = 1).
// jac: also form z_(j+1) = jac .* v_(j+1) (Jacobi preconditioner) in the same pass.
static void arnoldi_step(Ctx& c, const Matrix& A, Krylov& K, int mm, int j, const int* gate,
                         bool last = false, const double* jac = nullptr) {
  const int n = K.n;
  {
    SpmvArgs a;
    a.dotv = K.v(0);
    a.gate = gate;
    a.fin.kind = FIN_H;
    a.fin.st = K.st;
    a.fin.i = 0;
    a.fin.j = j;
    launch_spmv(c, A, K.z(j), K.w.p, Epi::StoreDot, a);
  }
  for (int i = 1; i <= j; ++i) {
    Fin f;
    f.kind = FIN_H;
    f.st = K.st;
    f.i = i;
    f.j = j;
    launch_mgs(c, n, K.w.p, K.v(i - 1), K.h(mm, i - 1, j), K.v(i), f, gate);
  }
  Fin f;
  f.kind = FIN_ARNOLDI;
  f.st = K.st;
  f.j = j;
  launch_mgs_last(c, n, K.w.p, K.v(j), K.h(mm, j, j), f, gate, !last);
  if (last) return;
  if (jac)  // breakdown sets stop (FIN_ARNOLDI), so the stop gate covers it
    launch_div_mul(c, n, K.w.p, K.wnorm(), K.v(j + 1), jac, K.z(j + 1), gate);
  else
    launch_div(c, n, K.w.p, K.wnorm(), K.v(j + 1), gate, K.breakdown());
}

// vanka_relax, KrylovWrapped (vanka.cpp:199-208): x += FGMRES_nu(K, b - K x;
// M = apply_vanka, tol 0, restart = max_iters = nu, zero inner guess).
// x_zero: x is known to be zero, so r = b and x = corr (the reference's
// spmv of a zero vector is exactly zero).
static void relax_kw(Ctx& c, const Matrix& K, const Vanka& f, Krylov& kr, double* x,
                     const double* b, int nu, bool x_zero) {
  if (nu <= 0) {
    if (x_zero) launch_zero(c, K.nrows, x);
    return;
  }
  const int n = K.nrows;
  Fin fb;
  fb.kind = FIN_BETA;
  fb.st = kr.st;
  fb.i = 1 | 4;  // ref = ||r|| (b of the inner solve), full (re)init with m = nu
  fb.j = nu;
  fb.tol = 0.0;
  const double* r;
  if (x_zero) {
    launch_ssq(c, n, b, fb);
    r = b;
  } else {
    SpmvArgs a;
    a.b = b;
    a.fin = fb;
    launch_spmv(c, K, x, kr.r.p, Epi::ResidSsq, a);
    r = kr.r.p;
  }
  launch_div(c, n, r, kr.beta(), kr.v(0), kr.stop());
  for (int j = 0; j < nu; ++j) {
    vanka_apply(c, f, kr.v(j), kr.z(j), kr.stop());
    arnoldi_step(c, K, kr, nu, j, kr.stop(), j == nu - 1);
  }
  launch_update_bs(c, n, x, kr.Z.p, (size_t)n, kr.st, nu, x_zero);
}

// vanka_relax, Stationary (vanka.cpp:190-197): x += omega * vanka(b - K x).
static void relax_stationary(Ctx& c, const Matrix& K, const Vanka& f, double* rbuf, double* x,
                             const double* b, int sweeps, double omega, bool x_zero) {
  if (x_zero) launch_zero(c, K.nrows, x);
  for (int s = 0; s < sweeps; ++s) {
    const double* r = b;
    if (!(s == 0 && x_zero)) {
      SpmvArgs a;
      a.b = b;
      launch_spmv(c, K, x, rbuf, Epi::Resid, a);
      r = rbuf;
    }
    vanka_apply_stationary(c, f, r, x, omega);
  }
}

struct KHeader {
  double ref, tol, bd, beta, rnorm, wnorm;
  int m, stop, breakdown, jeff, iterations, hist_len, hist_cap, converged;
};
static_assert(sizeof(KHeader) == sizeof(KState), "KState layout");

static KHeader read_header(Ctx& c, KState* st) {
  KHeader h;
  SAG_CUDA(cudaMemcpyAsync(&h, st, sizeof(KHeader), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

struct FgmresOut {
  int converged = 0, iterations = 0;
  double final_rel = 0.0;
  std::vector<double> hist;
};

using DevOp = std::function<void(const double* in, double* out)>;

// fgmres (krylov.cpp:17-121) with A = K, right preconditioner `prec`, x in/out
// on device. One host synchronisation per Arnoldi step.
static FgmresOut fgmres_dev(Ctx& c, const Matrix& A, const double* b, double* x, const DevOp& prec,
                            double tol, int max_iters, int restart, double bd, Krylov& K) {
  const int n = A.nrows;
  // reduction tickets start from zero (a fresh solve never inherits a count)
  SAG_CUDA(cudaMemsetAsync(c.ticket.p, 0, sizeof(unsigned) * c.ticket.n, c.stream));
  SAG_REQUIRE(restart >= 1 && K.m >= restart && K.n == n, SAG_CONFIG_ERROR,
              "fgmres: workspace does not match restart / size");
  launch_kinit(c, K.st, restart, tol, bd, K.hist_cap, false);
  {
    Fin f;
    f.kind = FIN_REF;
    f.st = K.st;
    launch_ssq(c, n, b, f);  // bnorm, ref (krylov.cpp:23-24)
  }
  FgmresOut out;
  // initial residual (krylov.cpp:26-35): history[0]
  {
    SpmvArgs a;
    a.b = b;
    a.fin.kind = FIN_BETA;
    a.fin.st = K.st;
    a.fin.i = 2;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
  }
  KHeader hd = read_header(c, K.st);
  int iters = 0;
  bool converged = hd.stop != 0;
  while (!converged && iters < max_iters) {
    // (re)start from the true residual (krylov.cpp:43-53)
    SpmvArgs a;
    a.b = b;
    a.fin.kind = FIN_BETA;
    a.fin.st = K.st;
    a.fin.i = 0;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
    hd = read_header(c, K.st);
    if (hd.stop) {
      converged = true;
      break;
    }
    launch_div(c, n, K.r.p, K.beta(), K.v(0), K.stop());
    for (int j = 0; j < restart && iters < max_iters; ++j) {
      prec(K.v(j), K.z(j));
      arnoldi_step(c, A, K, restart, j, K.stop());
      hd = read_header(c, K.st);
      iters = hd.iterations;
      if (hd.stop) break;
    }
    launch_backsub(c, K.st);
    launch_update(c, n, x, K.Z.p, (size_t)n, K.st, false);
    hd = read_header(c, K.st);
    if (hd.converged) converged = true;
  }
  // final true residual (krylov.cpp:116-119)
  {
    SpmvArgs a;
    a.b = b;
    a.fin.kind = FIN_FINAL;
    a.fin.st = K.st;
    a.fin.out = c.scal.p;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
  }
  hd = read_header(c, K.st);
  SAG_CUDA(cudaMemcpyAsync(&out.final_rel, c.scal.p, sizeof(double), cudaMemcpyDeviceToHost,
                           c.stream));
  out.iterations = hd.iterations;
  out.converged = hd.converged;
  const int hl = std::min(hd.hist_len, K.hist_cap);
  out.hist.resize(hl);
  if (hl)
    SAG_CUDA(cudaMemcpyAsync(out.hist.data(), ks_h(K.st) + (size_t)(restart + 1) * restart +
                                                  restart + restart + (restart + 1) + restart,
                             sizeof(double) * hl, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// ============================================ device-side convergence loop ==
// fgmres_dev decides convergence on the host (one status read per Arnoldi
// step). Inside a CUDA graph capture the same algorithm runs with conditional
// nodes (CUDA 12.4+): a WHILE node over restart cycles (condition: not
// converged and iterations < max_iters, krylov.cpp:42) whose body holds the
// restart residual and `restart` IF nodes, one per Arnoldi step (condition:
// not stopped and iterations < max_iters, krylov.cpp:58); the conditions are
// set on the device from KState. Same operations, same order, no host sync.

__global__ void cond_set_kernel(cudaGraphConditionalHandle h, const KState* st, int mode,
                                int max_iters) {
  const unsigned v = mode == 0 ? (!st->converged && st->iterations < max_iters)
                               : (!st->stop && st->iterations < max_iters);
  cudaGraphSetConditional(h, v);
}

// Adds a conditional node at the current point of c.stream's capture: set(h)
// launches the kernel that sets its condition (before the node); body(h) is
// captured into the node's body graph on a body stream (c.stream switched).
template <class Set, class Body>
static void cond_node(Ctx& c, cudaGraphConditionalNodeType type, Set set, Body body) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  SAG_CUDA(cudaStreamGetCaptureInfo(c.stream, &cs, nullptr, &g, &deps, &nd));
  SAG_REQUIRE(cs == cudaStreamCaptureStatusActive, SAG_CUDA_ERROR,
              "conditional node outside a stream capture");
  cudaGraphConditionalHandle h;
  SAG_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  set(h);
  SAG_CUDA(cudaStreamGetCaptureInfo(c.stream, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  SAG_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
  SAG_CUDA(cudaStreamUpdateCaptureDependencies(c.stream, &node, 1,
                                               cudaStreamSetCaptureDependencies));
  const int d = c.body_depth;
  SAG_REQUIRE(d < 4, SAG_ERROR, "conditional nodes nested too deep");
  if (!c.body_streams[d])
    SAG_CUDA(cudaStreamCreateWithFlags(&c.body_streams[d], cudaStreamNonBlocking));
  cudaStream_t outer = c.stream, bs = c.body_streams[d];
  SAG_CUDA(cudaStreamBeginCaptureToGraph(bs, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
  c.stream = bs;
  c.body_depth = d + 1;
  cudaGraph_t done = nullptr;
  try {
    body(h);
  } catch (...) {
    c.stream = outer;
    c.body_depth = d;
    cudaStreamEndCapture(bs, &done);
    throw;
  }
  c.stream = outer;
  c.body_depth = d;
  SAG_CUDA(cudaStreamEndCapture(bs, &done));
}

static bool stream_capturing(Ctx& c);

// fgmres (krylov.cpp:17-121) as conditional graph nodes, for a caller that is
// capturing c.stream; the result (x, KState) is the one fgmres_dev computes.
static void fgmres_graph(Ctx& c, const Matrix& A, const double* b, double* x, const DevOp& prec,
                         double tol, int max_iters, int restart, double bd, Krylov& K,
                         double* final_out) {
  const int n = A.nrows;
  SAG_CUDA(cudaMemsetAsync(c.ticket.p, 0, sizeof(unsigned) * c.ticket.n, c.stream));
  launch_kinit(c, K.st, restart, tol, bd, K.hist_cap, false);
  {
    Fin f;
    f.kind = FIN_REF;
    f.st = K.st;
    launch_ssq(c, n, b, f);
  }
  {
    SpmvArgs a;
    a.b = b;
    a.fin.kind = FIN_BETA;
    a.fin.st = K.st;
    a.fin.i = 2;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
  }
  auto set = [&](int mode) {
    return [&, mode](cudaGraphConditionalHandle h) {
      cond_set_kernel<<<1, 1, 0, c.stream>>>(h, K.st, mode, max_iters);
      SAG_LAUNCHED(c);
    };
  };
  cond_node(c, cudaGraphCondTypeWhile, set(0), [&](cudaGraphConditionalHandle hw) {
    SpmvArgs a;  // restart from the true residual (krylov.cpp:43-53)
    a.b = b;
    a.fin.kind = FIN_BETA;
    a.fin.st = K.st;
    a.fin.i = 0;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
    launch_div(c, n, K.r.p, K.beta(), K.v(0), K.stop());
    for (int j = 0; j < restart; ++j) {
      cond_node(c, cudaGraphCondTypeIf, set(1), [&](cudaGraphConditionalHandle) {
        prec(K.v(j), K.z(j));
        arnoldi_step(c, A, K, restart, j, K.stop());
      });
    }
    launch_backsub(c, K.st);
    launch_update(c, n, x, K.Z.p, (size_t)n, K.st, false);
    cond_set_kernel<<<1, 1, 0, c.stream>>>(hw, K.st, 0, max_iters);
    SAG_LAUNCHED(c);
  });
  {
    SpmvArgs a;  // final true residual (krylov.cpp:116-119)
    a.b = b;
    a.fin.kind = FIN_FINAL;
    a.fin.st = K.st;
    a.fin.out = final_out;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
  }
}

// ========================================================== coarse solve ==
// MonolithicSolver coarse level (preconditioner.cpp:47-54, :60-63): dense LU
// with partial pivoting of to_dense(K_L) (+ enclosed-flow pin), factorised on
// the device with the reference's elimination order. The solve applies the
// explicit inverse (columns = dense_lu_solve(lu, e_c)) as one coalesced dense
// mat-vec; SAG_COARSE=lu selects a row-oriented triangular solve instead.

__global__ void dense_scatter_kernel(int n, const int* rp, const int* ci, const double* v,
                                     double* A) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    for (int k = rp[r]; k < rp[r + 1]; ++k) A[(size_t)r * n + ci[k]] += v[k];
}

__global__ void pin_kernel(double* A, int n, int row, double pin) {
  A[(size_t)row * n + row] += pin;
}

// sparse.cpp:310-341 by one CTA on a row-major matrix in global memory.
__global__ void __launch_bounds__(1024) dense_lu_kernel(int n, double* A, int* piv, int* err) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int sp;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
  for (int i = tid; i < n; i += nt) piv[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = k + 1 + tid; i < n; i += nt) {
      const double v = fabs(A[(size_t)i * n + k]);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sv[wid] = bv;
      si[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int bidx = n;
      for (int w = 0; w < (nt >> 5); ++w)
        if (sv[w] > b || (sv[w] == b && si[w] < bidx)) {
          b = sv[w];
          bidx = si[w];
        }
      const double akk = fabs(A[(size_t)k * n + k]);
      int p = (b > akk) ? bidx : k;
      const double best = (b > akk) ? b : akk;
      if (best == 0.0) {
        *err = 1;
        p = -1;
      }
      sp = p;
    }
    __syncthreads();
    const int p = sp;
    if (p < 0) return;
    if (p != k) {
      for (int j = tid; j < n; j += nt) {
        const double t = A[(size_t)k * n + j];
        A[(size_t)k * n + j] = A[(size_t)p * n + j];
        A[(size_t)p * n + j] = t;
      }
      if (tid == 0) {
        const int t = piv[k];
        piv[k] = piv[p];
        piv[p] = t;
      }
    }
    __syncthreads();
    const double inv = __ddiv_rn(1.0, A[(size_t)k * n + k]);
    for (int i = k + 1 + tid; i < n; i += nt) A[(size_t)i * n + k] = __dmul_rn(A[(size_t)i * n + k], inv);
    __syncthreads();
    const int m = n - k - 1;
    for (long long e = tid; e < (long long)m * m; e += nt) {
      const int i = k + 1 + (int)(e / m), j = k + 1 + (int)(e % m);
      const double mult = A[(size_t)i * n + k];
      if (mult != 0.0) A[(size_t)i * n + j] = __dsub_rn(A[(size_t)i * n + j], __dmul_rn(mult, A[(size_t)k * n + j]));
    }
    __syncthreads();
  }
}

// inverse columns: thread c solves e_c with the reference's substitution order
__global__ void dense_inv_kernel(int n, const double* LU, const int* piv, double* X,
                                 double* Ainv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double* x = X + (size_t)c * n;
  for (int i = 0; i < n; ++i) x[i] = piv[i] == c ? 1.0 : 0.0;
  for (int i = 1; i < n; ++i) {
    double acc = x[i];
    for (int j = 0; j < i; ++j) acc = __dsub_rn(acc, __dmul_rn(LU[(size_t)i * n + j], x[j]));
    x[i] = acc;
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = x[i];
    for (int j = i + 1; j < n; ++j) acc = __dsub_rn(acc, __dmul_rn(LU[(size_t)i * n + j], x[j]));
    x[i] = __ddiv_rn(acc, LU[(size_t)i * n + i]);
  }
  for (int i = 0; i < n; ++i) Ainv[(size_t)i * n + c] = x[i];
}

// x = Ainv b, one warp per row
__global__ void dense_matvec_kernel(int n, const double* __restrict__ A,
                                    const double* __restrict__ b, double* __restrict__ x) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const double* row = A + (size_t)warp * n;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = fma(row[j], b[j], s);
  s = warp_sum(s);
  if (lane == 0) x[warp] = s;
}

// dense_lu_solve (sparse.cpp:343-369) by one warp: row-oriented sweeps, the
// per-row dot products as warp trees.
__global__ void dense_lu_solve_kernel(int n, const double* __restrict__ LU,
                                      const int* __restrict__ piv, const double* __restrict__ b,
                                      double* __restrict__ x) {
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) x[i] = b[piv[i]];
  __syncwarp();
  for (int i = 1; i < n; ++i) {
    double s = 0.0;
    for (int j = lane; j < i; j += 32) s = fma(LU[(size_t)i * n + j], x[j], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = x[i] - s;
    __syncwarp();
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1 + lane; j < n; j += 32) s = fma(LU[(size_t)i * n + j], x[j], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = (x[i] - s) / LU[(size_t)i * n + i];
    __syncwarp();
  }
}

struct Coarse {
  int n = 0;
  bool use_inv = true;
  DevBuf<double> lu, inv;
  DevBuf<int> piv;
  void setup(Ctx& c, const Matrix& K, int pin_row, double pin) {
    n = K.nrows;
    SAG_REQUIRE(n == K.ncols && n > 0, SAG_DIMENSION_MISMATCH, "coarse level must be square");
    SAG_REQUIRE(n <= 8192, SAG_ERROR, "coarse level too large for the dense solve");
    if (const char* e = getenv("SAG_COARSE")) use_inv = std::strcmp(e, "lu") != 0;
    lu.alloc((size_t)n * n);
    piv.alloc(n);
    SAG_CUDA(cudaMemsetAsync(lu.p, 0, sizeof(double) * n * n, c.stream));
    dense_scatter_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(n, K.rp.p, K.ci.p, K.v.p, lu.p);
    SAG_LAUNCHED(c);
    if (pin_row >= 0) {
      pin_kernel<<<1, 1, 0, c.stream>>>(lu.p, n, pin_row, pin);
      SAG_LAUNCHED(c);
    }
    DevBuf<int> err(1);
    SAG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
    dense_lu_kernel<<<1, 1024, 0, c.stream>>>(n, lu.p, piv.p, err.p);
    SAG_LAUNCHED(c);
    int herr = 0;
    SAG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    if (herr) throw Error(SAG_SINGULAR_MATRIX, "dense_lu_factor: singular pivot column (coarse level)");
    if (use_inv) {
      inv.alloc((size_t)n * n);
      DevBuf<double> X((size_t)n * n);
      dense_inv_kernel<<<(n + 63) / 64, 64, 0, c.stream>>>(n, lu.p, piv.p, X.p, inv.p);
      SAG_LAUNCHED(c);
      SAG_CUDA(cudaStreamSynchronize(c.stream));
    }
  }
  void solve(Ctx& c, const double* b, double* x) {
    if (use_inv) {
      dense_matvec_kernel<<<(n * 32 + 255) / 256, 256, 0, c.stream>>>(n, inv.p, b, x);
    } else {
      dense_lu_solve_kernel<<<1, 32, 0, c.stream>>>(n, lu.p, piv.p, b, x);
    }
    SAG_LAUNCHED(c);
  }
};

// ==================================================== monolithic solver ==

// A whole solve_stokes (FGMRES with its preconditioner) as one CUDA graph:
// the convergence loop as conditional nodes (fgmres_graph), every
// preconditioner application inline. Re-captured when the buffers or
// settings it was captured with change.
struct SolveGraph {
  cudaGraphExec_t exec = nullptr;
  const void* key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int restart = 0, max_iters = 0, enclosed = 0;
  double tol = 0.0;
  long long apply_fine = 0, apply_l1 = 0;  // relaxation units per application
  ~SolveGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

struct Level {
  const Matrix* K = nullptr;
  const Matrix* P = nullptr;
  std::unique_ptr<Matrix> R;  // P^T, built once (the reference rebuilds it per call, :72)
  int n_x = 0, n_y = 0, n_p = 0, n = 0;
  std::unique_ptr<Vanka> vanka;
  Krylov kry;
  DevBuf<double> b, x, r;
};

// SV transfer pieces (transfer.cpp:18-53): duplication P^p, mixed mass M_mix,
// Mcg with its scalar SA hierarchy (amg.cpp:231-296).
// ScalarHierarchy (amg.hpp:64-72) on device: levels A_l, prolongators P_l,
// R_l = P_l^T, Jacobi diagonals, V-cycle workspaces, dense coarse solve.
struct ScalarH {
  std::vector<const Matrix*> A;
  std::vector<const Matrix*> P;
  std::vector<std::unique_ptr<Matrix>> R;
  std::vector<DevBuf<double>> dinv, sb, sx, sr;
  std::vector<Krylov> kr;        // Jacobi-FGMRES(2) smoothing workspaces
  Coarse coarse;
  // sliced ELLPACK copies of A_l, R_l, P_l for the persistent kernels (built on demand)
  std::vector<std::unique_ptr<Sell>> ella, ellr, ellp;
  int tail_from = -1;            // levels >= tail_from run as one cluster launch
  TailParams tail;
  int n() const { return A.empty() ? 0 : A[0]->nrows; }
};

struct SvTransfer {
  const Matrix* pdup = nullptr;
  const Matrix* mmix = nullptr;
  ScalarH sh;                    // scalar SA hierarchy of Mcg
  Krylov outer;                  // FGMRES(20) on Mcg
  DevBuf<double> rhs, pcg;
  std::vector<int> iterations;
  DevBuf<int> fail;              // set when a graph-run projection did not converge
  // the whole projection as one persistent launch (sv_project_kernel)
  bool fused = false;
  ProjParams proj;
  DevBuf<unsigned long long> proj_sync;
  std::unique_ptr<Sell> sell_mmix;
  DevBuf<unsigned long long> proj_trace;  // SAG_PROJ_TRACE=1 (diagnostic)
};

__global__ void proj_check_kernel(const KState* st, int* fail) {
  if (!st->converged) *fail = 1;
}

// UzawaPreconditioner (preconditioner.hpp:118-141) on device.
struct Uzawa {
  Ctx* ctx = nullptr;
  const Matrix* B = nullptr;     // n_p x n_u
  int n_x = 0, n_y = 0, n_p = 0;
  ScalarH hx, hy, hp;            // hp unused for SV
  bool sv_exact_mass = false;
  DevBuf<double> areas;          // SV element areas (n_p / 3)
  DevBuf<double> t;              // r_p - B du
  DevBuf<double> pv;             // V(r_p - B du) before the sign flip (TH)
  DevBuf<double> din, dout;
  cudaGraphExec_t graph = nullptr;
  bool graph_ok = false;
  long long graph_launches = 0;
  SolveGraph solve_graph;
  ~Uzawa() {
    if (graph) cudaGraphExecDestroy(graph);
  }
};

struct Dc {
  Ctx* ctx = nullptr;
  const Matrix* K0 = nullptr;
  int n_x0 = 0, n_y0 = 0, n_p0 = 0, n0 = 0;
  bool sv = false;
  sag_solver_config cfg{};
  std::unique_ptr<Vanka> fine;
  Krylov fine_kry;
  DevBuf<double> fine_r;
  std::vector<Level> lv;
  Coarse coarse;
  std::unique_ptr<SvTransfer> svt;
  bool ho = false;  // HoAmgPreconditioner: V-cycle on a hierarchy whose level 0 is K0
  long long fine_units = 0, l1_units = 0;
  // outer solve workspace
  Krylov outer;
  DevBuf<double> din, dout;
  DevBuf<double> gam_rc, gam_e;  // gamma > 1 accumulators
  // CUDA graph of apply(din -> dout)
  cudaGraphExec_t graph = nullptr;
  bool graph_ok = false;
  long long graph_launches = 0;
  SolveGraph solve_graph;
  ~Dc() {
    if (graph) cudaGraphExecDestroy(graph);
  }
};

// MonolithicSolver::cycle_level (preconditioner.cpp:57-81) on lv[l]:
// input lv[l].b, output lv[l].x (from a zero guess).
static void cycle_level(Ctx& c, Dc& d, int l, int nu1, int nu2, bool skip_finest) {
  Level& L = d.lv[l];
  const int nl = (int)d.lv.size();
  if (l == nl - 1) {
    d.coarse.solve(c, L.b.p, L.x.p);
    return;
  }
  const bool relax_here = !(l == 0 && skip_finest);
  const bool pre = relax_here && nu1 > 0;
  if (pre)
    relax_kw(c, *L.K, *L.vanka, L.kry, L.x.p, L.b.p, nu1, true);
  else
    launch_zero(c, L.n, L.x.p);
  Level& C = d.lv[l + 1];
  if (pre) {
    if (nu1 == 1) {
      // x = y_0 z_0 and w = K z_0: r = b - y_0 w (= b - K x by linearity)
      launch_lin_resid(c, L.n, L.n, 1.0, 1.0, L.b.p, L.kry.w.p, L.kry.st, L.r.p);
    } else {
      SpmvArgs a;
      a.b = L.b.p;
      launch_spmv(c, *L.K, L.x.p, L.r.p, Epi::Resid, a);
    }
    launch_spmv(c, *L.R, L.r.p, C.b.p, Epi::Store);
  } else {
    launch_spmv(c, *L.R, L.b.p, C.b.p, Epi::Store);
  }
  cycle_level(c, d, l + 1, nu1, nu2, skip_finest);
  launch_spmv(c, *L.P, C.x.p, L.x.p, Epi::Add);
  if (relax_here && nu2 > 0) relax_kw(c, *L.K, *L.vanka, L.kry, L.x.p, L.b.p, nu2, false);
}

// ---- scalar V-cycle (amg.cpp:258-296) ---------------------------------------

// scalar_vcycle on level l of a scalar hierarchy: FGMRES(2) Jacobi smoothing
// from the current x, R = P^T, dense coarse solve.
static void scalar_level(Ctx& c, ScalarH& t, int l, const double* b, double* x);

static void jacobi_fgmres2(Ctx& c, ScalarH& t, int l, const double* b, double* x, bool x_zero) {
  // fgmres(matrix_operator(a), b, x, jacobi, {tol 0, max 2, restart 2}) with x in/out:
  // bnorm = ||b|| is the reference (krylov.cpp:23-24), the residual b - a x.
  // z_j = jacobi(v_j) is formed in the pass that forms v_j; v_2 (never used
  // by the update) is not formed.
  const Matrix& A = *t.A[l];
  Krylov& K = t.kr[l];
  const int n = A.nrows;
  Fin fr;
  fr.kind = FIN_REF;
  fr.st = K.st;
  Fin fb;
  fb.kind = FIN_BETA;
  fb.st = K.st;
  fb.i = 4;  // init m = 2, tol = 0 (ref kept from FIN_REF)
  fb.j = 2;
  fb.tol = 0.0;
  const double* r;
  if (x_zero) {
    launch_ssq2(c, n, b, fr, fb);  // r = b: ||b|| is both
    r = b;
  } else {
    // post-smoothing follows the pre-smoothing of the same b on this level's
    // KState, whose ref = ||b|| is still in place (same value, no pass).
    // Invariant: only scalar_level calls this with x_zero = false, right
    // after the x_zero = true call on the same level and b. With tol = 0 the
    // value of ref only matters as a positive number, and FIN_BETA falls
    // back to 1 when it was never set.
    SpmvArgs a;
    a.b = b;
    a.fin = fb;
    launch_spmv(c, A, x, K.r.p, Epi::ResidSsq, a);
    r = K.r.p;
  }
  const double* dinv = t.dinv[l].p;
  launch_div_mul(c, n, r, K.beta(), K.v(0), dinv, K.z(0), K.stop());
  arnoldi_step(c, A, K, 2, 0, K.stop(), false, dinv);
  arnoldi_step(c, A, K, 2, 1, K.stop(), true);
  launch_update_bs(c, n, x, K.Z.p, (size_t)n, K.st, 2, x_zero);
}

static void scalar_level(Ctx& c, ScalarH& t, int l, const double* b, double* x) {
  const int nl = (int)t.A.size();
  if (l == nl - 1) {
    t.coarse.solve(c, b, x);
    return;
  }
  if (l == t.tail_from) {
    TailParams p = t.tail;
    p.b0 = b;
    p.x0 = x;
    launch_scalar_tail(c, p);
    return;
  }
  const Matrix& A = *t.A[l];
  jacobi_fgmres2(c, t, l, b, x, true);
  SpmvArgs a;
  a.b = b;
  launch_spmv(c, A, x, t.sr[l].p, Epi::Resid, a);
  launch_spmv(c, *t.R[l], t.sr[l].p, t.sb[l + 1].p, Epi::Store);
  scalar_level(c, t, l + 1, t.sb[l + 1].p, t.sx[l + 1].p);
  launch_spmv(c, *t.P[l], t.sx[l + 1].p, x, Epi::Add);
  jacobi_fgmres2(c, t, l, b, x, false);
}

// scalar_vcycle (amg.cpp:290-296) from x = 0: x <- V(2,2) b
static void scalar_vcycle(Ctx& c, ScalarH& t, const double* b, double* x) {
  scalar_level(c, t, 0, b, x);
}

// build_scalar_hierarchy's device half: levels and prolongators come from
// the host build (amg.cpp:200-253); R = P^T, d_inv, coarse LU here.
static void scalar_setup(Ctx& c, ScalarH& t, int nl, const sag_matrix* const* a,
                         const sag_matrix* const* p, const char* what);

// ---- SV restriction: p_cg = Mcg^-1 (M_mix p_dg) (transfer.cpp:18-37) ------

static void sv_restrict(Ctx& c, Dc& d, const double* p_dg, double* p_cg) {
  SvTransfer& t = *d.svt;
  if (t.fused) {
    // M_mix product, FGMRES(20) and its V(2,2) cycles in one persistent launch
    ProjParams p = t.proj;
    p.p_dg = p_dg;
    p.x = p_cg;
    launch_sv_project(c, p);
    if (stream_capturing(c)) return;  // failure flagged on the device (t.fail)
    KHeader hd = read_header(c, t.outer.st);
    if (!hd.converged)
      throw Error(SAG_SOLVER_STAGNATION,
                  "SvPressureRestrict: mass projection did not reach tolerance in 200 iterations");
    t.iterations.push_back(hd.iterations);
    return;
  }
  launch_spmv(c, *t.mmix, p_dg, t.rhs.p, Epi::Store);
  launch_zero(c, t.mmix->nrows, p_cg);
  DevOp prec = [&](const double* in, double* out) { scalar_vcycle(c, t.sh, in, out); };
  if (stream_capturing(c)) {
    // inside the DC apply's CUDA graph: the device-side convergence loop; a
    // failure is flagged on the device and raised at the next host check
    // SAG_PROJ_RESTART (diagnostic only; default 20 = transfer.cpp:27) caps the
    // number of IF nodes per restart cycle of the graph
    const char* pr = getenv("SAG_PROJ_RESTART");
    const int rst = pr ? std::max(1, std::min(20, atoi(pr))) : 20;
    fgmres_graph(c, *t.sh.A[0], t.rhs.p, p_cg, prec, 1e-12, 200, rst, 1e-30, t.outer,
                 c.scal.p + 8);
    proj_check_kernel<<<1, 1, 0, c.stream>>>(t.outer.st, t.fail.p);
    SAG_LAUNCHED(c);
    return;
  }
  FgmresOut o = fgmres_dev(c, *t.sh.A[0], t.rhs.p, p_cg, prec, 1e-12, 200, 20, 1e-30, t.outer);
  if (!o.converged)
    throw Error(SAG_SOLVER_STAGNATION,
                "SvPressureRestrict: mass projection did not reach tolerance in 200 iterations");
  t.iterations.push_back(o.iterations);
}

// DCPreconditioner::apply (preconditioner.cpp:114-153), r -> z on device.
static void dc_apply_dev(Ctx& c, Dc& d, const double* r, double* z) {
  const sag_solver_config& cf = d.cfg;
  if (d.ho) {
    // HoAmgPreconditioner::apply (preconditioner.cpp:174-176): one V-cycle of
    // the hierarchy built on the high-order system itself, from x = 0
    Level& L0 = d.lv[0];
    launch_copy(c, L0.n, r, L0.b.p);
    cycle_level(c, d, 0, cf.nu1, cf.nu2, false);
    launch_copy(c, L0.n, L0.x.p, z);
    if (d.lv.size() > 1) d.fine_units += cf.nu1 + cf.nu2;
    return;
  }
  const bool relax_fine = cf.variant != SAG_DC_LO;
  const bool pre = relax_fine && cf.nu1 > 0;
  double* x = z;
  if (pre) {
    if (d.sv)
      relax_stationary(c, *d.K0, *d.fine, d.fine_r.p, x, r, cf.nu1, cf.omega0, true);
    else
      relax_kw(c, *d.K0, *d.fine, d.fine_kry, x, r, cf.nu1, true);
    d.fine_units += cf.nu1;
  } else {
    launch_zero(c, d.n0, x);
  }
  Level& L0 = d.lv[0];
  const int n_u0 = d.n_x0 + d.n_y0;
  // r1 = r - K0 x, eta weighting (transfer.cpp:127-135), TH restriction = copy
  double* rw = d.sv ? d.fine_r.p : L0.b.p;
  {
    SpmvArgs a;
    a.b = r;
    a.eta_u = cf.eta_u;
    a.eta_p = cf.eta_p;
    a.n_u = n_u0;
    if (pre && !d.sv && cf.nu1 == 1)
      launch_lin_resid(c, d.n0, n_u0, cf.eta_u, cf.eta_p, r, d.fine_kry.w.p, d.fine_kry.st, rw);
    else if (pre)
      launch_spmv(c, *d.K0, x, rw, Epi::ResidEta, a);
    else
      launch_eta(c, d.n0, n_u0, cf.eta_u, cf.eta_p, r, rw);  // r1 = r (preconditioner.cpp:128-129)
  }
  const int n_u1 = L0.n_x + L0.n_y;
  if (d.sv) {
    // velocity injection + pressure mass projection (transfer.cpp:112-125)
    launch_copy(c, n_u1, rw, L0.b.p);
    sv_restrict(c, d, rw + n_u0, L0.b.p + n_u1);
  }
  const bool skip_finest = cf.variant == SAG_DC_HO;
  const int nl = (int)d.lv.size();
  if (cf.gamma <= 1) {
    cycle_level(c, d, 0, cf.nu1, cf.nu2, skip_finest);
  } else {
    // e accumulates gamma V-cycles (preconditioner.cpp:131-145)
    DevBuf<double>& rc = d.gam_rc;
    DevBuf<double>& e = d.gam_e;
    launch_copy(c, L0.n, L0.b.p, rc.p);
    launch_zero(c, L0.n, e.p);
    for (int g = 0; g < cf.gamma; ++g) {
      if (g > 0) {
        SpmvArgs a;
        a.b = rc.p;
        launch_spmv(c, *L0.K, e.p, L0.b.p, Epi::Resid, a);
      } else {
        launch_copy(c, L0.n, rc.p, L0.b.p);
      }
      cycle_level(c, d, 0, cf.nu1, cf.nu2, skip_finest);
      launch_add(c, L0.n, e.p, L0.x.p);
    }
    launch_copy(c, L0.n, e.p, L0.x.p);
  }
  if (nl > 1 && !skip_finest) d.l1_units += (long long)cf.gamma * (cf.nu1 + cf.nu2);
  // prolong (transfer.cpp:97-110) and x += up
  if (!d.sv) {
    launch_add(c, d.n0, x, L0.x.p);
  } else {
    launch_add(c, n_u0, x, L0.x.p);
    SpmvArgs a;
    launch_spmv(c, *d.svt->pdup, L0.x.p + n_u1, x + n_u0, Epi::Add, a);
  }
  if (relax_fine && cf.nu2 > 0) {
    if (d.sv)
      relax_stationary(c, *d.K0, *d.fine, d.fine_r.p, x, r, cf.nu2, cf.omega0, false);
    else
      relax_kw(c, *d.K0, *d.fine, d.fine_kry, x, r, cf.nu2, false);
    d.fine_units += cf.nu2;
  }
}

static void check_config(const sag_solver_config& c) {
  // SolverConfig::check (preconditioner.cpp:30-38)
  SAG_REQUIRE(c.eta_u > 0.0 && c.eta_p > 0.0, SAG_CONFIG_ERROR, "eta_u and eta_p must be positive");
  SAG_REQUIRE(c.omega0 > 0.0 && c.omega0 < 2.0, SAG_CONFIG_ERROR, "omega0 must lie in (0, 2)");
  SAG_REQUIRE(c.nu1 >= 0 && c.nu2 >= 0, SAG_CONFIG_ERROR, "nu1 and nu2 must be non-negative");
  SAG_REQUIRE(c.gamma >= 1, SAG_CONFIG_ERROR, "gamma must be at least 1");
  SAG_REQUIRE(c.restart >= 1, SAG_CONFIG_ERROR, "restart must be at least 1");
  SAG_REQUIRE(c.tol > 0.0, SAG_CONFIG_ERROR, "tol must be positive");
  SAG_REQUIRE(c.max_iters >= 1, SAG_CONFIG_ERROR, "max_iters must be at least 1");
  SAG_REQUIRE(c.variant >= 0 && c.variant <= 4, SAG_CONFIG_ERROR, "unknown solver variant");
}

// DC apply as a CUDA graph over the fixed buffers din -> dout (SV excluded:
// its mass projection synchronises with the host for convergence).
// A caller capturing its own CUDA graph on the context stream (a graph launch
// cannot be captured): the launches go straight into the caller's graph.
static bool stream_capturing(Ctx& c) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  SAG_CUDA(cudaStreamIsCapturing(c.stream, &st));
  return st != cudaStreamCaptureStatusNone;
}

static void dc_apply_graph(Ctx& c, Dc& d) {
  // SV included: its mass projection runs as conditional graph nodes
  const bool use_graph = !(getenv("SAG_NO_GRAPH") && atoi(getenv("SAG_NO_GRAPH"))) &&
                         !(d.sv && getenv("SAG_SV_GRAPH") && !atoi(getenv("SAG_SV_GRAPH"))) &&
                         !stream_capturing(c);
  if (!use_graph) {
    dc_apply_dev(c, d, d.din.p, d.dout.p);
    return;
  }
  if (!d.graph_ok) {
    const long long fu = d.fine_units, lu = d.l1_units, la = c.launches;
    cudaGraph_t g;
    SAG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      dc_apply_dev(c, d, d.din.p, d.dout.p);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      throw;
    }
    SAG_CUDA(cudaStreamEndCapture(c.stream, &g));
    if (d.graph) cudaGraphExecDestroy(d.graph);
    SAG_CUDA(cudaGraphInstantiate(&d.graph, g, 0));
    cudaGraphDestroy(g);
    d.graph_ok = true;
    d.fine_units = fu;
    d.l1_units = lu;
    d.graph_launches = c.launches - la;
    c.launches = la;
  }
  SAG_CUDA(cudaGraphLaunch(d.graph, c.stream));
  c.launches += d.graph_launches;
  const sag_solver_config& cf = d.cfg;
  if (d.ho) {
    if (d.lv.size() > 1) d.fine_units += cf.nu1 + cf.nu2;
    return;
  }
  if (cf.variant != SAG_DC_LO) d.fine_units += cf.nu1 + cf.nu2;
  if (cf.variant != SAG_DC_HO && d.lv.size() > 1)
    d.l1_units += (long long)cf.gamma * (cf.nu1 + cf.nu2);
}

__global__ void neg_copy_kernel(int n, const double* __restrict__ in, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = -in[i];
}

// SV exact element mass inverse (preconditioner.cpp:201-211) applied to
// s = r_p - B du = -t: dp = (3/a)[[3,-1,-1],[-1,3,-1],[-1,-1,3]] t, the
// reference's operation order (negation is exact).
__global__ void sv_mass_inv_kernel(int ne, const double* __restrict__ areas,
                                   const double* __restrict__ s, double* __restrict__ dp) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const double cc = __ddiv_rn(3.0, areas[e]);
    const double t0 = -s[3 * e], t1 = -s[3 * e + 1], t2 = -s[3 * e + 2];
    dp[3 * e] = __dmul_rn(cc, __dsub_rn(__dsub_rn(__dmul_rn(3.0, t0), t1), t2));
    dp[3 * e + 1] = __dmul_rn(cc, __dsub_rn(__dadd_rn(-t0, __dmul_rn(3.0, t1)), t2));
    dp[3 * e + 2] = __dmul_rn(cc, __dadd_rn(__dsub_rn(-t0, t1), __dmul_rn(3.0, t2)));
  }
}

// UzawaPreconditioner::apply (preconditioner.cpp:186-218): du = scalar
// V-cycles on A_x, A_y; t = B du - r_p; dp = Q_B^-1 t (exact element mass
// inverse for SV, scalar V-cycle on Mp for TH/ISO). Computed as s = -t (the
// residual epilogue) and dp = -V(s) = V(t): FGMRES from x = 0 is odd in b.
static void uzawa_apply_dev(Ctx& c, Uzawa& u, const double* r, double* z) {
  const int n_u = u.n_x + u.n_y;
  scalar_vcycle(c, u.hx, r, z);
  scalar_vcycle(c, u.hy, r + u.n_x, z + u.n_x);
  SpmvArgs a;
  a.b = r + n_u;
  launch_spmv(c, *u.B, z, u.t.p, Epi::Resid, a);
  const int g = std::max(1, std::min((u.n_p + 255) / 256, c.num_sms * 8));
  if (u.sv_exact_mass) {
    sv_mass_inv_kernel<<<g, 256, 0, c.stream>>>(u.n_p / 3, u.areas.p, u.t.p, z + n_u);
    SAG_LAUNCHED(c);
  } else {
    scalar_vcycle(c, u.hp, u.t.p, u.pv.p);
    neg_copy_kernel<<<g, 256, 0, c.stream>>>(u.n_p, u.pv.p, z + n_u);
    SAG_LAUNCHED(c);
  }
}

// Uzawa apply din -> dout captured once into a CUDA graph (fixed sequence).
static void uzawa_apply_graph(Ctx& c, Uzawa& u) {
  const bool use_graph = !(getenv("SAG_NO_GRAPH") && atoi(getenv("SAG_NO_GRAPH"))) &&
                         !stream_capturing(c);
  if (!use_graph) {
    uzawa_apply_dev(c, u, u.din.p, u.dout.p);
    return;
  }
  if (!u.graph_ok) {
    const long long la = c.launches;
    cudaGraph_t g;
    SAG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      uzawa_apply_dev(c, u, u.din.p, u.dout.p);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      throw;
    }
    SAG_CUDA(cudaStreamEndCapture(c.stream, &g));
    if (u.graph) cudaGraphExecDestroy(u.graph);
    SAG_CUDA(cudaGraphInstantiate(&u.graph, g, 0));
    cudaGraphDestroy(g);
    u.graph_ok = true;
    u.graph_launches = c.launches - la;
    c.launches = la;
  }
  SAG_CUDA(cudaGraphLaunch(u.graph, c.stream));
  c.launches += u.graph_launches;
}

constexpr int kTailRows = 65536;  // largest level the cluster tail takes

static bool scalar_tail_from(Ctx& c, ScalarH& t, int from, TailParams& tp);

static void scalar_setup(Ctx& c, ScalarH& t, int nl, const sag_matrix* const* a,
                         const sag_matrix* const* p, const char* what) {
  SAG_REQUIRE(nl >= 1, SAG_DIMENSION_MISMATCH, std::string(what) + ": empty scalar hierarchy");
  SAG_NOTNULL(a);
  for (int l = 0; l < nl; ++l) {
    SAG_NOTNULL(a[l]);
    t.A.push_back(&a[l]->m);
    SAG_REQUIRE(t.A[l]->nrows == t.A[l]->ncols, SAG_DIMENSION_MISMATCH,
                std::string(what) + ": scalar level is not square");
  }
  t.kr.resize(nl);
  t.dinv.resize(nl);
  t.sb.resize(nl);
  t.sx.resize(nl);
  t.sr.resize(nl);
  for (int l = 0; l < nl; ++l) {
    const int n = t.A[l]->nrows;
    t.sb[l].alloc(n);
    t.sx[l].alloc(n);
    if (l + 1 < nl) {
      SAG_NOTNULL(p);
      SAG_NOTNULL(p[l]);
      t.P.push_back(&p[l]->m);
      SAG_REQUIRE(t.P[l]->nrows == n && t.P[l]->ncols == t.A[l + 1]->nrows,
                  SAG_DIMENSION_MISMATCH, std::string(what) + ": prolongator shape mismatch");
      t.R.push_back(transpose_dev(c, *t.P.back()));
      t.kr[l].init(n, 2, 0);
      t.dinv[l].alloc(n);
      t.sr[l].alloc(n);
      int* bad = reinterpret_cast<int*>(c.scal.p + 8);
      SAG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
      launch_inv_diag(c, *t.A[l], t.dinv[l].p, bad);
      int hb = 0;
      SAG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      SAG_CUDA(cudaStreamSynchronize(c.stream));
      SAG_REQUIRE(!hb, SAG_ZERO_DIAGONAL, std::string("inv_diagonal: zero diagonal (") + what + ")");
    }
  }
  t.coarse.setup(c, *t.A.back(), -1, 0.0);
  // the small levels as one cluster launch (SAG_SCALAR_TAIL=0: per-kernel path)
  const char* e = getenv("SAG_SCALAR_TAIL");
  if ((e && std::strcmp(e, "0") == 0) || !t.coarse.use_inv) return;
  for (int from = 0; from + 1 < nl; ++from) {
    TailParams tp;
    if (!scalar_tail_from(c, t, from, tp)) continue;  // too large for the shared memory: next level
    t.tail = tp;
    t.tail_from = from;
    return;
  }
}

// sliced ELLPACK copies of level l's matrices
static void scalar_sell(Ctx& c, ScalarH& t, int l) {
  const int nl = (int)t.A.size();
  if ((int)t.ella.size() < nl) {
    t.ella.resize(nl);
    t.ellr.resize(nl);
    t.ellp.resize(nl);
  }
  if (t.ella[l]) return;
  t.ella[l] = std::make_unique<Sell>();
  build_sell(c, *t.A[l], *t.ella[l]);
  if (l + 1 < nl) {
    t.ellr[l] = std::make_unique<Sell>();
    build_sell(c, *t.R[l], *t.ellr[l]);
    t.ellp[l] = std::make_unique<Sell>();
    build_sell(c, *t.P[l], *t.ellp[l]);
  }
}

// levels from.. of t as a cluster tail; false when they do not fit
static bool scalar_tail_from(Ctx& c, ScalarH& t, int from, TailParams& tp) {
  const int nl = (int)t.A.size();
  const char* er = getenv("SAG_TAIL_ROWS");
  const int rows_max = er ? atoi(er) : kTailRows;
  if (!t.coarse.use_inv || from < 0 || from >= nl) return false;
  if (t.A[from]->nrows > rows_max || nl - from > kTailMaxLev) return false;
  tp = TailParams();
  tp.nlev = nl - from;
  tp.cinv = t.coarse.inv.p;
  for (int l = from; l < nl; ++l) {
    TailLevel& L = tp.L[l - from];
    const Matrix& A = *t.A[l];
    L.n = A.nrows;
    L.arp = A.rp.p;
    L.aci = A.ci.p;
    L.av = A.v.p;
    if (l + 1 < nl) {
      L.rrp = t.R[l]->rp.p;
      L.rci = t.R[l]->ci.p;
      L.rv = t.R[l]->v.p;
      L.prp = t.P[l]->rp.p;
      L.pci = t.P[l]->ci.p;
      L.pv = t.P[l]->v.p;
      L.dinv = t.dinv[l].p;
    }
  }
  return scalar_tail_plan(c, tp);
}

// SvTransfer: plan the one-launch projection (sv_project_kernel) when the
// hierarchy splits into 1..kProjMaxGl grid levels + a cluster tail
// (SAG_PROJ_FUSED=1; the default is the multi-launch path)
static void sv_project_setup(Ctx& c, SvTransfer& t) {
  t.fused = false;
  // opt-in: measured slower than the multi-launch path on B200 (DESIGN 5c)
  const char* e = getenv("SAG_PROJ_FUSED");
  if (!e || std::strcmp(e, "1") != 0) return;
  ScalarH& h = t.sh;
  const int nl = (int)h.A.size();
  if (nl < 2 || !h.coarse.use_inv) return;
  // SAG_PROJ_TAIL_ROWS (diagnostic): largest level the tail cluster takes here
  const char* etr = getenv("SAG_PROJ_TAIL_ROWS");
  const int tail_rows = etr ? atoi(etr) : kTailRows;
  for (int from = 1; from < nl && from <= kProjMaxGl; ++from) {
    ProjParams p;
    if (h.A[from]->nrows > tail_rows) continue;
    if (!scalar_tail_from(c, h, from, p.tail)) continue;
    p.ngl = from;
    for (int l = 0; l < from; ++l) {
      ProjLevel& L = p.G[l];
      L.n = h.A[l]->nrows;
      scalar_sell(c, h, l);
      L.a = h.ella[l]->view();
      L.rt = h.ellr[l]->view();
      L.p = h.ellp[l]->view();
      L.dinv = h.dinv[l].p;
      L.nc = h.A[l + 1]->nrows;
      L.b = h.sb[l].p;
      L.x = h.sx[l].p;
      L.r = h.sr[l].p;
      L.z0 = h.kr[l].z(0);
      L.z1 = h.kr[l].z(1);
    }
    p.tail.b0 = h.sb[from].p;
    p.tail.x0 = h.sx[from].p;
    p.n = h.n();
    if (!t.sell_mmix) {
      t.sell_mmix = std::make_unique<Sell>();
      build_sell(c, *t.mmix, *t.sell_mmix);
    }
    p.mm = t.sell_mmix->view();
    p.rhs = t.rhs.p;
    p.V = t.outer.V.p;
    p.Z = t.outer.Z.p;
    p.st = t.outer.st;
    p.restart = 20;   // transfer.cpp:27
    p.max_iters = 200;
    p.tol = 1e-12;
    p.bd = 1e-30;
    p.fail = t.fail.p;
    if (!sv_project_plan(c, p) || p.workers > 256) continue;
    // [barrier counter, pad] + reduction slots, zeroed together at every launch
    t.proj_sync.alloc(1 + (size_t)2 * p.workers * 4);
    p.bar = reinterpret_cast<unsigned*>(t.proj_sync.p);
    p.ll = t.proj_sync.p + 1;
    p.sync_bytes = t.proj_sync.bytes();
    if (const char* et = getenv("SAG_PROJ_TRACE"); et && std::strcmp(et, "0") != 0) {
      p.trace_cap = 8192;
      t.proj_trace.alloc((size_t)4 * p.trace_cap);
      SAG_CUDA(cudaMemset(t.proj_trace.p, 0, sizeof(unsigned long long) * 4 * p.trace_cap));
      p.trace = t.proj_trace.p;
    }
    t.proj = p;
    t.fused = true;
    return;
  }
}

}  // namespace sag

// =================================================================== C-ABI
using namespace sag;

struct sag_dc {
  Dc d;
};
struct sag_uzawa {
  Uzawa u;
  Krylov outer;
};

namespace {

void dc_setup(Ctx& c, Dc& d, const Matrix* k0, int n_x0, int n_y0, int n_p0, int sv, int nlevels,
              const sag_level_desc* levels, const sag_solver_config& cfg) {
  check_config(cfg);
  SAG_REQUIRE(nlevels >= 1, SAG_DIMENSION_MISMATCH, "sag_dc_create: empty hierarchy");
  SAG_REQUIRE(k0->nrows == k0->ncols && k0->nrows == n_x0 + n_y0 + n_p0, SAG_DIMENSION_MISMATCH,
              "sag_dc_create: K0 does not match its block sizes");
  d.ctx = &c;
  d.K0 = k0;
  d.n_x0 = n_x0;
  d.n_y0 = n_y0;
  d.n_p0 = n_p0;
  d.n0 = k0->nrows;
  d.sv = sv != 0;
  d.cfg = cfg;
  SAG_REQUIRE(cfg.variant != SAG_UZAWA, SAG_CONFIG_ERROR,
              "sag_dc_create: the Uzawa preconditioner is built by sag_uzawa_create");
  // HoAmgPreconditioner (preconditioner.cpp:155-172): the hierarchy is built
  // on the high-order system, so its level 0 is K0 and there is no separate
  // fine relaxation or transfer
  d.ho = cfg.variant == SAG_HOAMG;
  if (d.ho) {
    SAG_REQUIRE(!d.sv || cfg.allow_sv_hoamg, SAG_UNSUPPORTED_DISCRETIZATION,
                "HO-AMG on Scott-Vogelius is refused by default (known poorly convergent); set "
                "the override to force it");
    SAG_REQUIRE(levels[0].k && levels[0].k->m.nrows == d.n0 && levels[0].n_x == n_x0 &&
                    levels[0].n_y == n_y0 && levels[0].n_p == n_p0,
                SAG_DIMENSION_MISMATCH, "HO-AMG: level 0 of the hierarchy must be K0");
    d.sv = false;
  }
  const int mrelax = std::max(std::max(cfg.nu1, cfg.nu2), 1);
  // fine-level Vanka (preconditioner.cpp:95-97)
  if (!d.ho) {
    auto p = build_patches_dev(c, *k0, n_x0, n_y0, n_p0, d.sv);
    d.fine = factor_patches_dev(c, *k0, *p, n_x0 + n_y0);
    if (!d.sv) d.fine_kry.init(d.n0, mrelax, 0);
  }
  d.fine_r.alloc(d.n0);
  // low-order hierarchy (preconditioner.cpp:40-55)
  d.lv.resize(nlevels);
  for (int l = 0; l < nlevels; ++l) {
    Level& L = d.lv[l];
    SAG_NOTNULL(levels[l].k);
    L.K = &levels[l].k->m;
    L.n_x = levels[l].n_x;
    L.n_y = levels[l].n_y;
    L.n_p = levels[l].n_p;
    L.n = L.K->nrows;
    SAG_REQUIRE(L.K->ncols == L.n && L.n == L.n_x + L.n_y + L.n_p, SAG_DIMENSION_MISMATCH,
                "sag_dc_create: level " + std::to_string(l) + " does not match its block sizes");
    L.b.alloc(L.n);
    L.x.alloc(L.n);
    if (l + 1 < nlevels) {
      SAG_REQUIRE(levels[l].p != nullptr, SAG_DIMENSION_MISMATCH,
                  "sag_dc_create: missing prolongator on level " + std::to_string(l));
      L.P = &levels[l].p->m;
      SAG_REQUIRE(L.P->nrows == L.n && L.P->ncols == levels[l + 1].k->m.nrows,
                  SAG_DIMENSION_MISMATCH, "sag_dc_create: prolongator shape mismatch");
      auto p = build_patches_dev(c, *L.K, L.n_x, L.n_y, L.n_p, false);
      L.vanka = factor_patches_dev(c, *L.K, *p, L.n_x + L.n_y);
      L.R = transpose_dev(c, *L.P);
      L.kry.init(L.n, mrelax, 0);
      L.r.alloc(L.n);
    }
  }
  Level& B = d.lv.back();
  int pin_row = -1;
  double pin = 0.0;
  if (cfg.enclosed_flow) {
    Matrix& K1 = const_cast<Matrix&>(*d.lv[0].K);
    compute_norm_inf(c, K1);
    pin_row = B.n_x + B.n_y;
    pin = 1e-12 * K1.norm_inf;  // preconditioner.cpp:49-53 (norm of the FINEST level)
  }
  d.coarse.setup(c, *B.K, pin_row, pin);
  if (!d.ho && !d.sv) {
    SAG_REQUIRE(d.lv[0].n == d.n0 && d.lv[0].n_x + d.lv[0].n_y == n_x0 + n_y0,
                SAG_DIMENSION_MISMATCH,
                "DCPreconditioner: transfer does not match the low-order system");
  } else if (!d.ho) {
    SAG_REQUIRE(d.lv[0].n_x + d.lv[0].n_y == n_x0 + n_y0, SAG_DIMENSION_MISMATCH,
                "DCPreconditioner: transfer does not match the low-order system");
  }
  if (cfg.gamma > 1) {
    d.gam_rc.alloc(d.lv[0].n);
    d.gam_e.alloc(d.lv[0].n);
  }
  d.din.alloc(d.n0);
  d.dout.alloc(d.n0);
}

// A mass projection run inside the DC graph that missed its tolerance
// (transfer.cpp:32-34) is flagged on the device; raised here at a host sync.
void check_sv_projection(Ctx& c, Dc& d) {
  if (!d.svt) return;
  int f = 0;
  SAG_CUDA(cudaMemcpyAsync(&f, d.svt->fail.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  if (f) {
    SAG_CUDA(cudaMemsetAsync(d.svt->fail.p, 0, sizeof(int), c.stream));
    throw Error(SAG_SOLVER_STAGNATION,
                "SvPressureRestrict: mass projection did not reach tolerance in 200 iterations");
  }
}

void require_ready(Dc& d) {
  SAG_REQUIRE(!d.sv || d.svt, SAG_CONFIG_ERROR,
              "SV preconditioner needs sag_dc_set_sv_transfer before use");
}

// solve_stokes (preconditioner.cpp:229-259): outer FGMRES on K0 from x = 0 with
// apply_prec = project -> prec -> project when enclosed_flow. The
// preconditioner runs on the fixed buffers din -> dout (`run`).
template <class Run>
void solve_stokes_dev(Ctx& c, const Matrix& K0, int n_u, int n_p, double* din, double* dout,
                      Run run, Krylov& outer, const sag_solver_config& cfg, const double* rhs,
                      double* x, sag_krylov_report* rep, double* history, int history_cap,
                      SolveGraph* sg = nullptr, long long* units_fine = nullptr,
                      long long* units_l1 = nullptr) {
  const int n = K0.nrows;
  InVec bi(c, rhs, n, 0);
  OutVec xo(c, x, n, 1, false);
  launch_zero(c, n, xo.d);
  const int hist_cap = cfg.max_iters + 2;
  if (outer.n != n || outer.m < cfg.restart || outer.hist_cap < hist_cap)
    outer.init(n, cfg.restart, hist_cap);
  double* mean_r = c.scal.p + 1;
  double* mean_z = c.scal.p + 2;
  const bool enclosed = cfg.enclosed_flow != 0;
  DevOp prec = [&](const double* v, double* z) {
    if (enclosed) {
      Fin f;
      f.kind = FIN_MEAN;
      f.i = n_p;
      f.out = mean_r;
      launch_sum(c, n_p, v + n_u, f);
      launch_project(c, n, n_u, v, mean_r, din);
    } else {
      launch_copy(c, n, v, din);
    }
    run();
    if (enclosed) {
      Fin f;
      f.kind = FIN_MEAN;
      f.i = n_p;
      f.out = mean_z;
      launch_sum(c, n_p, dout + n_u, f);
      launch_project(c, n, n_u, dout, mean_z, z);
    } else {
      launch_copy(c, n, dout, z);
    }
  };
  const bool whole = sg && !(getenv("SAG_SOLVE_GRAPH") && !atoi(getenv("SAG_SOLVE_GRAPH")));
  FgmresOut o;
  if (whole) {
    // the whole solve as one CUDA graph: no host synchronisation per Arnoldi step
    const void* key[6] = {bi.d, xo.d, &K0, din, dout, outer.st};
    const bool same = sg->exec && std::equal(key, key + 6, sg->key) &&
                      sg->restart == cfg.restart && sg->max_iters == cfg.max_iters &&
                      sg->tol == cfg.tol && sg->enclosed == cfg.enclosed_flow;
    if (!same) {
      const long long f0 = units_fine ? *units_fine : 0, l0 = units_l1 ? *units_l1 : 0;
      const long long la = c.launches;
      cudaGraph_t g;
      SAG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      try {
        launch_zero(c, n, xo.d);
        fgmres_graph(c, K0, bi.d, xo.d, prec, cfg.tol, cfg.max_iters, cfg.restart, 1e-30, outer,
                     c.scal.p);
      } catch (...) {
        cudaStreamEndCapture(c.stream, &g);
        throw;
      }
      SAG_CUDA(cudaStreamEndCapture(c.stream, &g));
      if (sg->exec) cudaGraphExecDestroy(sg->exec);
      sg->exec = nullptr;
      SAG_CUDA(cudaGraphInstantiate(&sg->exec, g, 0));
      cudaGraphDestroy(g);
      std::copy(key, key + 6, sg->key);
      sg->restart = cfg.restart;
      sg->max_iters = cfg.max_iters;
      sg->tol = cfg.tol;
      sg->enclosed = cfg.enclosed_flow;
      // one application per Arnoldi step was captured `restart` times
      sg->apply_fine = units_fine ? (*units_fine - f0) / std::max(cfg.restart, 1) : 0;
      sg->apply_l1 = units_l1 ? (*units_l1 - l0) / std::max(cfg.restart, 1) : 0;
      if (units_fine) *units_fine = f0;
      if (units_l1) *units_l1 = l0;
      c.launches = la;
    }
    SAG_CUDA(cudaGraphLaunch(sg->exec, c.stream));
    const KHeader hd = read_header(c, outer.st);
    o.iterations = hd.iterations;
    o.converged = hd.converged;
    SAG_CUDA(cudaMemcpyAsync(&o.final_rel, c.scal.p, sizeof(double), cudaMemcpyDeviceToHost,
                             c.stream));
    const int hl = std::min(hd.hist_len, outer.hist_cap);
    o.hist.resize(hl);
    if (hl)
      SAG_CUDA(cudaMemcpyAsync(o.hist.data(),
                               ks_h(outer.st) + (size_t)(cfg.restart + 1) * cfg.restart +
                                   cfg.restart + cfg.restart + (cfg.restart + 1) + cfg.restart,
                               sizeof(double) * hl, cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    if (units_fine) *units_fine += sg->apply_fine * o.iterations;
    if (units_l1) *units_l1 += sg->apply_l1 * o.iterations;
  } else {
    o = fgmres_dev(c, K0, bi.d, xo.d, prec, cfg.tol, cfg.max_iters, cfg.restart, 1e-30, outer);
  }
  xo.finish();
  if (rep) {
    rep->converged = o.converged;
    rep->iterations = o.iterations;
    rep->final_relative_residual = o.final_rel;
    rep->history_len = (int)o.hist.size();
  }
  if (history)
    for (int i = 0; i < history_cap && i < (int)o.hist.size(); ++i) history[i] = o.hist[i];
}

}  // namespace

extern "C" {

int sag_solver_config_default(sag_solver_config* cfg) {
  return guard([&] {
    SAG_NOTNULL(cfg);
    // preconditioner.hpp:20-33
    cfg->variant = SAG_DC_ALL;
    cfg->eta_u = 1.0;
    cfg->eta_p = 1.0;
    cfg->omega0 = 1.0;
    cfg->nu1 = 2;
    cfg->nu2 = 2;
    cfg->gamma = 1;
    cfg->restart = 20;
    cfg->tol = 1e-10;
    cfg->max_iters = 200;
    cfg->enclosed_flow = 0;
    cfg->allow_sv_hoamg = 0;
  });
}

int sag_solver_config_check(const sag_solver_config* cfg) {
  return guard([&] {
    SAG_NOTNULL(cfg);
    check_config(*cfg);
  });
}

int sag_vanka_relax(sag_ctx* ctx, const sag_matrix* k, const sag_vanka* f, double* x,
                    const double* b, int mode, int sweeps, double omega) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k);
    SAG_NOTNULL(f);
    auto& c = ctx->c;
    const int n = k->m.nrows;
    SAG_REQUIRE(f->f.n == n, SAG_DIMENSION_MISMATCH, "vanka_relax: factorization size mismatch");
    InVec bi(c, b, n, 0);
    OutVec xo(c, x, n, 1, true);
    if (sweeps > 0) {
      if (mode == SAG_RELAX_STATIONARY) {
        DevBuf<double> rbuf(n);
        relax_stationary(c, k->m, f->f, rbuf.p, xo.d, bi.d, sweeps, omega, false);
      } else {
        Krylov kr;
        kr.init(n, sweeps, 0);
        relax_kw(c, k->m, f->f, kr, xo.d, bi.d, sweeps, false);
        SAG_CUDA(cudaStreamSynchronize(c.stream));
      }
    }
    xo.finish();
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_fgmres(sag_ctx* ctx, const sag_matrix* a, const double* b, double* x, int prec_kind,
               const void* prec, const sag_fgmres_options* opt, sag_krylov_report* rep,
               double* history, int history_cap) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(opt);
    auto& c = ctx->c;
    const Matrix& A = a->m;
    const int n = A.nrows;
    SAG_REQUIRE(A.ncols == n, SAG_DIMENSION_MISMATCH, "fgmres: operator must be square");
    SAG_REQUIRE(opt->restart >= 1 && opt->max_iters >= 0, SAG_CONFIG_ERROR,
                "fgmres: restart must be >= 1");
    InVec bi(c, b, n, 0);
    OutVec xo(c, x, n, 1, true);
    DevBuf<double> dinv;
    DevOp op;
    switch (prec_kind) {
      case SAG_PREC_IDENTITY:
        op = [&](const double* in, double* out) { launch_copy(c, n, in, out); };
        break;
      case SAG_PREC_VANKA: {
        SAG_NOTNULL(prec);
        const Vanka& f = static_cast<const sag_vanka*>(prec)->f;
        SAG_REQUIRE(f.n == n, SAG_DIMENSION_MISMATCH, "fgmres: preconditioner size mismatch");
        op = [&c, &f](const double* in, double* out) { vanka_apply(c, f, in, out); };
        break;
      }
      case SAG_PREC_JACOBI: {
        SAG_NOTNULL(prec);
        const Matrix& D = static_cast<const sag_matrix*>(prec)->m;
        SAG_REQUIRE(D.nrows == n, SAG_DIMENSION_MISMATCH, "fgmres: preconditioner size mismatch");
        dinv.alloc(n);
        int* bad = reinterpret_cast<int*>(c.scal.p + 8);
        SAG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
        launch_inv_diag(c, D, dinv.p, bad);
        int hb = 0;
        SAG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        SAG_CUDA(cudaStreamSynchronize(c.stream));
        SAG_REQUIRE(!hb, SAG_ZERO_DIAGONAL, "inv_diagonal: zero diagonal");
        op = [&](const double* in, double* out) { launch_mul(c, n, dinv.p, in, out); };
        break;
      }
      case SAG_PREC_DC: {
        SAG_NOTNULL(prec);
        Dc& d = const_cast<sag_dc*>(static_cast<const sag_dc*>(prec))->d;
        require_ready(d);
        SAG_REQUIRE(d.n0 == n, SAG_DIMENSION_MISMATCH, "fgmres: preconditioner size mismatch");
        op = [&c, &d](const double* in, double* out) { dc_apply_dev(c, d, in, out); };
        break;
      }
      case SAG_PREC_UZAWA: {
        SAG_NOTNULL(prec);
        Uzawa& u = const_cast<sag_uzawa*>(static_cast<const sag_uzawa*>(prec))->u;
        SAG_REQUIRE(u.n_x + u.n_y + u.n_p == n, SAG_DIMENSION_MISMATCH,
                    "fgmres: preconditioner size mismatch");
        op = [&c, &u](const double* in, double* out) { uzawa_apply_dev(c, u, in, out); };
        break;
      }
      default:
        throw Error(SAG_CONFIG_ERROR, "fgmres: unknown preconditioner kind");
    }
    Krylov K;
    K.init(n, opt->restart, std::max(history_cap, 1));
    sag_krylov_report r{};
    if (opt->max_iters == 0) {
      // zero iterations: only the initial / final residual (krylov.cpp:26-35, :116)
    }
    FgmresOut o = fgmres_dev(c, A, bi.d, xo.d, op, opt->tol, opt->max_iters, opt->restart,
                             opt->breakdown, K);
    xo.finish();
    r.converged = o.converged;
    r.iterations = o.iterations;
    r.final_relative_residual = o.final_rel;
    r.history_len = o.iterations + 1;
    if (rep) *rep = r;
    if (history)
      for (int i = 0; i < history_cap && i < (int)o.hist.size(); ++i) history[i] = o.hist[i];
  });
}

int sag_dc_create(sag_ctx* ctx, const sag_matrix* k0, int n_x0, int n_y0, int n_p0, int sv,
                  int nlevels, const sag_level_desc* levels, const sag_solver_config* cfg,
                  sag_dc** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k0);
    SAG_NOTNULL(levels);
    SAG_NOTNULL(cfg);
    SAG_NOTNULL(out);
    *out = nullptr;
    auto h = std::make_unique<sag_dc>();
    dc_setup(ctx->c, h->d, &k0->m, n_x0, n_y0, n_p0, sv, nlevels, levels, *cfg);
    *out = h.release();
  });
}

int sag_dc_destroy(sag_dc* d) {
  return guard([&] {
    if (d) cudaDeviceSynchronize();  // its graph and buffers may still be in flight
    delete d;
  });
}

// Every setter that changes what a captured graph computes (parameters baked
// into kernel arguments by value, buffers re-allocated) drops both graphs:
// the standalone apply graph and the whole-solve graph.
static void invalidate_graphs(Dc& d) {
  if (d.ctx) SAG_CUDA(cudaStreamSynchronize(d.ctx->stream));  // nothing in flight uses them
  d.graph_ok = false;
  if (d.solve_graph.exec) {
    cudaGraphExecDestroy(d.solve_graph.exec);
    d.solve_graph.exec = nullptr;
  }
}

int sag_dc_set_coarse_pin(sag_ctx* ctx, sag_dc* h, double level0_norm_inf) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    Dc& d = h->d;
    SAG_REQUIRE(level0_norm_inf >= 0.0, SAG_CONFIG_ERROR, "norm must be non-negative");
    if (!d.cfg.enclosed_flow) return;
    Level& B = d.lv.back();
    // preconditioner.cpp:49-53 with the norm of the hierarchy's finest level
    // supplied by the caller (a rank holding only the coarse levels)
    invalidate_graphs(d);
    d.coarse.setup(ctx->c, *B.K, B.n_x + B.n_y, 1e-12 * level0_norm_inf);
  });
}

int sag_dc_set_parameters(sag_dc* h, double eta_u, double eta_p, double omega0) {
  return guard([&] {
    SAG_NOTNULL(h);
    sag_solver_config c = h->d.cfg;
    c.eta_u = eta_u;
    c.eta_p = eta_p;
    c.omega0 = omega0;
    check_config(c);
    h->d.cfg = c;
    invalidate_graphs(h->d);
  });
}

int sag_dc_set_sv_transfer(sag_dc* h, const sag_matrix* p_dup, const sag_matrix* m_mix, int nsl,
                           const sag_matrix* const* scalar_levels,
                           const sag_matrix* const* scalar_prolongators) {
  return guard([&] {
    SAG_NOTNULL(h);
    SAG_NOTNULL(p_dup);
    SAG_NOTNULL(m_mix);
    SAG_NOTNULL(scalar_levels);
    Dc& d = h->d;
    SAG_REQUIRE(d.sv, SAG_CONFIG_ERROR, "sag_dc_set_sv_transfer: preconditioner is not SV");
    Ctx& c = *d.ctx;
    auto t = std::make_unique<SvTransfer>();
    t->pdup = &p_dup->m;
    t->mmix = &m_mix->m;
    const int n_p1 = d.lv[0].n_p;
    SAG_REQUIRE(t->pdup->nrows == d.n_p0 && t->pdup->ncols == n_p1 && t->mmix->nrows == n_p1 &&
                    t->mmix->ncols == d.n_p0,
                SAG_DIMENSION_MISMATCH, "sag_dc_set_sv_transfer: transfer shapes mismatch");
    scalar_setup(c, t->sh, nsl, scalar_levels, scalar_prolongators, "Mcg hierarchy");
    SAG_REQUIRE(t->sh.n() == n_p1, SAG_DIMENSION_MISMATCH,
                "sag_dc_set_sv_transfer: Mcg size mismatch");
    t->outer.init(n_p1, 20, 202);
    t->rhs.alloc(n_p1);
    t->fail.alloc(1);
    SAG_CUDA(cudaMemsetAsync(t->fail.p, 0, sizeof(int), c.stream));
    sv_project_setup(c, *t);
    invalidate_graphs(d);
    d.svt = std::move(t);
  });
}

int sag_dc_apply(sag_ctx* ctx, sag_dc* h, const double* r, double* z) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    auto& c = ctx->c;
    Dc& d = h->d;
    require_ready(d);
    InVec ri(c, r, d.n0, 0);
    OutVec zo(c, z, d.n0, 1, false);
    launch_copy(c, d.n0, ri.d, d.din.p);
    dc_apply_graph(c, d);
    launch_copy(c, d.n0, d.dout.p, zo.d);
    zo.finish();  // host output: copied back and synchronised; device: stream-ordered
    if (d.sv && !stream_capturing(c)) check_sv_projection(c, d);
  });
}

int sag_dc_vcycle(sag_ctx* ctx, sag_dc* h, const double* b, double* x, int nu1, int nu2) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    auto& c = ctx->c;
    Dc& d = h->d;
    const int n = d.lv[0].n;
    InVec bi(c, b, n, 0);
    OutVec xo(c, x, n, 1, false);
    launch_copy(c, n, bi.d, d.lv[0].b.p);
    SAG_REQUIRE(nu1 <= d.lv[0].kry.m && nu2 <= d.lv[0].kry.m, SAG_CONFIG_ERROR,
                "vcycle: nu exceeds the configured relaxation workspace");
    cycle_level(c, d, 0, nu1, nu2, false);
    launch_copy(c, n, d.lv[0].x.p, xo.d);
    xo.finish();
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_dc_counters(const sag_dc* h, long long* counters) {
  return guard([&] {
    SAG_NOTNULL(h);
    SAG_NOTNULL(counters);
    counters[0] = h->d.fine_units;
    counters[1] = h->d.l1_units;
  });
}

int sag_dc_info(const sag_dc* h, long long* out, int cap) {
  return guard([&] {
    SAG_NOTNULL(h);
    SAG_NOTNULL(out);
    const Dc& d = h->d;
    std::vector<long long> v;
    v.push_back((long long)d.lv.size());
    v.push_back(d.n0);
    for (const auto& L : d.lv) v.push_back(L.n);
    long long fb = d.fine ? d.fine->blob_bytes : 0;
    for (const auto& L : d.lv)
      if (L.vanka) fb += L.vanka->blob_bytes;
    v.push_back(fb);
    v.push_back(d.graph_launches);
    // SV mass projection as one launch: fused, grid levels, CTAs, workers
    const bool fu = d.svt && d.svt->fused;
    v.push_back(fu ? 1 : 0);
    v.push_back(fu ? d.svt->proj.ngl : 0);
    v.push_back(fu ? d.svt->proj.grid : 0);
    v.push_back(fu ? d.svt->proj.workers : 0);
    for (int i = 0; i < cap && i < (int)v.size(); ++i) out[i] = v[i];
  });
}

int sag_dc_proj_trace(sag_ctx* ctx, sag_dc* h, unsigned long long* out, long long cap) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    SAG_NOTNULL(out);
    Dc& d = h->d;
    SAG_REQUIRE(d.svt && d.svt->fused && d.svt->proj.trace, SAG_CONFIG_ERROR,
                "sag_dc_proj_trace: no traced one-launch projection (SAG_PROJ_TRACE=1 at setup)");
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    const long long n = std::min<long long>(cap, 4LL * d.svt->proj.trace_cap);
    SAG_CUDA(cudaMemcpy(out, d.svt->proj.trace, sizeof(unsigned long long) * n,
                        cudaMemcpyDeviceToHost));
  });
}

int sag_solve_stokes(sag_ctx* ctx, sag_dc* h, const double* rhs, double* x,
                     const sag_solver_config* cfg, sag_krylov_report* rep, double* history,
                     int history_cap) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    SAG_NOTNULL(cfg);
    check_config(*cfg);
    auto& c = ctx->c;
    Dc& d = h->d;
    require_ready(d);
    solve_stokes_dev(c, *d.K0, d.n_x0 + d.n_y0, d.n_p0, d.din.p, d.dout.p,
                     [&] { dc_apply_graph(c, d); }, d.outer, *cfg, rhs, x, rep, history,
                     history_cap, &d.solve_graph, &d.fine_units, &d.l1_units);
    if (d.sv) check_sv_projection(c, d);
  });
}

int sag_uzawa_create(sag_ctx* ctx, const sag_matrix* b, int n_x, int n_y, int n_p,
                     const sag_scalar_hierarchy* hx, const sag_scalar_hierarchy* hy,
                     const sag_scalar_hierarchy* hp, const double* sv_element_areas,
                     const sag_solver_config* cfg, sag_uzawa** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(b);
    SAG_NOTNULL(hx);
    SAG_NOTNULL(hy);
    SAG_NOTNULL(cfg);
    SAG_NOTNULL(out);
    check_config(*cfg);
    auto& c = ctx->c;
    auto u = std::make_unique<sag_uzawa>();
    Uzawa& z = u->u;
    z.ctx = &c;
    z.B = &b->m;
    z.n_x = n_x;
    z.n_y = n_y;
    z.n_p = n_p;
    SAG_REQUIRE(z.B->nrows == n_p && z.B->ncols == n_x + n_y, SAG_DIMENSION_MISMATCH,
                "UzawaPreconditioner: B must be n_p x n_u");
    scalar_setup(c, z.hx, hx->nlevels, hx->a, hx->p, "A_x hierarchy");
    scalar_setup(c, z.hy, hy->nlevels, hy->a, hy->p, "A_y hierarchy");
    SAG_REQUIRE(z.hx.n() == n_x && z.hy.n() == n_y, SAG_DIMENSION_MISMATCH,
                "UzawaPreconditioner: velocity hierarchies do not match n_x / n_y");
    if (sv_element_areas) {
      // SV: exact element mass inverse (preconditioner.cpp:191-193)
      SAG_REQUIRE(n_p % 3 == 0, SAG_DIMENSION_MISMATCH,
                  "UzawaPreconditioner: SV pressure count must be 3 per element");
      z.sv_exact_mass = true;
      z.areas.alloc(std::max(n_p / 3, 1));
      SAG_CUDA(cudaMemcpyAsync(z.areas.p, sv_element_areas, sizeof(double) * (n_p / 3),
                               cudaMemcpyDefault, c.stream));
    } else {
      SAG_NOTNULL(hp);
      scalar_setup(c, z.hp, hp->nlevels, hp->a, hp->p, "Mp hierarchy");
      SAG_REQUIRE(z.hp.n() == n_p, SAG_DIMENSION_MISMATCH,
                  "UzawaPreconditioner: pressure mass hierarchy does not match n_p");
      z.pv.alloc(n_p);
    }
    z.t.alloc(std::max(n_p, 1));
    z.din.alloc(n_x + n_y + n_p);
    z.dout.alloc(n_x + n_y + n_p);
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    *out = u.release();
  });
}

int sag_uzawa_destroy(sag_uzawa* u) {
  return guard([&] {
    if (u) cudaDeviceSynchronize();  // its graph and buffers may still be in flight
    delete u;
  });
}

int sag_uzawa_apply(sag_ctx* ctx, sag_uzawa* h, const double* r, double* z) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(h);
    auto& c = ctx->c;
    Uzawa& u = h->u;
    const int n = u.n_x + u.n_y + u.n_p;
    InVec ri(c, r, n, 0);
    OutVec zo(c, z, n, 1, false);
    launch_copy(c, n, ri.d, u.din.p);
    uzawa_apply_graph(c, u);
    launch_copy(c, n, u.dout.p, zo.d);
    zo.finish();
  });
}

int sag_solve_stokes_uzawa(sag_ctx* ctx, const sag_matrix* k0, sag_uzawa* h, const double* rhs,
                           double* x, const sag_solver_config* cfg, sag_krylov_report* rep,
                           double* history, int history_cap) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k0);
    SAG_NOTNULL(h);
    SAG_NOTNULL(cfg);
    check_config(*cfg);
    auto& c = ctx->c;
    Uzawa& u = h->u;
    const int n_u = u.n_x + u.n_y;
    SAG_REQUIRE(k0->m.nrows == n_u + u.n_p && k0->m.ncols == k0->m.nrows, SAG_DIMENSION_MISMATCH,
                "solve_stokes: K0 does not match the preconditioner size");
    solve_stokes_dev(c, k0->m, n_u, u.n_p, u.din.p, u.dout.p, [&] { uzawa_apply_graph(c, u); },
                     h->outer, *cfg, rhs, x, rep, history, history_cap, &u.solve_graph);
  });
}

}  // extern "C"

// ======================================================================
// Partitioned solve: one rank's share of solve_stokes with the
// DC preconditioner over the row/patch partition planned by plan_rank
// (sag_dist_plan.cpp). K0 and the low-order level 0 are distributed (owned
// rows for the SpMV, own Vanka patches with the global partition-of-unity
// weights, forward and reverse halos with the neighbours only); the coarser
// levels are agglomerated (every rank runs the HO-AMG form of the device
// V-cycle on them; the restriction is a partial (P0 on the owned rows)^T r
// summed over the ranks). FGMRES dots and norms are masked partial sums +
// an all-reduce, every Krylov scalar stays on the device, so with a
// capturable communicator (NCCL, or one rank) the whole solve is one CUDA
// graph -- the same conditional-node loop as the single-GPU solve, the
// collectives captured in it. A host-staged communicator (sag_comm_ops:
// gloo, MPI, sockets) runs the same sequence with one status read per
// Arnoldi step.
// ======================================================================

struct sag_comm {
  virtual ~sag_comm() = default;
  int size = 1, rank = 0;
  virtual bool capturable() const = 0;
  // buf (device, n doubles) <- the sum over the ranks, ordered on c.stream
  virtual void allreduce(sag::Ctx& c, double* buf, long long n) = 0;
  struct Msg {
    int peer;
    double* buf;  // device
    long long n;
  };
  virtual void exchange(sag::Ctx& c, const std::vector<Msg>& sends,
                        const std::vector<Msg>& recvs) = 0;
};

namespace sag {
namespace {

// NCCL, resolved at run time (no link dependency): the library already in
// the process (torch's) or the system's libnccl.so.2
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (!loaded) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    SAG_REQUIRE(h, SAG_CUDA_ERROR, "NCCL (libnccl.so.2) not found");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      SAG_REQUIRE(p, SAG_CUDA_ERROR, std::string("NCCL symbol missing: ") + s);
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
  }
  return api;
}

#define SAG_NCCL(x)                                                                        \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      throw ::sag::Error(SAG_CUDA_ERROR, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct NcclComm : sag_comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  void allreduce(Ctx& c, double* buf, long long n) override {
    if (size == 1 || n == 0) return;
    SAG_NCCL(nccl().AllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, comm, c.stream));
  }
  void exchange(Ctx& c, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) override {
    if (sends.empty() && recvs.empty()) return;
    SAG_NCCL(nccl().GroupStart());
    for (const auto& m : sends) SAG_NCCL(nccl().Send(m.buf, (size_t)m.n, ncclDouble, m.peer, comm, c.stream));
    for (const auto& m : recvs) SAG_NCCL(nccl().Recv(m.buf, (size_t)m.n, ncclDouble, m.peer, comm, c.stream));
    SAG_NCCL(nccl().GroupEnd());
  }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
};

// collectives staged through host memory and the caller's callbacks
struct HostComm : sag_comm {
  sag_comm_ops ops{};
  std::vector<double> h;
  bool capturable() const override { return size == 1; }
  void allreduce(Ctx& c, double* buf, long long n) override {
    if (size == 1 || n == 0) return;
    h.resize(n);
    SAG_CUDA(cudaMemcpyAsync(h.data(), buf, 8 * n, cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    SAG_REQUIRE(ops.allreduce_sum(ops.user, h.data(), n) == 0, SAG_ERROR,
                "sag_comm_ops.allreduce_sum failed");
    SAG_CUDA(cudaMemcpyAsync(buf, h.data(), 8 * n, cudaMemcpyHostToDevice, c.stream));
  }
  void exchange(Ctx& c, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) override {
    if (size == 1) return;
    std::vector<std::vector<double>> sb(sends.size()), rb(recvs.size());
    for (size_t i = 0; i < sends.size(); ++i) {
      sb[i].resize(sends[i].n);
      SAG_CUDA(cudaMemcpyAsync(sb[i].data(), sends[i].buf, 8 * sends[i].n, cudaMemcpyDeviceToHost,
                               c.stream));
    }
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int> to(sends.size()), from(recvs.size());
    std::vector<const double*> sp(sends.size());
    std::vector<double*> rp(recvs.size());
    std::vector<long long> sc(sends.size()), rc(recvs.size());
    for (size_t i = 0; i < sends.size(); ++i) {
      to[i] = sends[i].peer;
      sp[i] = sb[i].data();
      sc[i] = sends[i].n;
    }
    for (size_t i = 0; i < recvs.size(); ++i) {
      rb[i].resize(recvs[i].n);
      from[i] = recvs[i].peer;
      rp[i] = rb[i].data();
      rc[i] = recvs[i].n;
    }
    SAG_REQUIRE(ops.exchange(ops.user, (int)sends.size(), to.data(), sp.data(), sc.data(),
                             (int)recvs.size(), from.data(), rp.data(), rc.data()) == 0,
                SAG_ERROR, "sag_comm_ops.exchange failed");
    for (size_t i = 0; i < recvs.size(); ++i)
      SAG_CUDA(cudaMemcpyAsync(recvs[i].buf, rb[i].data(), 8 * recvs[i].n,
                               cudaMemcpyHostToDevice, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));  // rb leaves scope
  }
};

struct Halo {
  std::vector<int> peers;
  std::vector<DevBuf<int>> idx;
  std::vector<DevBuf<double>> buf;
  std::vector<int> cnt;
  void set(const std::map<int, std::vector<int>>& m) {
    for (const auto& [q, ids] : m) {
      peers.push_back(q);
      cnt.push_back((int)ids.size());
      idx.emplace_back(ids.size());
      SAG_CUDA(cudaMemcpy(idx.back().p, ids.data(), 4 * ids.size(), cudaMemcpyHostToDevice));
      buf.emplace_back(ids.size());
    }
  }
  std::vector<sag_comm::Msg> msgs() {
    std::vector<sag_comm::Msg> out;
    for (size_t i = 0; i < peers.size(); ++i) out.push_back({peers[i], buf[i].p, cnt[i]});
    return out;
  }
};

struct DistLevel {
  std::unique_ptr<Matrix> K_int, K_bnd;
  std::unique_ptr<Vanka> f_int, f_bnd;
  DevBuf<double> r, v0, z0, w;
  Krylov kr;  // one rank: the single-GPU fused relaxation
};

std::unique_ptr<Matrix> upload_local(Ctx& c, const LocalCsr& m, int ncols) {
  return matrix_upload(c, m.n, ncols, (long long)m.ci.size(), m.rp.data(), m.ci.data(),
                       m.v.data());
}

std::unique_ptr<Vanka> local_vanka(Ctx& c, const LocalCsr& ext, const LocalPatches& p, int n_u,
                                   const std::vector<double>& w) {
  if (p.count() == 0) return nullptr;
  auto K = upload_local(c, ext, ext.n);
  DevBuf<int> pptr(p.pptr.size()), pidx(std::max<size_t>(p.pidx.size(), 1)),
      vptr(p.vptr.size()), vidx(std::max<size_t>(p.vidx.size(), 1)), nx(p.nx.size());
  auto up = [&](DevBuf<int>& d, const std::vector<int>& h) {
    if (!h.empty()) SAG_CUDA(cudaMemcpy(d.p, h.data(), 4 * h.size(), cudaMemcpyHostToDevice));
  };
  up(pptr, p.pptr);
  up(pidx, p.pidx);
  up(vptr, p.vptr);
  up(vidx, p.vidx);
  up(nx, p.nx);
  auto pt = patches_from_lists(c, p.count(), pptr.p, pidx.p, vptr.p, vidx.p, nx.p);
  auto f = factor_patches_dev(c, *K, *pt, n_u);
  SAG_CUDA(cudaMemcpy(f->w.p, w.data(), 8 * w.size(), cudaMemcpyHostToDevice));
  f->w_ext = true;
  return f;
}

}  // namespace
}  // namespace sag

struct sag_dist {
  sag::Ctx* c = nullptr;
  sag_comm* comm = nullptr;
  sag_solver_config cfg{};
  int nl = 0, n_u_loc = 0, n_p = 0, n1 = 0, n_own = 0, npatch = 0;
  std::vector<long long> l2g;
  std::vector<unsigned char> owned;
  sag::DevBuf<unsigned char> mask;
  sag::DevBuf<double> ones;
  sag::Halo fs, fr, rs, rr;
  sag::DistLevel k0, l0;
  std::unique_ptr<sag::Matrix> P, R;
  std::vector<sag_matrix*> coarse_mats;
  sag_dc* coarse = nullptr;
  sag::DevBuf<double> rc, xc;
  sag::Krylov outer;
  sag::DevBuf<double> din, dout, t, b0, x0, gam_rc, gam_e, sc;
  cudaGraphExec_t graph = nullptr;
  const void* gkey[2] = {nullptr, nullptr};
  ~sag_dist() {
    if (graph) cudaGraphExecDestroy(graph);
    if (coarse) sag_dc_destroy(coarse);
    for (auto* m : coarse_mats) sag_matrix_destroy(m);
  }
};

namespace sag {
namespace {

using Dist = sag_dist;

void halo_fwd(Ctx& c, Dist& d, double* x) {
  for (size_t i = 0; i < d.fs.peers.size(); ++i)
    launch_gather_idx(c, d.fs.cnt[i], d.fs.idx[i].p, x, d.fs.buf[i].p);
  d.comm->exchange(c, d.fs.msgs(), d.fr.msgs());
  for (size_t i = 0; i < d.fr.peers.size(); ++i)
    launch_scatter_idx(c, d.fr.cnt[i], d.fr.idx[i].p, d.fr.buf[i].p, x, 0);
}

// partial sums at ghosts to their owners, added in rank order
void halo_rev(Ctx& c, Dist& d, double* z) {
  for (size_t i = 0; i < d.rs.peers.size(); ++i)
    launch_gather_idx(c, d.rs.cnt[i], d.rs.idx[i].p, z, d.rs.buf[i].p);
  d.comm->exchange(c, d.rs.msgs(), d.rr.msgs());
  for (size_t i = 0; i < d.rr.peers.size(); ++i)
    launch_scatter_idx(c, d.rr.cnt[i], d.rr.idx[i].p, d.rr.buf[i].p, z, 1);
}

// *out = global (a, b) over the owned entries
void mdot(Ctx& c, Dist& d, const double* a, const double* b, double* out) {
  launch_dot_mask(c, d.nl, a, b, d.mask.p, out);
  d.comm->allreduce(c, out, 1);
}

// y = K x (Store), aux - K x (Resid; y may be aux) or y + K x (Add) on the owned rows
void apply_op(Ctx& c, Dist& d, DistLevel& L, double* x, double* y, Epi e,
              const double* aux = nullptr) {
  halo_fwd(c, d, x);
  SpmvArgs a;
  a.b = aux;
  launch_spmv(c, *L.K_int, x, y, e, a);
  if (L.K_bnd) {
    if (e == Epi::Resid) {
      SpmvArgs b;
      b.b = y;
      launch_spmv(c, *L.K_bnd, x, y, Epi::Resid, b);
    } else {
      launch_spmv(c, *L.K_bnd, x, y, Epi::Add);
    }
  }
}

// z = apply_vanka(v) over the partition (vanka.cpp:151-184)
void vanka(Ctx& c, Dist& d, DistLevel& L, double* v, double* z) {
  halo_fwd(c, d, v);
  if (L.f_int)
    vanka_apply(c, *L.f_int, v, z);
  else
    launch_zero(c, d.nl, z);
  if (L.f_bnd) vanka_apply_stationary(c, *L.f_bnd, v, z, 1.0);
  halo_rev(c, d, z);
}

// vanka_relax, Krylov-wrapped with nu = 1 (vanka.cpp:199-208): the one-step
// FGMRES on device scalars
void relax1(Ctx& c, Dist& d, DistLevel& L, double* x, const double* b, bool x_zero) {
  if (d.comm->size == 1 && L.f_int && !L.f_bnd && !L.K_bnd) {
    // one rank (no ghosts): the single-GPU fused kernels, same operations
    relax_kw(c, *L.K_int, *L.f_int, L.kr, x, b, 1, x_zero);
    return;
  }
  double* s = d.sc.p;
  const double* r = b;
  if (!x_zero) {
    apply_op(c, d, L, x, L.r.p, Epi::Resid, b);
    r = L.r.p;
  }
  mdot(c, d, r, r, s + 0);                          // ||r||^2
  launch_div_dev(c, d.nl, r, s + 0, 1, L.v0.p);     // v_0 = r / ||r||
  vanka(c, d, L, L.v0.p, L.z0.p);                   // z_0 = M v_0
  apply_op(c, d, L, L.z0.p, L.w.p, Epi::Store);     // w = K z_0
  mdot(c, d, L.w.p, L.v0.p, s + 1);                 // h_00
  launch_axpy_dev(c, d.nl, s + 1, -1.0, L.v0.p, L.w.p);
  mdot(c, d, L.w.p, L.w.p, s + 2);                  // h_10^2
  launch_fgmres1_coef(c, s + 0, s + 1, s + 2, s + 3);
  if (x_zero) launch_zero(c, d.nl, x);
  launch_axpy_dev(c, d.nl, s + 3, 1.0, L.z0.p, x);  // x += y_0 z_0
}

// MonolithicSolver::cycle_level on level 0 (preconditioner.cpp:57-81)
void cycle0(Ctx& c, Dist& d, double* b, double* x, bool skip_finest) {
  const auto& cf = d.cfg;
  const bool relax = !skip_finest;
  const double* r = b;
  if (relax && cf.nu1 > 0) {
    relax1(c, d, d.l0, x, b, true);
    if (d.l0.kr.st)  // one rank: r = b - y_0 w (= b - K x by linearity, as cycle_level)
      launch_lin_resid(c, d.nl, d.nl, 1.0, 1.0, b, d.l0.kr.w.p, d.l0.kr.st, d.l0.r.p);
    else
      apply_op(c, d, d.l0, x, d.l0.r.p, Epi::Resid, b);
    r = d.l0.r.p;
  } else {
    launch_zero(c, d.nl, x);
  }
  launch_spmv(c, *d.R, r, d.rc.p, Epi::Store);      // partial restriction (owned rows)
  d.comm->allreduce(c, d.rc.p, d.n1);
  dc_apply_dev(c, d.coarse->d, d.rc.p, d.xc.p);      // agglomerated V-cycle below level 0
  launch_spmv(c, *d.P, d.xc.p, x, Epi::Add);         // x += P x_c on the owned rows
  if (relax && cf.nu2 > 0) relax1(c, d, d.l0, x, b, false);
}

// DCPreconditioner::apply (preconditioner.cpp:114-153), Taylor-Hood
void dist_dc_apply(Ctx& c, Dist& d, double* r, double* z) {
  const auto& cf = d.cfg;
  const bool relax_fine = cf.variant != SAG_DC_LO;
  double* x = z;
  const double* r1 = r;
  if (relax_fine && cf.nu1 > 0 && d.k0.kr.st) {
    // one rank: the residual by linearity fused with the eta weighting, as
    // dc_apply_dev
    relax1(c, d, d.k0, x, r, true);
    launch_lin_resid(c, d.nl, d.n_u_loc, cf.eta_u, cf.eta_p, r, d.k0.kr.w.p, d.k0.kr.st,
                     d.b0.p);
  } else {
    if (relax_fine && cf.nu1 > 0) {
      relax1(c, d, d.k0, x, r, true);
      apply_op(c, d, d.k0, x, d.t.p, Epi::Resid, r);
      r1 = d.t.p;
    } else {
      launch_zero(c, d.nl, x);
    }
    launch_eta(c, d.nl, d.n_u_loc, cf.eta_u, cf.eta_p, r1, d.b0.p);  // transfer.cpp:127-135
  }
  const bool skip = cf.variant == SAG_DC_HO;
  if (cf.gamma <= 1) {
    cycle0(c, d, d.b0.p, d.x0.p, skip);
    launch_add(c, d.nl, x, d.x0.p);
  } else {
    launch_copy(c, d.nl, d.b0.p, d.gam_rc.p);
    launch_zero(c, d.nl, d.gam_e.p);
    for (int g = 0; g < cf.gamma; ++g) {
      if (g > 0)
        apply_op(c, d, d.l0, d.gam_e.p, d.b0.p, Epi::Resid, d.gam_rc.p);
      else
        launch_copy(c, d.nl, d.gam_rc.p, d.b0.p);
      cycle0(c, d, d.b0.p, d.x0.p, skip);
      launch_add(c, d.nl, d.gam_e.p, d.x0.p);
    }
    launch_add(c, d.nl, x, d.gam_e.p);
  }
  if (relax_fine && cf.nu2 > 0) relax1(c, d, d.k0, x, r, false);
}

// y = x with the global pressure mean removed (preconditioner.cpp:235-240)
void dist_project(Ctx& c, Dist& d, const double* x, double* y, double* s) {
  const int nu = d.n_u_loc;
  if (d.comm->size == 1) {  // preconditioner.cpp:235-240 as the single-GPU path
    Fin f;
    f.kind = FIN_MEAN;
    f.i = d.nl - nu;
    f.out = s;
    launch_sum(c, d.nl - nu, x + nu, f);
    launch_project(c, d.nl, nu, x, s, y);
    return;
  }
  launch_dot_mask(c, d.nl - nu, x + nu, d.ones.p + nu, d.mask.p + nu, s);
  d.comm->allreduce(c, s, 1);
  if (y != x) launch_copy(c, nu, x, y);
  launch_sub_mean(c, d.nl - nu, x + nu, s, (double)d.n_p, y + nu);
}

void dist_prec(Ctx& c, Dist& d, const double* v, double* z) {
  if (d.cfg.enclosed_flow) {
    dist_project(c, d, v, d.din.p, d.sc.p + 4);
    dist_dc_apply(c, d, d.din.p, d.dout.p);
    dist_project(c, d, d.dout.p, z, d.sc.p + 5);
  } else {
    launch_copy(c, d.nl, v, d.din.p);
    dist_dc_apply(c, d, d.din.p, z);
  }
}

// the fgmres of krylov.cpp:17-121 over the partition, every scalar on the
// device: graph = conditional nodes (a capturing caller), else one status
// read per Arnoldi step
void dist_fgmres(Ctx& c, Dist& d, const double* b, double* x, bool graph) {
  Krylov& K = d.outer;
  const auto& cf = d.cfg;
  const int m = cf.restart, n = d.nl;
  double* s = d.sc.p + 8;
  SAG_CUDA(cudaMemsetAsync(c.ticket.p, 0, sizeof(unsigned) * c.ticket.n, c.stream));
  launch_kinit(c, K.st, m, cf.tol, 1e-30, K.hist_cap, false);
  launch_zero(c, n, x);
  auto fin = [&](FinKind k, int i, int j, double* out = nullptr) {
    Fin f;
    f.kind = k;
    f.st = K.st;
    f.i = i;
    f.j = j;
    f.out = out;
    return f;
  };
  // one rank (no ghosts): the single-GPU fused reductions, same operations
  const bool one = d.comm->size == 1 && !d.k0.K_bnd;
  if (one) {
    launch_ssq(c, n, b, fin(FIN_REF, 0, 0));
  } else {
    mdot(c, d, b, b, s);
    launch_fin_from(c, fin(FIN_REF, 0, 0), s);                 // ref = ||b||
  }
  auto residual = [&](int hist) {
    if (one) {
      SpmvArgs a;
      a.b = b;
      a.fin = fin(FIN_BETA, hist, 0);
      launch_spmv(c, *d.k0.K_int, x, K.r.p, Epi::ResidSsq, a);
      return;
    }
    apply_op(c, d, d.k0, x, K.r.p, Epi::Resid, b);
    mdot(c, d, K.r.p, K.r.p, s + 1);
    launch_fin_from(c, fin(FIN_BETA, hist, 0), s + 1);         // beta, g, stop
  };
  residual(2);                                                 // history[0]
  auto step = [&](int j) {
    dist_prec(c, d, K.v(j), K.z(j));
    if (one) {
      arnoldi_step(c, *d.k0.K_int, K, m, j, K.stop());
      return;
    }
    apply_op(c, d, d.k0, K.z(j), K.w.p, Epi::Store);
    for (int i = 0; i <= j; ++i) {                             // MGS (krylov.cpp:63-67)
      mdot(c, d, K.w.p, K.v(i), s + 2 + i);
      launch_fin_from(c, fin(FIN_H, i, j), s + 2 + i);
      launch_axpy_dev(c, n, K.h(m, i, j), -1.0, K.v(i), K.w.p);
    }
    mdot(c, d, K.w.p, K.w.p, s + 2 + j + 1);
    launch_fin_from(c, fin(FIN_ARNOLDI, 0, j), s + 2 + j + 1);  // Givens, residual estimate
    launch_div(c, n, K.w.p, K.wnorm(), K.v(j + 1), K.stop(), K.breakdown());
  };
  auto cycle_body = [&] {
    residual(0);                                               // restart (krylov.cpp:43-53)
    launch_div(c, n, K.r.p, K.beta(), K.v(0), K.stop());
  };
  if (graph) {
    auto set = [&](int mode) {
      return [&, mode](cudaGraphConditionalHandle h) {
        cond_set_kernel<<<1, 1, 0, c.stream>>>(h, K.st, mode, cf.max_iters);
        SAG_LAUNCHED(c);
      };
    };
    cond_node(c, cudaGraphCondTypeWhile, set(0), [&](cudaGraphConditionalHandle hw) {
      cycle_body();
      for (int j = 0; j < m; ++j)
        cond_node(c, cudaGraphCondTypeIf, set(1), [&](cudaGraphConditionalHandle) { step(j); });
      launch_backsub(c, K.st);
      launch_update(c, n, x, K.Z.p, (size_t)n, K.st, false);
      cond_set_kernel<<<1, 1, 0, c.stream>>>(hw, K.st, 0, cf.max_iters);
      SAG_LAUNCHED(c);
    });
  } else {
    KHeader hd = read_header(c, K.st);
    while (!hd.converged && hd.iterations < cf.max_iters) {
      cycle_body();
      hd = read_header(c, K.st);
      if (hd.stop) break;
      for (int j = 0; j < m && hd.iterations < cf.max_iters; ++j) {
        step(j);
        hd = read_header(c, K.st);
        if (hd.stop) break;
      }
      launch_backsub(c, K.st);
      launch_update(c, n, x, K.Z.p, (size_t)n, K.st, false);
      hd = read_header(c, K.st);
    }
  }
  if (one) {                                                   // final true residual
    SpmvArgs a;
    a.b = b;
    a.fin = fin(FIN_FINAL, 0, 0, c.scal.p);
    launch_spmv(c, *d.k0.K_int, x, K.r.p, Epi::ResidSsq, a);
    return;
  }
  apply_op(c, d, d.k0, x, K.r.p, Epi::Resid, b);
  mdot(c, d, K.r.p, K.r.p, s + 1);
  launch_fin_from(c, fin(FIN_FINAL, 0, 0, c.scal.p), s + 1);
}

void check_status(int st) {
  if (st != SAG_OK) throw Error(st, sag_last_error());
}

double host_norm_inf(const HostCsr& m) {  // norm_inf (sparse.cpp:229-237)
  double best = 0.0;
  for (int r = 0; r < m.nrows; ++r) {
    double s = 0.0;
    for (int k = m.rp[r]; k < m.rp[r + 1]; ++k) s += std::abs(m.v[k]);
    best = std::max(best, s);
  }
  return best;
}

HostCsr host_csr(const sag_csr& m) {
  HostCsr h;
  h.nrows = m.nrows;
  h.ncols = m.ncols;
  h.rp = m.row_offsets;
  h.ci = m.col_indices;
  h.v = m.values;
  return h;
}

}  // namespace
}  // namespace sag

using namespace sag;

struct sag_plan {
  RankPlan p;
};

extern "C" {

int sag_nccl_unique_id(unsigned char* id) {
  return guard([&] {
    SAG_NOTNULL(id);
    ncclUniqueId u;
    SAG_NCCL(nccl().GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof(u));
  });
}

int sag_comm_create_nccl(sag_ctx* ctx, int nranks, int rank, const unsigned char* id,
                         sag_comm** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(id);
    SAG_NOTNULL(out);
    SAG_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, SAG_CONFIG_ERROR,
                "sag_comm_create_nccl: rank out of range");
    auto cm = std::make_unique<NcclComm>();
    cm->size = nranks;
    cm->rank = rank;
    if (nranks > 1) {
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof(u));
      SAG_CUDA(cudaSetDevice(ctx->c.device));
      SAG_NCCL(nccl().CommInitRank(&cm->comm, nranks, u, rank));
    }
    *out = cm.release();
  });
}

int sag_comm_create_host(int nranks, int rank, const sag_comm_ops* ops, sag_comm** out) {
  return guard([&] {
    SAG_NOTNULL(out);
    SAG_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, SAG_CONFIG_ERROR,
                "sag_comm_create_host: rank out of range");
    SAG_REQUIRE(nranks == 1 || (ops && ops->allreduce_sum && ops->exchange), SAG_INVALID_ARGUMENT,
                "sag_comm_create_host: missing callbacks");
    auto cm = std::make_unique<HostComm>();
    cm->size = nranks;
    cm->rank = rank;
    if (ops) cm->ops = *ops;
    *out = cm.release();
  });
}

int sag_comm_allreduce(sag_ctx* ctx, sag_comm* comm, double* buf, long long n) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(comm);
    SAG_REQUIRE(is_device_ptr(buf) || n == 0, SAG_INVALID_ARGUMENT,
                "sag_comm_allreduce: device buffer expected");
    comm->allreduce(ctx->c, buf, n);
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sag_comm_destroy(sag_comm* comm) {
  return guard([&] { delete comm; });
}

int sag_plan_create(int nranks, int rank, const sag_csr* k0, const sag_csr* l0, const sag_csr* p0,
                    int n_x, int n_y, int n_p, sag_plan** out) {
  return guard([&] {
    SAG_NOTNULL(k0);
    SAG_NOTNULL(l0);
    SAG_NOTNULL(out);
    const HostCsr hk = host_csr(*k0), hl = host_csr(*l0);
    HostCsr hp;
    if (p0) hp = host_csr(*p0);
    auto pl = std::make_unique<sag_plan>();
    try {
      pl->p = plan_rank(nranks, rank, hk, hl, p0 ? &hp : nullptr, n_x, n_y, n_p);
    } catch (const std::runtime_error& e) {
      throw Error(SAG_CONFIG_ERROR, e.what());
    }
    *out = pl.release();
  });
}

int sag_plan_destroy(sag_plan* plan) {
  return guard([&] { delete plan; });
}

int sag_plan_array(const sag_plan* plan, int which, int peer, void* out, long long* count) {
  return guard([&] {
    SAG_NOTNULL(plan);
    SAG_NOTNULL(count);
    const RankPlan& p = plan->p;
    auto give = [&](const auto& v) {
      using T = typename std::decay_t<decltype(v)>::value_type;
      *count = (long long)v.size();
      if (out && !v.empty()) std::memcpy(out, v.data(), sizeof(T) * v.size());
    };
    auto halo = [&](const std::map<int, std::vector<int>>& m) {
      static const std::vector<int> none;
      auto it = m.find(peer);
      give(it == m.end() ? none : it->second);
    };
    const LocalLevel& L = (which / 100) == 1 ? p.l0 : p.k0;
    switch (which % 100) {
      case SAG_PLAN_L2G: give(p.l2g); break;
      case SAG_PLAN_OWNED: give(p.owned); break;
      case SAG_PLAN_FWD_SEND: halo(p.fwd_send); break;
      case SAG_PLAN_FWD_RECV: halo(p.fwd_recv); break;
      case SAG_PLAN_REV_SEND: halo(p.rev_send); break;
      case SAG_PLAN_REV_RECV: halo(p.rev_recv); break;
      case SAG_PLAN_EXT_RP: give(L.ext.rp); break;
      case SAG_PLAN_EXT_CI: give(L.ext.ci); break;
      case SAG_PLAN_EXT_V: give(L.ext.v); break;
      case SAG_PLAN_INT_PVIDX: give(L.p_int.vidx); break;
      case SAG_PLAN_BND_PVIDX: give(L.p_bnd.vidx); break;
      case SAG_PLAN_WEIGHTS: give(L.w); break;
      case SAG_PLAN_P_RP: give(p.p_own.rp); break;
      case SAG_PLAN_P_CI: give(p.p_own.ci); break;
      case SAG_PLAN_INFO: {
        const std::vector<long long> info = {p.nl(), p.n_u_loc, p.patch_lo, p.patch_hi, p.n1,
                                             (long long)p.fwd_send.size(),
                                             (long long)p.fwd_recv.size()};
        give(info);
        break;
      }
      default:
        throw Error(SAG_INVALID_ARGUMENT, "sag_plan_array: unknown array");
    }
  });
}

int sag_dist_create(sag_ctx* ctx, sag_comm* comm, const sag_csr* k0, int n_x, int n_y, int n_p,
                    int nlevels, const sag_csr* levels, const sag_csr* prolongators,
                    const int* level_nxyz, const sag_solver_config* cfg, sag_dist** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(comm);
    SAG_NOTNULL(k0);
    SAG_NOTNULL(levels);
    SAG_NOTNULL(level_nxyz);
    SAG_NOTNULL(cfg);
    SAG_NOTNULL(out);
    check_config(*cfg);
    SAG_REQUIRE(cfg->variant == SAG_DC_ALL || cfg->variant == SAG_DC_LO ||
                    cfg->variant == SAG_DC_HO,
                SAG_CONFIG_ERROR, "sag_dist_create: DC-all / DC-LO / DC-HO only");
    SAG_REQUIRE(cfg->nu1 <= 1 && cfg->nu2 <= 1, SAG_CONFIG_ERROR,
                "sag_dist_create: nu1, nu2 <= 1 (one-step Krylov-wrapped relaxation)");
    SAG_REQUIRE(nlevels >= 2 && prolongators, SAG_CONFIG_ERROR,
                "sag_dist_create: a hierarchy of at least two levels");
    Ctx& c = ctx->c;
    const HostCsr hk = host_csr(*k0), hl = host_csr(levels[0]), hp = host_csr(prolongators[0]);
    RankPlan pl;
    try {
      pl = plan_rank(comm->size, comm->rank, hk, hl, &hp, n_x, n_y, n_p);
    } catch (const std::runtime_error& e) {
      throw Error(SAG_CONFIG_ERROR, e.what());
    }
    auto d = std::make_unique<sag_dist>();
    d->c = &c;
    d->comm = comm;
    d->cfg = *cfg;
    d->nl = pl.nl();
    d->n_u_loc = pl.n_u_loc;
    d->n_p = n_p;
    d->n1 = pl.n1;
    d->l2g = pl.l2g;
    d->owned = pl.owned;
    d->npatch = (int)(pl.patch_hi - pl.patch_lo);
    for (unsigned char o : pl.owned) d->n_own += o;
    const int nl = d->nl;
    d->mask.alloc(nl);
    SAG_CUDA(cudaMemcpy(d->mask.p, pl.owned.data(), nl, cudaMemcpyHostToDevice));
    d->ones.alloc(nl);
    {
      std::vector<double> o(nl, 1.0);
      SAG_CUDA(cudaMemcpy(d->ones.p, o.data(), 8 * (size_t)nl, cudaMemcpyHostToDevice));
    }
    d->fs.set(pl.fwd_send);
    d->fr.set(pl.fwd_recv);
    d->rs.set(pl.rev_send);
    d->rr.set(pl.rev_recv);
    const int n_u_loc = pl.n_u_loc;
    auto level = [&](DistLevel& L, const LocalLevel& ll) {
      L.K_int = upload_local(c, ll.rows_int, nl);
      if (!ll.rows_bnd.ci.empty()) L.K_bnd = upload_local(c, ll.rows_bnd, nl);
      L.f_int = local_vanka(c, ll.ext, ll.p_int, n_u_loc, ll.w);
      L.f_bnd = local_vanka(c, ll.ext, ll.p_bnd, n_u_loc, ll.w);
      L.r.alloc(nl);
      L.v0.alloc(nl);
      L.z0.alloc(nl);
      L.w.alloc(nl);
      if (comm->size == 1) L.kr.init(nl, 1, 4);
    };
    level(d->k0, pl.k0);
    level(d->l0, pl.l0);
    d->P = upload_local(c, pl.p_own, pl.n1);
    d->R = transpose_dev(c, *d->P);
    // agglomerated levels 1..: the HO-AMG form of the device V-cycle, the
    // coarsest pinned with the norm of level 0 (preconditioner.cpp:49-53)
    std::vector<sag_level_desc> lv(nlevels - 1);
    for (int l = 1; l < nlevels; ++l) {
      sag_matrix* k = nullptr;
      check_status(sag_matrix_create(ctx, levels[l].nrows, levels[l].ncols,
                                     levels[l].row_offsets[levels[l].nrows],
                                     levels[l].row_offsets, levels[l].col_indices,
                                     levels[l].values, &k));
      d->coarse_mats.push_back(k);
      lv[l - 1].k = k;
      lv[l - 1].p = nullptr;
      if (l + 1 < nlevels) {
        sag_matrix* p = nullptr;
        const sag_csr& pm = prolongators[l];
        check_status(sag_matrix_create(ctx, pm.nrows, pm.ncols, pm.row_offsets[pm.nrows],
                                       pm.row_offsets, pm.col_indices, pm.values, &p));
        d->coarse_mats.push_back(p);
        lv[l - 1].p = p;
      }
      lv[l - 1].n_x = level_nxyz[3 * l];
      lv[l - 1].n_y = level_nxyz[3 * l + 1];
      lv[l - 1].n_p = level_nxyz[3 * l + 2];
    }
    sag_solver_config ccfg = *cfg;
    ccfg.variant = SAG_HOAMG;
    check_status(sag_dc_create(ctx, lv[0].k, lv[0].n_x, lv[0].n_y, lv[0].n_p, 0, nlevels - 1,
                               lv.data(), &ccfg, &d->coarse));
    if (cfg->enclosed_flow)
      check_status(sag_dc_set_coarse_pin(ctx, d->coarse, host_norm_inf(hl)));
    d->rc.alloc(pl.n1);
    d->xc.alloc(pl.n1);
    d->outer.init(nl, cfg->restart, cfg->max_iters + 2);
    for (auto* b : {&d->din, &d->dout, &d->t, &d->b0, &d->x0, &d->gam_rc, &d->gam_e})
      b->alloc(nl);
    d->sc.alloc(64 + 2 * (size_t)cfg->restart);
    SAG_CUDA(cudaDeviceSynchronize());
    *out = d.release();
  });
}

int sag_dist_destroy(sag_dist* d) {
  return guard([&] {
    if (d) cudaDeviceSynchronize();
    delete d;
  });
}

int sag_dist_info(const sag_dist* d, long long* out) {
  return guard([&] {
    SAG_NOTNULL(d);
    SAG_NOTNULL(out);
    out[0] = d->nl;
    out[1] = d->n_own;
    out[2] = d->nl - d->n_own;
    out[3] = (long long)std::max(d->fs.peers.size(), d->fr.peers.size());
    out[4] = d->npatch;
    out[5] = d->n1;
    out[6] = d->n_u_loc;
  });
}

int sag_dist_local_dofs(const sag_dist* d, long long* l2g, unsigned char* owned) {
  return guard([&] {
    SAG_NOTNULL(d);
    if (l2g) std::memcpy(l2g, d->l2g.data(), 8 * d->l2g.size());
    if (owned) std::memcpy(owned, d->owned.data(), d->owned.size());
  });
}

int sag_dist_step(sag_ctx* ctx, sag_dist* d, const double* x, double* delta, double* y) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(d);
    Ctx& c = ctx->c;
    const int nl = d->nl;
    InVec xi(c, x, nl, 0);
    double* xw = c.stage_buf(3, nl);  // ghosts are overwritten by the halo
    launch_copy(c, nl, xi.d, xw);
    OutVec dv(c, delta, nl, 1, false), yv(c, y, nl, 2, false);
    DistLevel& L = d->k0;
    halo_fwd(c, *d, xw);
    if (L.f_int)
      vanka_apply(c, *L.f_int, xw, dv.d);
    else
      launch_zero(c, nl, dv.d);
    launch_spmv(c, *L.K_int, xw, yv.d, Epi::Store);
    if (L.f_bnd) vanka_apply_stationary(c, *L.f_bnd, xw, dv.d, 1.0);
    if (L.K_bnd) launch_spmv(c, *L.K_bnd, xw, yv.d, Epi::Add);
    halo_rev(c, *d, dv.d);
    dv.finish();
    yv.finish();
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_dist_solve_stokes(sag_ctx* ctx, sag_dist* d, const double* rhs, double* x,
                          sag_krylov_report* rep, double* history, int history_cap) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(d);
    Ctx& c = ctx->c;
    const int nl = d->nl;
    InVec bi(c, rhs, nl, 0);
    OutVec xo(c, x, nl, 1, false);
    const bool graph = d->comm->capturable() &&
                       !(getenv("SAG_SOLVE_GRAPH") && !atoi(getenv("SAG_SOLVE_GRAPH")));
    if (graph) {
      const void* key[2] = {bi.d, xo.d};
      if (!d->graph || key[0] != d->gkey[0] || key[1] != d->gkey[1]) {
        if (d->graph) cudaGraphExecDestroy(d->graph);
        d->graph = nullptr;
        cudaGraph_t g;
        const long long la = c.launches;
        SAG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        try {
          dist_fgmres(c, *d, bi.d, xo.d, true);
        } catch (...) {
          cudaStreamEndCapture(c.stream, &g);
          throw;
        }
        SAG_CUDA(cudaStreamEndCapture(c.stream, &g));
        SAG_CUDA(cudaGraphInstantiate(&d->graph, g, 0));
        cudaGraphDestroy(g);
        d->gkey[0] = key[0];
        d->gkey[1] = key[1];
        c.launches = la;
      }
      SAG_CUDA(cudaGraphLaunch(d->graph, c.stream));
    } else {
      dist_fgmres(c, *d, bi.d, xo.d, false);
    }
    const KHeader hd = read_header(c, d->outer.st);
    if (rep) {
      rep->converged = hd.converged;
      rep->iterations = hd.iterations;
      SAG_CUDA(cudaMemcpyAsync(&rep->final_relative_residual, c.scal.p, sizeof(double),
                               cudaMemcpyDeviceToHost, c.stream));
    }
    const int m = d->cfg.restart;
    const int hl = std::min({hd.hist_len, d->outer.hist_cap, history ? history_cap : 0});
    if (history && hl > 0)
      SAG_CUDA(cudaMemcpyAsync(history, ks_h(d->outer.st) + (size_t)(m + 1) * m + m + m + (m + 1) + m,
                               sizeof(double) * hl, cudaMemcpyDeviceToHost, c.stream));
    if (rep) rep->history_len = hd.hist_len;
    xo.finish();
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
