// libsag core: context, CSR upload/validation, SpMV with fused epilogues,
// deterministic BLAS-1 reductions, Krylov scalar finishers, transpose, and the
// C-ABI for those pieces (include/sag.h).
//
// Reference behaviour restated here:
//   spmv            sparse.cpp:78-91   (row sums; here G lanes per row + shuffle tree)
//   norm2 / dot     sparse.cpp:217-227 (here fixed-order two-stage reductions)
//   norm_inf        sparse.cpp:229-237
//   transpose       sparse.cpp:93-111  (rows of P^T in ascending order)
//   FGMRES scalars  krylov.cpp:42-110  (finishers below)
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.cuh"
#include "tma.cuh"

namespace sag {

namespace cg = cooperative_groups;

// ------------------------------------------------------------ finishers --

__device__ void apply_fin(const Fin& f, double tot) {
  KState* st = f.st;
  switch (f.kind) {
    case FIN_STORE:
      *f.out = tot;
      break;
    case FIN_SQRT:
      *f.out = sqrt(tot);
      break;
    case FIN_MEAN:
      *f.out = tot / (double)f.i;
      break;
    case FIN_REF: {
      const double b = sqrt(tot);
      st->ref = b > 0.0 ? b : 1.0;
      break;
    }
    case FIN_BETA: {
      // f.i bit0: also set ref (inner solve: ||b|| == ||r|| for x0 = 0)
      // f.i bit1: push the residual to the history
      const double beta = sqrt(tot);
      if (f.i & 4) {
        st->m = f.j;
        st->tol = f.tol;
        st->bd = 1e-30;
        st->iterations = 0;
        st->converged = 0;
        st->hist_len = 0;
        st->hist_cap = 0;
      }
      if (f.i & 1) st->ref = beta > 0.0 ? beta : 1.0;
      // a restart whose ref was never set (a KState fresh from Krylov::init,
      // ref = 0): FIN_REF's own zero-norm rule. Exact for the tol = 0 inner
      // solves (stop iff beta == 0); a caller that needs a tolerance relative
      // to ||b|| must run FIN_REF first (jacobi_fgmres2's post-smoothing keeps
      // the pre-smoothing's ref of the same b).
      if (!(st->ref > 0.0)) st->ref = 1.0;
      st->beta = beta;
      st->rnorm = beta;
      double* g = ks_g(st);
      g[0] = beta;
      for (int i = 1; i <= st->m; ++i) g[i] = 0.0;
      st->jeff = 0;
      st->breakdown = 0;
      st->stop = (beta / st->ref <= st->tol) ? 1 : 0;
      if (st->stop) st->converged = 1;
      if (f.i & 2) {
        if (st->hist_len < st->hist_cap) ks_hist(st)[st->hist_len] = beta;
        st->hist_len++;
      }
      break;
    }
    case FIN_H:
      ks_h(st)[(size_t)f.i * st->m + f.j] = tot;
      break;
    case FIN_ARNOLDI: {
      const int m = st->m, j = f.j;
      double* h = ks_h(st);
      double* cs = ks_cs(st);
      double* sn = ks_sn(st);
      double* g = ks_g(st);
      const double wnorm = sqrt(tot);
      st->wnorm = wnorm;
      h[(size_t)(j + 1) * m + j] = wnorm;
      const int bd = wnorm < st->bd;
      st->breakdown = bd;
      for (int i = 0; i < j; ++i) {
        const double a = h[(size_t)i * m + j], b = h[(size_t)(i + 1) * m + j];
        const double t = cs[i] * a + sn[i] * b;
        h[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
        h[(size_t)i * m + j] = t;
      }
      const double a = h[(size_t)j * m + j], b = h[(size_t)(j + 1) * m + j];
      const double denom = hypot(a, b);
      if (denom > 0.0) {
        cs[j] = a / denom;
        sn[j] = b / denom;
      } else {
        cs[j] = 1.0;
        sn[j] = 0.0;
      }
      h[(size_t)j * m + j] = cs[j] * a + sn[j] * b;
      h[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      st->iterations++;
      const double rn = fabs(g[j + 1]);
      st->rnorm = rn;
      if (st->hist_len < st->hist_cap) ks_hist(st)[st->hist_len] = rn;
      st->hist_len++;
      st->jeff = j + 1;
      const int conv = rn / st->ref <= st->tol;
      if (conv) st->converged = 1;
      if (conv || bd) st->stop = 1;
      break;
    }
    case FIN_FINAL: {
      const double fr = sqrt(tot) / st->ref;
      *f.out = fr;
      if (fr <= st->tol) st->converged = 1;
      break;
    }
    default:
      break;
  }
}

// Block partial -> last block sums partials in order -> finisher.
__device__ __forceinline__ void reduce_finish(double red, const Fin& fin, double* partials,
                                              unsigned* ticket) {
  __shared__ double sh[32];
  const double bs = block_sum(red, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
  if (last_block(ticket)) {
    const double tot = sum_partials(partials, gridDim.x, sh);
    if (threadIdx.x == 0) {
      apply_fin(fin, tot);
      *ticket = 0u;
    }
  }
}

// Epilogue operand of a row (loaded before the row product so its latency
// overlaps the gathers) and the fused epilogue itself.
template <Epi E>
__device__ __forceinline__ double spmv_pre(const SpmvArgs& a, const double* y, int row, bool lead) {
  if (!lead) return 0.0;
  if constexpr (E == Epi::StoreDot) return __ldg(a.dotv + row);
  if constexpr (E == Epi::Resid || E == Epi::ResidEta || E == Epi::ResidSsq) return __ldg(a.b + row);
  if constexpr (E == Epi::Add) return y[row];
  return 0.0;
}
template <Epi E>
__device__ __forceinline__ void spmv_epi(const SpmvArgs& a, double* y, int row, double s,
                                         double pre, double& red) {
  if constexpr (E == Epi::Store) {
    y[row] = s;
  } else if constexpr (E == Epi::Resid) {
    y[row] = pre - s;
  } else if constexpr (E == Epi::ResidEta) {
    y[row] = (row < a.n_u ? a.eta_u : a.eta_p) * (pre - s);
  } else if constexpr (E == Epi::Add) {
    y[row] = pre + s;
  } else if constexpr (E == Epi::StoreDot) {
    y[row] = s;
    red = fma(s, pre, red);
  } else if constexpr (E == Epi::ResidSsq) {
    const double r = pre - s;
    y[row] = r;
    red = fma(r, r, red);
  }
}

// ------------------------------------------------------------------ SpMV --
// G lanes per row; the warp iterates over groups of rows with a warp-uniform
// trip count so the segmented shuffle tree is always executed by full warps.
template <int G, Epi E>
__global__ void __launch_bounds__(256, 8) spmv_kernel(int nrows, const int* __restrict__ rp,
                                                   const int* __restrict__ ci,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, SpmvArgs a,
                                                   double* partials, unsigned* ticket) {
  if (a.gate && *a.gate) return;
  constexpr bool kRed = (E == Epi::StoreDot || E == Epi::ResidSsq);
  constexpr int RPW = 32 / G;  // rows per warp per step
  const int lane = threadIdx.x & 31;
  const int sub = lane & (G - 1);
  const int grp = lane / G;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  double red = 0.0;
  for (int base = warp * RPW; base < nrows; base += nwarps * RPW) {
    const int row = base + grp;
    double s = 0.0;
    const bool lead = sub == 0 && row < nrows;
    if (row < nrows) {
      const int beg = __ldg(rp + row), end = __ldg(rp + row + 1);
      // four strides per pass with predicated loads: all values/columns of a
      // pass are requested before any x, so a row costs three dependent
      // round trips (rp, ci, x) instead of two per stride
      for (int k0 = beg + sub; k0 < end; k0 += 4 * G) {
        double v[4], xv[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * G;
          const bool in = k < end;
          v[u] = in ? __ldcs(val + k) : 0.0;
          cc[u] = in ? __ldcs(ci + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = (k0 + u * G < end) ? __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) s = fma(v[u], xv[u], s);
      }
    }
    // the epilogue operand is requested before the shuffle tree, whose
    // latency it overlaps (loading it before the row product instead costs
    // registers under the 32-register cap: 113 vs 99 us for Resid on K0)
    const double pre = spmv_pre<E>(a, y, row, lead);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
    if (lead) spmv_epi<E>(a, y, row, s, pre, red);
  }
  if constexpr (kRed) reduce_finish(red, a.fin, partials, ticket);
}

template <int G>
static void spmv_dispatch_e(Ctx& c, const Matrix& m, const double* x, double* y, Epi e,
                            const SpmvArgs& a, int r0 = 0, int r1 = -1) {
  // rows [r0, r1) only (Store): row offsets are absolute, so the kernel runs
  // on the shifted row-offset array and output
  const int nrows = r1 < 0 ? m.nrows : r1 - r0;
  y += r0;
  const int rows_per_block = 256 / G;
  long long need = (nrows + rows_per_block - 1) / rows_per_block;
  auto* rp = m.rp.p + r0;
  auto* ci = m.ci.p;
  auto* v = m.v.p;
  // persistent grid of exactly the resident blocks: a partial second wave of
  // a grid-stride kernel leaves most SMs idle at the tail (measured 209 us vs
  // 122 us for the reducing variants at 1184 blocks)
  auto grid_of = [&](auto kern) {
    static thread_local int occ[6] = {0, 0, 0, 0, 0, 0};
    int& o = occ[static_cast<int>(e)];
    if (!o) {
      SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, 0));
      o = std::max(o, 1);
    }
    const long long cap = std::min<long long>((long long)o * c.num_sms, kMaxRedGrid);
    return (int)std::max(1LL, std::min(need, cap));
  };
  switch (e) {
#define CASE(EE)                                                                              \
  case Epi::EE:                                                                               \
    spmv_kernel<G, Epi::EE><<<grid_of(spmv_kernel<G, Epi::EE>), 256, 0, c.stream>>>(          \
        nrows, rp, ci, v, x, y, a, c.partials.p, c.ticket.p);                                 \
    break;
    CASE(Store)
    CASE(Resid)
    CASE(ResidEta)
    CASE(Add)
    CASE(StoreDot)
    CASE(ResidSsq)
#undef CASE
  }
  SAG_LAUNCHED(c);
}

void launch_spmv(Ctx& c, const Matrix& m, const double* x, double* y, Epi e, const SpmvArgs& a) {
  if (m.nrows == 0) return;
  switch (m.group) {
    case 2: spmv_dispatch_e<2>(c, m, x, y, e, a); break;
    case 4: spmv_dispatch_e<4>(c, m, x, y, e, a); break;
    case 8: spmv_dispatch_e<8>(c, m, x, y, e, a); break;
    case 16: spmv_dispatch_e<16>(c, m, x, y, e, a); break;
    default: spmv_dispatch_e<32>(c, m, x, y, e, a); break;
  }
}
// The Store product on a few row ranges in one launch (the pipelined
// host-buffer step: one graph node per stage instead of one per range).
template <int G>
__global__ void __launch_bounds__(256, 8) spmv_ranges_kernel(RowRanges R, const int* __restrict__ rp,
                                                          const int* __restrict__ ci,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y) {
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int sub = lane & (G - 1);
  const int grp = lane / G;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int total = R.total();
  for (int base = warp * RPW; base < total; base += nwarps * RPW) {
    const int v = base + grp;
    const bool ok = v < total;
    const int row = ok ? R.row(v) : 0;
    double s = 0.0;
    if (ok) {
      const int beg = __ldg(rp + row), end = __ldg(rp + row + 1);
      for (int k0 = beg + sub; k0 < end; k0 += 4 * G) {
        double vv[4], xv[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * G;
          const bool in = k < end;
          vv[u] = in ? __ldcs(val + k) : 0.0;
          cc[u] = in ? __ldcs(ci + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = (k0 + u * G < end) ? __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) s = fma(vv[u], xv[u], s);
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
    if (ok && sub == 0) y[row] = s;
  }
}

template <int G>
static void spmv_ranges_g(Ctx& c, const Matrix& m, const RowRanges& R, const double* x, double* y,
                          cudaStream_t st) {
  static thread_local int occ = 0;
  if (!occ) {
    SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_ranges_kernel<G>, 256, 0));
    occ = std::max(occ, 1);
  }
  const int rows_per_block = 256 / G;
  const long long need = (R.total() + rows_per_block - 1) / rows_per_block;
  const int grid = (int)std::max(1LL, std::min(need, (long long)occ * c.num_sms));
  spmv_ranges_kernel<G><<<grid, 256, 0, st>>>(R, m.rp.p, m.ci.p, m.v.p, x, y);
  SAG_LAUNCHED(c);
}
void launch_spmv_ranges(Ctx& c, const Matrix& m, const RowRanges& R, const double* x, double* y,
                        cudaStream_t st) {
  if (R.total() <= 0) return;
  switch (m.group) {
    case 2: spmv_ranges_g<2>(c, m, R, x, y, st); break;
    case 4: spmv_ranges_g<4>(c, m, R, x, y, st); break;
    case 8: spmv_ranges_g<8>(c, m, R, x, y, st); break;
    case 16: spmv_ranges_g<16>(c, m, R, x, y, st); break;
    default: spmv_ranges_g<32>(c, m, R, x, y, st); break;
  }
}

void launch_spmv_rows(Ctx& c, const Matrix& m, int r0, int r1, const double* x, double* y) {
  if (r1 <= r0) return;
  const SpmvArgs a;
  switch (m.group) {
    case 2: spmv_dispatch_e<2>(c, m, x, y, Epi::Store, a, r0, r1); break;
    case 4: spmv_dispatch_e<4>(c, m, x, y, Epi::Store, a, r0, r1); break;
    case 8: spmv_dispatch_e<8>(c, m, x, y, Epi::Store, a, r0, r1); break;
    case 16: spmv_dispatch_e<16>(c, m, x, y, Epi::Store, a, r0, r1); break;
    default: spmv_dispatch_e<32>(c, m, x, y, Epi::Store, a, r0, r1); break;
  }
}

// --------------------------------------------------------------- BLAS-1 --

__global__ void __launch_bounds__(kRedBlock) dot_kernel(int n, const double* __restrict__ a,
                                                        const double* __restrict__ b, Fin fin,
                                                        const int* gate, double* partials,
                                                        unsigned* ticket) {
  if (gate && *gate) return;
  // four grid strides per pass: eight independent loads in flight per thread
  // (these vectors are streamed once; one load per trip leaves HBM idle)
  const int st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  for (; i + 3 * st < n; i += 4 * st) {
    const double a0 = a[i], a1 = a[i + st], a2 = a[i + 2 * st], a3 = a[i + 3 * st];
    const double b0 = b[i], b1 = b[i + st], b2 = b[i + 2 * st], b3 = b[i + 3 * st];
    s = fma(a0, b0, s);
    s = fma(a1, b1, s);
    s = fma(a2, b2, s);
    s = fma(a3, b3, s);
  }
  for (; i < n; i += st) s = fma(a[i], b[i], s);
  reduce_finish(s, fin, partials, ticket);
}

// ||a||^2 finished twice (e.g. FIN_REF then FIN_BETA of an inner solve whose
// residual is its right-hand side): one pass instead of two identical ones
__global__ void __launch_bounds__(kRedBlock) ssq2_kernel(int n, const double* __restrict__ a,
                                                         Fin f1, Fin f2, double* partials,
                                                         unsigned* ticket) {
  const int st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  for (; i + 3 * st < n; i += 4 * st) {
    const double a0 = a[i], a1 = a[i + st], a2 = a[i + 2 * st], a3 = a[i + 3 * st];
    s = fma(a0, a0, s);
    s = fma(a1, a1, s);
    s = fma(a2, a2, s);
    s = fma(a3, a3, s);
  }
  for (; i < n; i += st) s = fma(a[i], a[i], s);
  __shared__ double sh[32];
  const double bs = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
  if (last_block(ticket)) {
    const double tot = sum_partials(partials, gridDim.x, sh);
    if (threadIdx.x == 0) {
      apply_fin(f1, tot);
      apply_fin(f2, tot);
      *ticket = 0u;
    }
  }
}

__global__ void __launch_bounds__(kRedBlock) sum_kernel(int n, const double* __restrict__ a,
                                                        Fin fin, double* partials,
                                                        unsigned* ticket) {
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    s += a[i];
  reduce_finish(s, fin, partials, ticket);
}

// Elementwise pass with four grid strides per trip: all loads of a trip are
// issued before any use (load(i) returns the operands, store(i, ops) writes),
// so each thread keeps several independent requests in flight.
template <class Load, class Store>
__device__ __forceinline__ void ew4(int n, Load load, Store store) {
  const int st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * st < n; i += 4 * st) {
    const auto o0 = load(i), o1 = load(i + st), o2 = load(i + 2 * st), o3 = load(i + 3 * st);
    store(i, o0);
    store(i + st, o1);
    store(i + 2 * st, o2);
    store(i + 3 * st, o3);
  }
  for (; i < n; i += st) store(i, load(i));
}

__global__ void div_kernel(int n, const double* __restrict__ x, const double* s,
                           double* __restrict__ y, const int* gate, const int* gate2) {
  if ((gate && *gate) || (gate2 && *gate2)) return;
  const double d = *s;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void __launch_bounds__(kRedBlock) mgs_kernel(int n, double* __restrict__ w,
                                                        const double* __restrict__ vprev,
                                                        const double* h,
                                                        const double* __restrict__ vnext,
                                                        Fin fin, const int* gate,
                                                        double* partials, unsigned* ticket) {
  if (gate && *gate) return;
  const double hh = vprev ? *h : 0.0;
  const int st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (vprev) {
    for (; i + 3 * st < n; i += 4 * st) {
      double wv[4], pv[4], nv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wv[u] = w[i + u * st];
        pv[u] = vprev[i + u * st];
        nv[u] = vnext[i + u * st];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wv[u] = fma(-hh, pv[u], wv[u]);
        w[i + u * st] = wv[u];
        s = fma(wv[u], nv[u], s);
      }
    }
  }
  for (; i < n; i += st) {
    double wi = w[i];
    if (vprev) {
      wi = fma(-hh, vprev[i], wi);
      w[i] = wi;
    }
    s = fma(wi, vnext[i], s);
  }
  reduce_finish(s, fin, partials, ticket);
}

// write_w = 0: the orthogonalised w is only needed for its norm (last Arnoldi
// step of a fixed-length inner solve, whose v_(j+1) is never used), so w keeps
// A z_j -- which the relaxation reuses for the next residual.
__global__ void __launch_bounds__(kRedBlock) mgs_last_kernel(int n, double* __restrict__ w,
                                                             const double* __restrict__ v,
                                                             const double* h, Fin fin,
                                                             const int* gate, int write_w,
                                                             double* partials, unsigned* ticket) {
  if (gate && *gate) return;
  const double hh = *h;
  const int st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  for (; i + 3 * st < n; i += 4 * st) {
    double wv[4], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      wv[u] = w[i + u * st];
      vv[u] = v[i + u * st];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double wi = fma(-hh, vv[u], wv[u]);
      if (write_w) w[i + u * st] = wi;
      s = fma(wi, wi, s);
    }
  }
  for (; i < n; i += st) {
    const double wi = fma(-hh, v[i], w[i]);
    if (write_w) w[i] = wi;
    s = fma(wi, wi, s);
  }
  reduce_finish(s, fin, partials, ticket);
}

// r = eta .* (b - y_0 w) with w = K z_0 from a one-step relaxation x = y_0 z_0
// (so r = eta .* (b - K x) by linearity); r = eta .* b when the relaxation
// made no step (jeff == 0, zero residual).
__global__ void lin_resid_kernel(int n, int n_u, double eu, double ep,
                                 const double* __restrict__ b, const double* __restrict__ w,
                                 const KState* st, double* __restrict__ r) {
  const bool step = st->jeff > 0;
  const double y0 = step ? ks_y(const_cast<KState*>(st))[0] : 0.0;
  ew4(n, [&](int i) { return make_double2(b[i], step ? w[i] : 0.0); },
      [&](int i, double2 v) {
        const double t = step ? fma(-y0, v.y, v.x) : v.x;
        r[i] = (i < n_u ? eu : ep) * t;
      });
}

// krylov.cpp:102-107, one thread (j <= restart)
__global__ void backsub_kernel(KState* st) {
  const int j = st->jeff, m = st->m;
  const double* h = ks_h(st);
  const double* g = ks_g(st);
  double* y = ks_y(st);
  for (int i = j - 1; i >= 0; --i) {
    double s = g[i];
    for (int k = i + 1; k < j; ++k) s -= h[(size_t)i * m + k] * y[k];
    y[i] = s / h[(size_t)i * m + i];
  }
}

// krylov.cpp:108-110 (+ vanka.cpp:208 for relaxation): x += sum_i y_i Z_i
__global__ void update_kernel(int n, double* __restrict__ x, const double* __restrict__ Z,
                              size_t zs, const KState* st, int store) {
  const int j = st->jeff;
  if (j == 0 && !store) return;
  const double* y = ks_y(const_cast<KState*>(st));
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double corr = 0.0;
#pragma unroll 4
    for (int i = 0; i < j; ++i) corr = fma(y[i], Z[(size_t)i * zs + k], corr);
    x[k] = store ? corr : x[k] + corr;
  }
}

// y = x / *s and z = d .* y in one pass (v_0 = r / beta, z_0 = M v_0 for a
// Jacobi-preconditioned inner solve, amg.cpp:265-276)
__global__ void div_mul_kernel(int n, const double* __restrict__ x, const double* s,
                               double* __restrict__ y, const double* __restrict__ d,
                               double* __restrict__ z, const int* gate) {
  if (gate && *gate) return;
  const double q = *s;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = x[i] / q;
    y[i] = v;
    z[i] = d[i] * v;
  }
}

// backsub_kernel + update_kernel in one launch for short inner solves
// (jeff <= kUpdBsMax): every block back-substitutes the small Hessenberg
// system itself (the same operations as backsub_kernel), block 0 stores y
__global__ void update_bs_kernel(int n, double* __restrict__ x, const double* __restrict__ Z,
                                 size_t zs, KState* st, int store) {
  __shared__ double ys[kUpdBsMax];
  const int j = st->jeff, m = st->m;
  if (threadIdx.x == 0) {
    const double* h = ks_h(st);
    const double* g = ks_g(st);
    double y[kUpdBsMax];
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < j; ++k) s -= h[(size_t)i * m + k] * y[k];
      y[i] = s / h[(size_t)i * m + i];
    }
    for (int i = 0; i < j; ++i) {
      ys[i] = y[i];
      if (blockIdx.x == 0) ks_y(st)[i] = y[i];
    }
  }
  __syncthreads();
  if (j == 0 && !store) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double corr = 0.0;
#pragma unroll 4
    for (int i = 0; i < j; ++i) corr = fma(ys[i], Z[(size_t)i * zs + k], corr);
    x[k] = store ? corr : x[k] + corr;
  }
}

__global__ void mul_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = a[i] * b[i];
}

// inv_diagonal (sparse.cpp:208-215)
__global__ void inv_diag_kernel(int n, const int* rp, const int* ci, const double* v,
                                double* dinv, int* bad) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k)
      if (ci[k] == r) d = v[k];
    if (d == 0.0) atomicOr(bad, 1);
    dinv[r] = 1.0 / d;
  }
}

__global__ void kinit_kernel(KState* st, int m, double tol, double bd, int hist_cap,
                             int keep_ref) {
  if (!keep_ref) st->ref = 1.0;
  st->tol = tol;
  st->bd = bd;
  st->m = m;
  st->stop = 0;
  st->breakdown = 0;
  st->jeff = 0;
  st->iterations = 0;
  st->hist_len = 0;
  st->hist_cap = hist_cap;
  st->converged = 0;
  st->beta = 0.0;
  st->rnorm = 0.0;
}

__global__ void copy_kernel(int n, const double* __restrict__ x, double* __restrict__ y) {
  ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = v; });
}
__global__ void zero_kernel(int n, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = 0.0;
}
__global__ void project_kernel(int n, int n_u, const double* __restrict__ x, const double* mean,
                               double* __restrict__ y) {
  const double mu = *mean;
  ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = i < n_u ? v : v - mu; });
}
__global__ void eta_kernel(int n, int n_u, double eu, double ep, const double* __restrict__ x,
                           double* __restrict__ y) {
  ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = (i < n_u ? eu : ep) * v; });
}
__global__ void add_kernel(int n, double* __restrict__ x, const double* __restrict__ y) {
  ew4(n, [&](int i) { return make_double2(x[i], y[i]); },
      [&](int i, double2 v) { x[i] = v.x + v.y; });
}
__global__ void axpy_kernel(int n, double* __restrict__ x, double omega,
                            const double* __restrict__ d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = x[i] + omega * d[i];
}

static int ew_grid(Ctx& c, long long n) {
  long long g = (n + 255) / 256;
  return (int)std::max(1LL, std::min(g, (long long)c.num_sms * 16));
}

// Reduction grids: red_grid(n), but never more blocks than are resident at
// once -- a partial second wave of a grid-stride reduction idles most SMs at
// the tail (as measured for the fused SpMV reductions).
template <class K>
static int red_grid_fit(Ctx& c, K kern, long long n) {
  static thread_local int occ = 0;
  if (!occ) {
    SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRedBlock, 0));
    occ = std::max(occ, 1);
  }
  return std::max(1, std::min(red_grid(n), occ * c.num_sms));
}

void launch_dot(Ctx& c, int n, const double* a, const double* b, const Fin& fin,
                const int* gate) {
  dot_kernel<<<red_grid_fit(c, dot_kernel, n), kRedBlock, 0, c.stream>>>(n, a, b, fin, gate, c.partials.p,
                                                      c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_ssq(Ctx& c, int n, const double* a, const Fin& fin, const int* gate) {
  dot_kernel<<<red_grid_fit(c, dot_kernel, n), kRedBlock, 0, c.stream>>>(n, a, a, fin, gate, c.partials.p,
                                                      c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_sum(Ctx& c, int n, const double* a, const Fin& fin) {
  sum_kernel<<<red_grid(n), kRedBlock, 0, c.stream>>>(n, a, fin, c.partials.p, c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_div(Ctx& c, int n, const double* x, const double* s, double* y, const int* gate,
                const int* gate2) {
  div_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, s, y, gate, gate2);
  SAG_LAUNCHED(c);
}
void launch_mgs(Ctx& c, int n, double* w, const double* vprev, const double* h,
                const double* vnext, const Fin& fin, const int* gate) {
  mgs_kernel<<<red_grid_fit(c, mgs_kernel, n), kRedBlock, 0, c.stream>>>(n, w, vprev, h, vnext, fin, gate,
                                                      c.partials.p, c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_mgs_last(Ctx& c, int n, double* w, const double* v, const double* h, const Fin& fin,
                     const int* gate, bool write_w) {
  mgs_last_kernel<<<red_grid_fit(c, mgs_last_kernel, n), kRedBlock, 0, c.stream>>>(n, w, v, h, fin, gate, write_w ? 1 : 0,
                                                           c.partials.p, c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_lin_resid(Ctx& c, int n, int n_u, double eta_u, double eta_p, const double* b,
                      const double* w, const KState* st, double* r) {
  lin_resid_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, n_u, eta_u, eta_p, b, w, st, r);
  SAG_LAUNCHED(c);
}
void launch_backsub(Ctx& c, KState* st) {
  backsub_kernel<<<1, 1, 0, c.stream>>>(st);
  SAG_LAUNCHED(c);
}
void launch_update(Ctx& c, int n, double* x, const double* Z, size_t zstride, KState* st,
                   bool store) {
  update_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, Z, zstride, st, store ? 1 : 0);
  SAG_LAUNCHED(c);
}
void launch_ssq2(Ctx& c, int n, const double* a, const Fin& f1, const Fin& f2) {
  ssq2_kernel<<<red_grid_fit(c, ssq2_kernel, n), kRedBlock, 0, c.stream>>>(n, a, f1, f2,
                                                                           c.partials.p, c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_div_mul(Ctx& c, int n, const double* x, const double* s, double* y, const double* d,
                    double* z, const int* gate) {
  div_mul_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, s, y, d, z, gate);
  SAG_LAUNCHED(c);
}
void launch_update_bs(Ctx& c, int n, double* x, const double* Z, size_t zstride, KState* st,
                      int m, bool store) {
  if (m > kUpdBsMax) {
    launch_backsub(c, st);
    launch_update(c, n, x, Z, zstride, st, store);
    return;
  }
  update_bs_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, Z, zstride, st, store ? 1 : 0);
  SAG_LAUNCHED(c);
}
void launch_mul(Ctx& c, int n, const double* a, const double* b, double* y) {
  mul_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, a, b, y);
  SAG_LAUNCHED(c);
}
void launch_inv_diag(Ctx& c, const Matrix& m, double* dinv, int* bad) {
  inv_diag_kernel<<<ew_grid(c, m.nrows), 256, 0, c.stream>>>(m.nrows, m.rp.p, m.ci.p, m.v.p, dinv,
                                                             bad);
  SAG_LAUNCHED(c);
}
void launch_kinit(Ctx& c, KState* st, int m, double tol, double bd, int hist_cap,
                  bool keep_ref) {
  kinit_kernel<<<1, 1, 0, c.stream>>>(st, m, tol, bd, hist_cap, keep_ref ? 1 : 0);
  SAG_LAUNCHED(c);
}
void launch_copy(Ctx& c, int n, const double* x, double* y) {
  copy_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, y);
  SAG_LAUNCHED(c);
}
void launch_zero(Ctx& c, int n, double* y) {
  zero_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, y);
  SAG_LAUNCHED(c);
}
void launch_project(Ctx& c, int n, int n_u, const double* x, const double* mean, double* y) {
  project_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, n_u, x, mean, y);
  SAG_LAUNCHED(c);
}
void launch_eta(Ctx& c, int n, int n_u, double eta_u, double eta_p, const double* x, double* y) {
  eta_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, n_u, eta_u, eta_p, x, y);
  SAG_LAUNCHED(c);
}
void launch_add(Ctx& c, int n, double* x, const double* y) {
  add_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, y);
  SAG_LAUNCHED(c);
}
void launch_axpy(Ctx& c, int n, double* x, double omega, const double* d) {
  axpy_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, omega, d);
  SAG_LAUNCHED(c);
}

// ---------------------------------------------------- matrix validation --

__global__ void validate_csr_kernel(int nrows, int ncols, long long nnz, const int* rp,
                                    const int* ci, int* bad) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int b = rp[r], e = rp[r + 1];
    if (b > e || b < 0 || (long long)e > nnz) {
      atomicOr(bad, 1);
      continue;
    }
    for (int k = b; k < e; ++k) {
      const int c = ci[k];
      if (c < 0 || c >= ncols) atomicOr(bad, 2);
      if (k > b && c <= ci[k - 1]) atomicOr(bad, 4);
    }
  }
}

__global__ void norm_inf_kernel(int nrows, const int* rp, const double* v, double* out) {
  __shared__ double sh[32];
  double best = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) s += fabs(v[k]);
    best = fmax(best, s);
  }
  // max-reduce in one block (gridDim.x == 1)
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b = fmax(b, sh[i]);
    *out = b;
  }
}

void compute_norm_inf(Ctx& c, Matrix& m) {
  if (m.norm_inf >= 0.0) return;
  norm_inf_kernel<<<1, 1024, 0, c.stream>>>(m.nrows, m.rp.p, m.v.p, c.scal.p);
  SAG_LAUNCHED(c);
  SAG_CUDA(cudaMemcpyAsync(&m.norm_inf, c.scal.p, sizeof(double), cudaMemcpyDeviceToHost,
                           c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
}

// ------------------------------------------------------------ transpose --

__global__ void row_of_kernel(int nrows, const int* rp, int* row_of) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x)
    for (int k = rp[r]; k < rp[r + 1]; ++k) row_of[k] = r;
}
__global__ void iota_kernel(long long n, int* a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}
__global__ void count_kernel(long long n, const int* key, int* cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + key[i], 1);
}
__global__ void permute_kernel(long long n, const int* perm, const int* row_of, const double* v,
                               int* ciT, double* vT) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int o = perm[q];
    ciT[q] = row_of[o];
    vT[q] = v[o];
  }
}

static int pick_group(long long nnz, int nrows) {
  if (const char* e = getenv("SAG_SPMV_GROUP")) return atoi(e);
  // ~4 entries per lane: each lane issues its 4-wide pass of loads at once,
  // and the shuffle tree (on the same LSU data pipe as the gathers) stays
  // short -- on K0 (17 entries per row) G = 4 runs in 97 us, G = 8 in 117 us
  const double avg = nrows > 0 ? (double)nnz / nrows : 0.0;
  if (avg <= 4.0) return 2;
  if (avg <= 24.0) return 4;
  if (avg <= 64.0) return 8;
  if (avg <= 128.0) return 16;
  return 32;
}

std::unique_ptr<Matrix> transpose_dev(Ctx& c, const Matrix& a) {
  auto t = std::make_unique<Matrix>();
  t->ctx = &c;
  t->nrows = a.ncols;
  t->ncols = a.nrows;
  t->nnz = a.nnz;
  t->rp.alloc(a.ncols + 1 + kCsrPad);
  t->ci.alloc(a.nnz + kCsrPad);
  t->v.alloc(a.nnz + kCsrPad);
  const long long n = a.nnz;
  DevBuf<int> row_of(n), idx(n), keys_out(n), perm(n), cnt(a.ncols + 1);
  const int g = ew_grid(c, n);
  row_of_kernel<<<ew_grid(c, a.nrows), 256, 0, c.stream>>>(a.nrows, a.rp.p, row_of.p);
  SAG_LAUNCHED(c);
  iota_kernel<<<g, 256, 0, c.stream>>>(n, idx.p);
  SAG_LAUNCHED(c);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (a.ncols + 1), c.stream));
  count_kernel<<<g, 256, 0, c.stream>>>(n, a.ci.p, cnt.p);
  SAG_LAUNCHED(c);
  size_t tmp = 0, tmp2 = 0;
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, t->rp.p, a.ncols + 1, c.stream));
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, a.ci.p, keys_out.p, idx.p, perm.p,
                                           (int)n, 0, 32, c.stream));
  DevBuf<unsigned char> ws(std::max(tmp, tmp2));
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, tmp, cnt.p, t->rp.p, a.ncols + 1, c.stream));
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, tmp2, a.ci.p, keys_out.p, idx.p, perm.p,
                                           (int)n, 0, 32, c.stream));
  permute_kernel<<<g, 256, 0, c.stream>>>(n, perm.p, row_of.p, a.v.p, t->ci.p, t->v.p);
  SAG_LAUNCHED(c);
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  t->group = pick_group(t->nnz, t->nrows);
  return t;
}

std::unique_ptr<Matrix> matrix_upload(Ctx& c, int nrows, int ncols, long long nnz,
                                      const int* rp, const int* ci, const double* v) {
  SAG_REQUIRE(nrows >= 0 && ncols >= 0 && nnz >= 0, SAG_DIMENSION_MISMATCH,
              "sag_matrix_create: negative size");
  SAG_REQUIRE(nnz < (1LL << 31), SAG_DIMENSION_MISMATCH, "sag_matrix_create: nnz exceeds int32");
  SAG_REQUIRE(rp && (nnz == 0 || (ci && v)), SAG_INVALID_ARGUMENT, "sag_matrix_create: null array");
  auto m = std::make_unique<Matrix>();
  m->ctx = &c;
  m->nrows = nrows;
  m->ncols = ncols;
  m->nnz = nnz;
  m->rp.alloc(nrows + 1 + kCsrPad);
  m->ci.alloc(nnz + kCsrPad);
  m->v.alloc(nnz + kCsrPad);
  SAG_CUDA(cudaMemcpyAsync(m->rp.p, rp, sizeof(int) * (nrows + 1), cudaMemcpyDefault, c.stream));
  if (nnz) {
    SAG_CUDA(cudaMemcpyAsync(m->ci.p, ci, sizeof(int) * nnz, cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaMemcpyAsync(m->v.p, v, sizeof(double) * nnz, cudaMemcpyDefault, c.stream));
  }
  int* bad = reinterpret_cast<int*>(c.scal.p);
  SAG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
  validate_csr_kernel<<<ew_grid(c, nrows), 256, 0, c.stream>>>(nrows, ncols, nnz, m->rp.p,
                                                               m->ci.p, bad);
  SAG_LAUNCHED(c);
  int hb = 0, first = 0, last = 0;
  SAG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaMemcpyAsync(&first, m->rp.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaMemcpyAsync(&last, m->rp.p + nrows, sizeof(int), cudaMemcpyDeviceToHost,
                           c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  SAG_REQUIRE(first == 0 && last == nnz, SAG_DIMENSION_MISMATCH,
              "sag_matrix_create: row_offsets do not span [0, nnz]");
  SAG_REQUIRE(!(hb & 1), SAG_DIMENSION_MISMATCH, "sag_matrix_create: row_offsets not monotone");
  SAG_REQUIRE(!(hb & 2), SAG_DIMENSION_MISMATCH, "sag_matrix_create: column index out of range");
  SAG_REQUIRE(!(hb & 4), SAG_ERROR,
              "sag_matrix_create: rows must be canonical (strictly increasing columns)");
  m->group = pick_group(nnz, nrows);
  return m;
}

// ------------------------------------------ partitioned-solve primitives --
// Building blocks for a caller that distributes the solve over ranks
// (paper_2306_06795_b200/dist.py): every scalar stays in device memory, so a
// reduction -> all-reduce -> axpy chain is stream-ordered with no host sync.

// *out = sum over i with mask[i] (all i when mask is null) of a_i b_i
__global__ void __launch_bounds__(kRedBlock) dot_mask_kernel(int n, const double* __restrict__ a,
                                                             const double* __restrict__ b,
                                                             const unsigned char* __restrict__ mask,
                                                             Fin fin, double* partials,
                                                             unsigned* ticket) {
  const int st = gridDim.x * blockDim.x;
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    if (!mask || mask[i]) s = fma(a[i], b[i], s);
  reduce_finish(s, fin, partials, ticket);
}
// y = y + sign * (*s) x   (MGS: w[k] -= h_ij v_i[k], krylov.cpp:66)
__global__ void axpy_dev_kernel(int n, const double* s, double sign, const double* __restrict__ x,
                                double* __restrict__ y) {
  const double h = *s;
  ew4(n, [&](int i) { return make_double2(y[i], x[i]); },
      [&](int i, double2 v) { y[i] = sign < 0.0 ? v.x - h * v.y : v.x + h * v.y; });
}
// y = x / d, d = *s or sqrt(*s)   (v_0 = r / ||r||, krylov.cpp:47-48); y = 0
// when d == 0 (a zero residual, whose Krylov step the reference skips)
__global__ void div_dev_kernel(int n, const double* __restrict__ x, const double* s, int take_sqrt,
                               double* __restrict__ y) {
  const double d = take_sqrt ? sqrt(*s) : *s;
  ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = d != 0.0 ? v / d : 0.0; });
}
// One-step FGMRES coefficient (krylov.cpp:42-110 with m = max_iters = 1, tol
// 0, zero guess): from ||r||^2, h_00 = (A z_0, v_0) and ||w||^2 after the MGS
// step, the Givens rotation and the back substitution give y_0 (x += y_0 z_0);
// 0 when r = 0 (the reference returns before the step).
__global__ void fgmres1_coef_kernel(const double* ssq_r, const double* h00p, const double* ssq_w,
                                    double* y0) {
  const double beta = sqrt(*ssq_r), h00 = *h00p, h10 = sqrt(*ssq_w);
  if (beta == 0.0) {
    *y0 = 0.0;
    return;
  }
  const double denom = hypot(h00, h10);
  double cs = 1.0, sn = 0.0;
  if (denom > 0.0) {
    cs = h00 / denom;
    sn = h10 / denom;
  }
  const double hjj = cs * h00 + sn * h10;
  const double g0 = cs * beta;
  *y0 = g0 / hjj;
}
// y = x - (*sum) / count   (project_pressure, preconditioner.cpp:235-240)
__global__ void sub_mean_kernel(int n, const double* __restrict__ x, const double* sum,
                                double count, double* __restrict__ y) {
  const double mean = *sum / count;
  ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = v - mean; });
}
// y = a x + b y; a == b == 0: y = 0; b == 0: y = a x; b == 1: y = y + a x
// (x += y_i z_i, krylov.cpp:108-110)
__global__ void axpby_kernel(int n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  if (a == 0.0 && b == 0.0) {
    ew4(n, [&](int i) { return 0.0; }, [&](int i, double v) { y[i] = v; });
  } else if (b == 0.0) {
    ew4(n, [&](int i) { return x[i]; }, [&](int i, double v) { y[i] = a * v; });
  } else if (b == 1.0) {
    ew4(n, [&](int i) { return make_double2(y[i], x[i]); },
        [&](int i, double2 v) { y[i] = v.x + a * v.y; });
  } else {
    ew4(n, [&](int i) { return make_double2(y[i], x[i]); },
        [&](int i, double2 v) { y[i] = a * v.y + b * v.x; });
  }
}
// halo pack / unpack: dst[i] = src[idx[i]]; dst[idx[i]] (+)= src[i] (idx unique)
__global__ void gather_idx_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                  double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
// reverse halo over peer memory: dst (a neighbour's buffer, mapped by CUDA
// IPC) receives src[idx[i]] by NVLink stores; the system-scope fence orders
// them before the kernel's completion is observed by the neighbour
__global__ void push_idx_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
  __threadfence_system();
}
__global__ void scatter_idx_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                   double* __restrict__ dst, int add) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = idx[i];
    dst[d] = add ? dst[d] + src[i] : src[i];
  }
}

// internal launchers of the partitioned-solve primitives (no pointer-kind
// queries: usable while a stream is being captured)
__global__ void fin_from_kernel(Fin f, const double* tot) { apply_fin(f, *tot); }
void launch_fin_from(Ctx& c, const Fin& f, const double* tot) {
  fin_from_kernel<<<1, 1, 0, c.stream>>>(f, tot);
  SAG_LAUNCHED(c);
}
void launch_dot_mask(Ctx& c, int n, const double* a, const double* b, const unsigned char* mask,
                     double* out) {
  Fin f;
  f.kind = FIN_STORE;
  f.out = out;
  dot_mask_kernel<<<red_grid_fit(c, dot_mask_kernel, n), kRedBlock, 0, c.stream>>>(
      n, a, b, mask, f, c.partials.p, c.ticket.p);
  SAG_LAUNCHED(c);
}
void launch_axpy_dev(Ctx& c, int n, const double* s, double sign, const double* x, double* y) {
  if (n <= 0) return;
  axpy_dev_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, s, sign, x, y);
  SAG_LAUNCHED(c);
}
void launch_div_dev(Ctx& c, int n, const double* x, const double* s, int take_sqrt, double* y) {
  if (n <= 0) return;
  div_dev_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, s, take_sqrt, y);
  SAG_LAUNCHED(c);
}
void launch_fgmres1_coef(Ctx& c, const double* ssq_r, const double* h00, const double* ssq_w,
                         double* y0) {
  fgmres1_coef_kernel<<<1, 1, 0, c.stream>>>(ssq_r, h00, ssq_w, y0);
  SAG_LAUNCHED(c);
}
void launch_sub_mean(Ctx& c, int n, const double* x, const double* sum, double count, double* y) {
  if (n <= 0) return;
  sub_mean_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, x, sum, count, y);
  SAG_LAUNCHED(c);
}
void launch_axpby(Ctx& c, int n, double a, const double* x, double b, double* y) {
  if (n <= 0) return;
  axpby_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, a, x, b, y);
  SAG_LAUNCHED(c);
}
void launch_gather_idx(Ctx& c, int n, const int* idx, const double* src, double* dst) {
  if (n <= 0) return;
  gather_idx_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, idx, src, dst);
  SAG_LAUNCHED(c);
}
void launch_scatter_idx(Ctx& c, int n, const int* idx, const double* src, double* dst, int add) {
  if (n <= 0) return;
  scatter_idx_kernel<<<ew_grid(c, n), 256, 0, c.stream>>>(n, idx, src, dst, add);
  SAG_LAUNCHED(c);
}

// ------------------------------------------------------ sliced ELLPACK --
__global__ void sell_width_kernel(int nrows, int g, const int* __restrict__ rp,
                                  int* __restrict__ width) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int rs = 32 >> g;
  if (s * rs >= nrows) return;
  const int r = s * rs + (lane >> g);
  const int G = 1 << g;
  int steps = r < nrows ? (rp[r + 1] - rp[r] + G - 1) >> g : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
  if (lane == 0) width[s] = steps;
}
__global__ void sell_fill_kernel(int nrows, int ncols, int g, const int* __restrict__ rp,
                                 const int* __restrict__ ci, const double* __restrict__ v,
                                 const int* __restrict__ sptr, int* __restrict__ oc,
                                 double* __restrict__ ov) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int rs = 32 >> g, G = 1 << g;
  if (s * rs >= nrows) return;
  const int r = s * rs + (lane >> g), sub = lane & (G - 1);
  const int beg = r < nrows ? rp[r] : 0, len = r < nrows ? rp[r + 1] - beg : 0;
  const int pad = len > 0 ? ci[beg + len - 1] : min(max(r, 0), ncols - 1);
  const int p0 = sptr[s], w = (sptr[s + 1] - p0) >> 5;
  for (int j = 0; j < w; ++j) {
    const int k = j * G + sub;
    oc[p0 + 32 * j + lane] = k < len ? ci[beg + k] : pad;
    ov[p0 + 32 * j + lane] = k < len ? v[beg + k] : 0.0;
  }
}

void build_sell(Ctx& c, const Matrix& m, Sell& out) {
  // lanes per row from the mean row length (SAG_SELL_G: diagnostic override)
  const double mean = m.nrows > 0 ? (double)m.nnz / m.nrows : 0.0;
  int g = mean <= 8.0 ? 0 : mean <= 16.0 ? 1 : mean <= 32.0 ? 2 : mean <= 64.0 ? 3 : 4;
  if (const char* e = getenv("SAG_SELL_G")) g = std::max(0, std::min(5, atoi(e)));
  out.g = g;
  const int rs = 32 >> g;
  const int ns = (m.nrows + rs - 1) / rs;
  DevBuf<int> width(std::max(ns, 1));
  const int wpb = 8, blocks = (ns + wpb - 1) / wpb;
  if (ns > 0) sell_width_kernel<<<blocks, wpb * 32, 0, c.stream>>>(m.nrows, g, m.rp.p, width.p);
  SAG_LAUNCHED(c);
  std::vector<int> hw(std::max(ns, 1), 0), hp(ns + 1, 0);
  SAG_CUDA(cudaMemcpyAsync(hw.data(), width.p, sizeof(int) * ns, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  long long tot = 0;
  for (int i = 0; i < ns; ++i) {
    hp[i] = (int)tot;
    tot += 32LL * hw[i];
    SAG_REQUIRE(tot < (1LL << 31), SAG_DIMENSION_MISMATCH, "sliced ELLPACK copy exceeds int32 offsets");
  }
  hp[ns] = (int)tot;
  out.entries = tot;
  out.sptr.alloc(ns + 1);
  out.ci.alloc((size_t)std::max<long long>(tot, 1));
  out.v.alloc((size_t)std::max<long long>(tot, 1));
  SAG_CUDA(cudaMemcpyAsync(out.sptr.p, hp.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice,
                           c.stream));
  if (ns > 0)
    sell_fill_kernel<<<blocks, wpb * 32, 0, c.stream>>>(m.nrows, m.ncols, g, m.rp.p, m.ci.p, m.v.p,
                                                        out.sptr.p, out.ci.p, out.v.p);
  SAG_LAUNCHED(c);
  SAG_CUDA(cudaStreamSynchronize(c.stream));  // hp lives on this stack
}

// ------------------------------------------------- scalar V-cycle tail --
// One cluster runs the small levels of scalar_vcycle (amg.cpp:258-296). CTA q
// of the cluster owns rows [q chunk, (q+1) chunk) of every level and keeps
// that chunk of each level vector in its shared memory; SpMV gathers of other
// rows are DSMEM loads from the owning CTA. A reduction is a fixed-order
// block sum, a cluster barrier, and a fixed-order sum of the CS block
// partials read over DSMEM -- the same total in every CTA, so the Krylov
// scalars (KState in shared memory, updated by apply_fin exactly as the
// multi-launch path does) and every branch on them agree cluster-wide.
// Measured (tools/cluster_phase_probe.cu): a barrier phase with one
// dependent L2 load + store costs ~1.2 us, ~0.3 us with shared memory only.

constexpr int kTailThreads = 1024;
constexpr int kTailWarps = kTailThreads / 32;
constexpr int kTailMaxCs = 16;
enum { TB = 0, TX, TR, TRS, TW, TV0, TV1, TZ0, TZ1 };

// cluster barrier with release/acquire at cluster scope
__device__ __forceinline__ void cluster_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct TailSh {
  double part[2][4];            // this CTA's partials (two alternating slots)
  double wp[kTailWarps][4];
  double tot[4];
  double ks[32];                // KState for m = 2, no history (kstate_bytes(2, 0) <= 256)
  double* base[kTailMaxCs];     // generic address of each CTA's dynamic shared memory
};

// a level as seen by one CTA
struct TL {
  int n, chunk, off, r0, nloc;
  float inv;
};
__device__ __forceinline__ TL tl_make(const TailLevel& L, int q) {
  TL t;
  t.n = L.n;
  t.chunk = L.chunk;
  t.off = L.off;
  t.r0 = q * L.chunk;
  t.nloc = max(0, min(L.n - t.r0, L.chunk));
  t.inv = 1.0f / (float)L.chunk;
  return t;
}
__device__ __forceinline__ double* tl_vec(double* sm, const TL& t, int k) {
  return sm + t.off + k * t.chunk;
}
// vector k of level t at global row col (any CTA's chunk)
__device__ __forceinline__ double tl_get(const TailSh& s, const TL& t, int k, int col) {
  int q = (int)((float)col * t.inv);
  if (q * t.chunk > col) --q;
  else if ((q + 1) * t.chunk <= col) ++q;
  return s.base[q][t.off + k * t.chunk + col - q * t.chunk];
}

template <int K>
__device__ __forceinline__ void tail_reduce(cg::cluster_group& cl, TailSh& s, int& slot,
                                            double (&v)[K]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double t = warp_sum(v[k]);
    if (lane == 0) s.wp[wid][k] = t;
  }
  __syncthreads();
  if (wid < K) {
    const double t = warp_sum(s.wp[lane][wid]);
    if (lane == 0) s.part[slot][wid] = t;
  }
  cluster_bar();
  if (wid < K) {
    double t = 0.0;
    if (lane < (int)cl.num_blocks()) t = *cl.map_shared_rank(&s.part[slot][wid], lane);
    t = warp_sum(t);
    if (lane == 0) s.tot[wid] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = s.tot[k];
  slot ^= 1;
}

// rows [r0, r0 + nloc) of y = A x with A in sliced ELLPACK (r0 a multiple of
// 32): G lanes per row, each warp takes two slices at a time (all their
// index / value loads, then all their gathers, are issued together).
// getx(col) reads x; epi(local row, sum) runs on the row's first lane.
template <class G, class F>
__device__ __forceinline__ void sell_spmv(const SellView& A, int r0, int nloc, G getx, F epi) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = A.g, rs = 32 >> g;
  const int s0 = r0 >> (5 - g), nsl = (nloc + rs - 1) >> (5 - g);
  for (int sa = wid; sa < nsl; sa += 2 * kTailWarps) {
    const int sb = sa + kTailWarps;
    const bool hb = sb < nsl;
    const int p0 = __ldg(A.sptr + s0 + sa), q0 = __ldg(A.sptr + s0 + sa + 1);
    int p1 = 0, q1 = 0;
    if (hb) {
      p1 = __ldg(A.sptr + s0 + sb);
      q1 = __ldg(A.sptr + s0 + sb + 1);
    }
    const int n0 = (q0 - p0) >> 5, n1 = (q1 - p1) >> 5;
    const int* c0 = A.ci + p0 + lane;
    const double* v0 = A.v + p0 + lane;
    const int* c1 = A.ci + p1 + lane;
    const double* v1 = A.v + p1 + lane;
    double a0 = 0.0, a1 = 0.0;
    const int nmax = max(n0, n1);
    for (int k = 0; k < nmax; k += 4) {
      double va[4], vb[4], xa[4], xb[4];
      int ca[4], cb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool oa = k + u < n0, ob = k + u < n1;
        ca[u] = oa ? __ldg(c0 + 32 * (k + u)) : -1;
        va[u] = oa ? __ldg(v0 + 32 * (k + u)) : 0.0;
        cb[u] = ob ? __ldg(c1 + 32 * (k + u)) : -1;
        vb[u] = ob ? __ldg(v1 + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xa[u] = ca[u] >= 0 ? getx(ca[u]) : 0.0;  // warp-uniform conditions
        xb[u] = cb[u] >= 0 ? getx(cb[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(va[u], xa[u], a0);
        a1 = fma(vb[u], xb[u], a1);
      }
    }
    for (int o = (1 << g) >> 1; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if ((lane & ((1 << g) - 1)) == 0) {
      const int l0 = sa * rs + (lane >> g), l1 = sb * rs + (lane >> g);
      if (l0 < nloc) epi(l0, a0);
      if (hb && l1 < nloc) epi(l1, a1);
    }
  }
}

// own rows of y = A x (x = vector k of level xt, gathered over DSMEM),
// 4 lanes per row, four strides per pass with the value/column loads issued
// before the gathers; epi(local row, sum) on the lead lane
template <class F>
__device__ __forceinline__ void tail_spmv(const TailSh& s, const int* __restrict__ rp,
                                          const int* __restrict__ ci,
                                          const double* __restrict__ v, int r0, int nloc,
                                          const TL& xt, int k, F epi) {
  const int lane = threadIdx.x & 31, sub = lane & 3, grp = lane >> 2, wid = threadIdx.x >> 5;
  for (int base = wid * 8; base < nloc; base += kTailWarps * 8) {
    const int li = base + grp;
    double acc = 0.0;
    if (li < nloc) {
      const int row = r0 + li;
      const int beg = __ldg(rp + row), end = __ldg(rp + row + 1);
      for (int k0 = beg + sub; k0 < end; k0 += 16) {
        double vv[4], xv[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = k0 + 4 * u;
          vv[u] = kk < end ? __ldg(v + kk) : 0.0;
          cc[u] = kk < end ? __ldg(ci + kk) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = cc[u] >= 0 ? tl_get(s, xt, k, cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = fma(vv[u], xv[u], acc);
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (sub == 0 && li < nloc) epi(li, acc);
  }
}

__device__ __forceinline__ void tail_fin(TailSh& s, Fin f, double tot) {
  if (threadIdx.x == 0) {
    f.st = reinterpret_cast<KState*>(s.ks);
    apply_fin(f, tot);
  }
  __syncthreads();
}

// fgmres(A, b, x, jacobi, {tol 0, max 2, restart 2}) (amg.cpp:265-276,
// krylov.cpp:17-121) on level t, x in/out (x_zero: x is known to be zero)
__device__ void tail_smooth(cg::cluster_group& cl, TailSh& s, double* sm, int& slot,
                            const TailLevel& L, const TL& t, bool x_zero) {
  KState* st = reinterpret_cast<KState*>(s.ks);
  const int i0 = threadIdx.x, nloc = t.nloc;
  double* b = tl_vec(sm, t, TB);
  double* x = tl_vec(sm, t, TX);
  double* rs = tl_vec(sm, t, TRS);
  double* w = tl_vec(sm, t, TW);
  double* v0 = tl_vec(sm, t, TV0);
  double* v1 = tl_vec(sm, t, TV1);
  double* z0 = tl_vec(sm, t, TZ0);
  double* z1 = tl_vec(sm, t, TZ1);
  const double* dinv = L.dinv + t.r0;
  // ref = ||b|| and the (re)start residual r = b - A x, beta = ||r||
  {
    double red[2] = {0.0, 0.0};
    for (int i = i0; i < nloc; i += kTailThreads) red[0] = fma(b[i], b[i], red[0]);
    if (x_zero) {
      red[1] = red[0];
    } else {
      double acc = 0.0;
      tail_spmv(s, L.arp, L.aci, L.av, t.r0, nloc, t, TX, [&](int li, double sum) {
        const double ri = b[li] - sum;
        rs[li] = ri;
        acc = fma(ri, ri, acc);
      });
      red[1] = acc;
    }
    tail_reduce<2>(cl, s, slot, red);
    Fin f;
    f.kind = FIN_REF;
    tail_fin(s, f, red[0]);
    f.kind = FIN_BETA;
    f.i = 4;
    f.j = 2;
    f.tol = 0.0;
    tail_fin(s, f, red[1]);
  }
  const double* r = x_zero ? b : rs;
  if (!st->stop) {
    const double beta = st->beta;
    for (int i = i0; i < nloc; i += kTailThreads) {
      const double vi = r[i] / beta;
      v0[i] = vi;
      z0[i] = __ldg(dinv + i) * vi;
    }
    cluster_bar();
    // Arnoldi step 0: w = A z0, h00 = (w, v0); w -= h00 v0, ||w||
    {
      double red[1] = {0.0};
      tail_spmv(s, L.arp, L.aci, L.av, t.r0, nloc, t, TZ0, [&](int li, double sum) {
        w[li] = sum;
        red[0] = fma(sum, v0[li], red[0]);
      });
      tail_reduce<1>(cl, s, slot, red);
      Fin f;
      f.kind = FIN_H;
      f.i = 0;
      f.j = 0;
      tail_fin(s, f, red[0]);
    }
    {
      const double h = ks_h(st)[0];
      double red[1] = {0.0};
      for (int i = i0; i < nloc; i += kTailThreads) {
        const double wi = fma(-h, v0[i], w[i]);
        w[i] = wi;
        red[0] = fma(wi, wi, red[0]);
      }
      tail_reduce<1>(cl, s, slot, red);
      Fin f;
      f.kind = FIN_ARNOLDI;
      f.j = 0;
      tail_fin(s, f, red[0]);
    }
    if (!st->stop) {
      const double wn = st->wnorm;
      for (int i = i0; i < nloc; i += kTailThreads) {
        const double vi = w[i] / wn;
        v1[i] = vi;
        z1[i] = __ldg(dinv + i) * vi;
      }
      cluster_bar();
      // Arnoldi step 1: w = A z1, h01 = (w, v0); w -= h01 v0, h11 = (w, v1);
      // w -= h11 v1, ||w|| (v2 is never used by the update, so not formed)
      {
        double red[1] = {0.0};
        tail_spmv(s, L.arp, L.aci, L.av, t.r0, nloc, t, TZ1, [&](int li, double sum) {
          w[li] = sum;
          red[0] = fma(sum, v0[li], red[0]);
        });
        tail_reduce<1>(cl, s, slot, red);
        Fin f;
        f.kind = FIN_H;
        f.i = 0;
        f.j = 1;
        tail_fin(s, f, red[0]);
      }
      {
        const double h = ks_h(st)[1];
        double red[1] = {0.0};
        for (int i = i0; i < nloc; i += kTailThreads) {
          const double wi = fma(-h, v0[i], w[i]);
          w[i] = wi;
          red[0] = fma(wi, v1[i], red[0]);
        }
        tail_reduce<1>(cl, s, slot, red);
        Fin f;
        f.kind = FIN_H;
        f.i = 1;
        f.j = 1;
        tail_fin(s, f, red[0]);
      }
      {
        const double h = ks_h(st)[3];
        double red[1] = {0.0};
        for (int i = i0; i < nloc; i += kTailThreads) {
          const double wi = fma(-h, v1[i], w[i]);
          w[i] = wi;
          red[0] = fma(wi, wi, red[0]);
        }
        tail_reduce<1>(cl, s, slot, red);
        Fin f;
        f.kind = FIN_ARNOLDI;
        f.j = 1;
        tail_fin(s, f, red[0]);
      }
    }
  }
  // back-substitution (krylov.cpp:102-107) and x (+)= y_0 z_0 + y_1 z_1
  if (threadIdx.x == 0) {
    const int j = st->jeff, m = st->m;
    const double* h = ks_h(st);
    const double* g = ks_g(st);
    double* y = ks_y(st);
    for (int i = j - 1; i >= 0; --i) {
      double sum = g[i];
      for (int k = i + 1; k < j; ++k) sum -= h[i * m + k] * y[k];
      y[i] = sum / h[i * m + i];
    }
  }
  __syncthreads();
  const int j = st->jeff;
  if (j > 0 || x_zero) {
    const double* y = ks_y(st);
    for (int i = i0; i < nloc; i += kTailThreads) {
      double corr = 0.0;
      if (j > 0) corr = fma(y[0], z0[i], corr);
      if (j > 1) corr = fma(y[1], z1[i], corr);
      x[i] = x_zero ? corr : x[i] + corr;
    }
  }
  cluster_bar();
}

// diagnostic timestamps of tail CTA 0 inside sv_project_kernel (null otherwise)
struct TailTrace {
  unsigned long long* t = nullptr;
  int cap = 0;
  int* n = nullptr;
};
__device__ __forceinline__ void tail_mark(const TailTrace& tr, int tag) {
  if (tr.t && threadIdx.x == 0 && blockIdx.x == 0 && *tr.n < tr.cap) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    tr.t[2 * *tr.n] = (unsigned long long)tag;
    tr.t[2 * *tr.n + 1] = ns;
    ++*tr.n;
  }
}

// The cluster's whole pass: b0 (global) -> x0 (global). b0 may have been
// written earlier in the same launch (sv_project_kernel), so it is read
// through L2.
__device__ void tail_run(cg::cluster_group& cl, TailSh& s, double* sm, const TailParams& p,
                         const TailTrace& tr = TailTrace()) {
  const int q = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  if (threadIdx.x < cs) s.base[threadIdx.x] = cl.map_shared_rank(sm, (int)threadIdx.x);
  int slot = 0;
  const int nl = p.nlev;
  {
    const TL t = tl_make(p.L[0], q);
    double* b = tl_vec(sm, t, TB);
    for (int i = threadIdx.x; i < t.nloc; i += kTailThreads) b[i] = __ldcg(p.b0 + t.r0 + i);
  }
  cluster_bar();
  // down: pre-smoothing from zero, r = b - A x, b_(l+1) = R r
  for (int l = 0; l + 1 < nl; ++l) {
    const TailLevel& L = p.L[l];
    const TL t = tl_make(L, q);
    tail_mark(tr, 600 + l);
    tail_smooth(cl, s, sm, slot, L, t, true);
    tail_mark(tr, 610 + l);
    {
      const double* b = tl_vec(sm, t, TB);
      double* r = tl_vec(sm, t, TR);
      tail_spmv(s, L.arp, L.aci, L.av, t.r0, t.nloc, t, TX,
                [&](int li, double sum) { r[li] = b[li] - sum; });
    }
    cluster_bar();
    const TL tc = tl_make(p.L[l + 1], q);
    {
      double* bc = tl_vec(sm, tc, TB);
      tail_spmv(s, L.rrp, L.rci, L.rv, tc.r0, tc.nloc, t, TR,
                [&](int li, double sum) { bc[li] = sum; });
    }
    cluster_bar();
  }
  // coarse: x = K^-1 b (dense inverse), one warp per row
  tail_mark(tr, 620);
  {
    const TL tc = tl_make(p.L[nl - 1], q);
    double* xc = tl_vec(sm, tc, TX);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int li = wid; li < tc.nloc; li += kTailWarps) {
      const double* a = p.cinv + (size_t)(tc.r0 + li) * tc.n;
      double sum = 0.0;
      for (int j0 = lane; j0 < tc.n; j0 += 128) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + 32 * u;
          av[u] = j < tc.n ? __ldg(a + j) : 0.0;
          bv[u] = j < tc.n ? tl_get(s, tc, TB, j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) sum = fma(av[u], bv[u], sum);
      }
      sum = warp_sum(sum);
      if (lane == 0) xc[li] = sum;
    }
    cluster_bar();
  }
  // up: x_l += P x_(l+1), post-smoothing
  for (int l = nl - 2; l >= 0; --l) {
    const TailLevel& L = p.L[l];
    const TL t = tl_make(L, q);
    const TL tc = tl_make(p.L[l + 1], q);
    {
      double* x = tl_vec(sm, t, TX);
      tail_spmv(s, L.prp, L.pci, L.pv, t.r0, t.nloc, tc, TX,
                [&](int li, double sum) { x[li] = x[li] + sum; });
    }
    cluster_bar();
    tail_mark(tr, 630 + l);
    tail_smooth(cl, s, sm, slot, L, t, false);
    tail_mark(tr, 640 + l);
  }
  {
    const TL t = tl_make(p.L[0], q);
    const double* x = tl_vec(sm, t, TX);
    for (int i = threadIdx.x; i < t.nloc; i += kTailThreads) p.x0[t.r0 + i] = x[i];
  }
  // no CTA may go on (or exit) while another can still read its shared memory
  cluster_bar();
}

__global__ void __launch_bounds__(kTailThreads, 1) scalar_tail_kernel(TailParams p) {
  __shared__ TailSh s;
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  tail_run(cl, s, sm, p);
}

// -------------------------------------- SV mass projection, one launch --
// sv_project_kernel (internal.cuh: ProjParams). The pointwise vectors of a
// worker's rows live in its shared memory (every phase boundary below holds
// a __syncthreads); the gathered vectors are global and need a grid barrier
// between their producer and their consumers.

constexpr int kProjKsDoubles =
    10 + (kProjMaxRestart + 1) * kProjMaxRestart + 4 * kProjMaxRestart + 1;
static_assert(sizeof(KState) == 80, "KState header is 10 doubles");

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct ProjCtx {
  unsigned target;
  int slot;
  int wk, W;  // worker index (< 0: a CTA of the tail cluster), workers
  int nt;     // trace entries written (diagnostic)
  unsigned seq;  // reduction phase number
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// diagnostic: (tag, ns) pairs of worker 0 / tail CTA 0 when p.trace is set
__device__ __forceinline__ void proj_trace(const ProjParams& p, ProjCtx& g, int tag) {
  if (p.trace && threadIdx.x == 0 && (g.wk == 0 || blockIdx.x == 0) && g.nt < p.trace_cap) {
    unsigned long long* t = p.trace + (g.wk == 0 ? 0 : 2 * (size_t)p.trace_cap);
    t[2 * g.nt] = (unsigned long long)tag;
    t[2 * g.nt + 1] = globaltimer_ns();
    ++g.nt;
  }
}

// grid-wide barrier: every CTA adds one to a counter that only grows and
// waits for the launch's running target
__device__ __forceinline__ void grid_bar(const ProjParams& p, ProjCtx& g, int tag) {
  unsigned* bar = p.bar;
  g.target += gridDim.x;
  const unsigned target = g.target;
  proj_trace(p, g, tag);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    atomicAdd(bar, 1u);
    // watchdog: a CTA that waits ~2 s (a lost arrival: never seen, but a hang
    // would take the whole device) opens every barrier of the launch; the
    // caller sees the top bit of the counter and reports a failed projection
    const long long t0 = clock64();
    while (ld_acquire_u32(bar) < target) {
      if (clock64() - t0 > 4000000000LL) atomicOr(bar, 0x80000000u);
    }
  }
  __syncthreads();
  proj_trace(p, g, tag + 1000);
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// sum of v[k] over the grid, the same bits in every CTA, without a barrier:
// each worker publishes its block sum as two {32 bits of the value, phase}
// words (8-byte stores are single-copy atomic, so a word whose phase matches
// carries this phase's data); warp k of every CTA polls all workers' words of
// value k and sums them in worker order (lane-strided, then the shuffle
// tree). Slots alternate between two sets: a worker can be at most one phase
// ahead of the slowest CTA, which has then already read the older set.
template <int K>
__device__ __forceinline__ void grid_reduce(TailSh& s, const ProjParams& p, ProjCtx& g,
                                            double (&v)[K], int tag) {
  static_assert(K <= 2, "two values per reduction slot");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  proj_trace(p, g, tag);
  const unsigned seq = ++g.seq;
  unsigned long long* set = p.ll + (size_t)(seq & 1u) * g.W * 4;
  if (g.wk >= 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double t = warp_sum(v[k]);
      if (lane == 0) s.wp[wid][k] = t;
    }
    __syncthreads();
    if (wid < K) {
      const double t = warp_sum(s.wp[lane][wid]);
      if (lane < 2) {
        const unsigned half = lane == 0 ? (unsigned)__double2loint(t) : (unsigned)__double2hiint(t);
        st_relaxed_u64(set + (size_t)g.wk * 4 + wid * 2 + lane,
                       ((unsigned long long)seq << 32) | half);
      }
    }
  }
  if (wid < K) {
    // lane q polls workers q, q + 32, ..: all their words are loaded together
    // (one L2 round trip per poll), until every phase number matches
    constexpr int kMaxPer = 8;  // workers <= 256
    unsigned long long lo[kMaxPer], hi[kMaxPer];
    const long long t0 = clock64();
    unsigned spins = 0;
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int u = 0; u < kMaxPer; ++u) {
        const int q = lane + 32 * u;
        if (q < g.W) {
          const unsigned long long* a = set + (size_t)q * 4 + wid * 2;
          lo[u] = ld_relaxed_u64(a);
          hi[u] = ld_relaxed_u64(a + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < kMaxPer; ++u)
        if (lane + 32 * u < g.W)
          ok = ok && (unsigned)(lo[u] >> 32) == seq && (unsigned)(hi[u] >> 32) == seq;
      if (__all_sync(0xffffffffu, ok)) break;
      // watchdog (see grid_bar): give up when the launch was opened or after ~2 s
      if ((++spins & 255u) == 0u) {
        if (clock64() - t0 > 4000000000LL) atomicOr(p.bar, 0x80000000u);
        if (ld_acquire_u32(p.bar) & 0x80000000u) break;
      }
    }
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < kMaxPer; ++u)
      if (lane + 32 * u < g.W) t += __hiloint2double((int)(unsigned)hi[u], (int)(unsigned)lo[u]);
    t = warp_sum(t);
    if (lane == 0) s.tot[wid] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = s.tot[k];
  proj_trace(p, g, tag + 1000);
}

// a grid level's product: x in global memory. Plain (L1-cached) loads: every
// read of a gathered vector follows a grid barrier after its last write, and
// the barrier's acquire invalidates this SM's L1.
template <class F>
__device__ __forceinline__ void grid_spmv(const SellView& A, int r0, int nloc, const double* x,
                                          F epi) {
  sell_spmv(A, r0, nloc, [&](int col) { return x[col]; }, epi);
}

__device__ __forceinline__ void proj_fin(KState* st, Fin f, double tot) {
  if (threadIdx.x == 0) {
    f.st = st;
    apply_fin(f, tot);
  }
  __syncthreads();
}

__device__ __forceinline__ void proj_backsub(KState* st) {
  if (threadIdx.x == 0) {
    const int j = st->jeff, m = st->m;
    const double* h = ks_h(st);
    const double* g = ks_g(st);
    double* y = ks_y(st);
    for (int i = j - 1; i >= 0; --i) {
      double sum = g[i];
      for (int k = i + 1; k < j; ++k) sum -= h[(size_t)i * m + k] * y[k];
      y[i] = sum / h[(size_t)i * m + i];
    }
  }
  __syncthreads();
}

// a worker's rows of a level with n rows in chunks of `chunk`
struct Rows {
  int r0, nloc;
};
__device__ __forceinline__ Rows proj_rows(const ProjCtx& g, int n, int chunk) {
  Rows r;
  if (g.wk < 0) {
    r.r0 = n;
    r.nloc = 0;
  } else {
    r.r0 = min(n, g.wk * chunk);
    r.nloc = max(0, min(n - r.r0, chunk));
  }
  return r;
}

// fgmres(A, b, x, jacobi, {tol 0, max 2, restart 2}) on a grid level
// (amg.cpp:265-276; the operations of jacobi_fgmres2 / tail_smooth), b and x
// in global memory; x of the other workers is visible on entry (x_zero: x is
// known to be zero and is only written). The caller puts a grid barrier
// after it.
__device__ void grid_smooth(TailSh& s, double* sm, int cmax, const ProjParams& p, ProjCtx& g,
                            const ProjLevel& L, const double* bg, double* xg, bool x_zero) {
  KState* st = reinterpret_cast<KState*>(s.ks);
  const Rows R = proj_rows(g, L.n, L.chunk);
  const int r0 = R.r0, nloc = R.nloc, i0 = threadIdx.x;
  double* sb = sm;
  double* v0 = sm + cmax;
  double* v1 = sm + 2 * (size_t)cmax;
  double* w = sm + 3 * (size_t)cmax;
  const double* dinv = L.dinv + r0;
  {
    double red[2] = {0.0, 0.0};
    for (int i = i0; i < nloc; i += kTailThreads) {
      const double bi = __ldcg(bg + r0 + i);
      sb[i] = bi;
      red[0] = fma(bi, bi, red[0]);
    }
    if (x_zero) {
      red[1] = red[0];
    } else {
      __syncthreads();  // sb rows are read by the rows' SpMV lanes
      double acc = 0.0;
      grid_spmv(L.a, r0, nloc, xg, [&](int li, double sum) {
        const double ri = sb[li] - sum;
        sb[li] = ri;
        acc = fma(ri, ri, acc);
      });
      red[1] = acc;
    }
    grid_reduce<2>(s, p, g, red, 1);
    Fin f;
    f.kind = FIN_REF;
    proj_fin(st, f, red[0]);
    f.kind = FIN_BETA;
    f.i = 4;
    f.j = 2;
    f.tol = 0.0;
    proj_fin(st, f, red[1]);
  }
  if (!st->stop) {
    const double beta = st->beta;
    for (int i = i0; i < nloc; i += kTailThreads) {
      const double vi = sb[i] / beta;
      v0[i] = vi;
      L.z0[r0 + i] = __ldg(dinv + i) * vi;
    }
    grid_bar(p, g, 2);
    {
      double red[1] = {0.0};
      grid_spmv(L.a, r0, nloc, L.z0, [&](int li, double sum) {
        w[li] = sum;
        red[0] = fma(sum, v0[li], red[0]);
      });
      grid_reduce<1>(s, p, g, red, 3);
      Fin f;
      f.kind = FIN_H;
      f.i = 0;
      f.j = 0;
      proj_fin(st, f, red[0]);
    }
    {
      const double h = ks_h(st)[0];
      double red[1] = {0.0};
      for (int i = i0; i < nloc; i += kTailThreads) {
        const double wi = fma(-h, v0[i], w[i]);
        w[i] = wi;
        red[0] = fma(wi, wi, red[0]);
      }
      grid_reduce<1>(s, p, g, red, 4);
      Fin f;
      f.kind = FIN_ARNOLDI;
      f.j = 0;
      proj_fin(st, f, red[0]);
    }
    if (!st->stop) {
      const double wn = st->wnorm;
      for (int i = i0; i < nloc; i += kTailThreads) {
        const double vi = w[i] / wn;
        v1[i] = vi;
        L.z1[r0 + i] = __ldg(dinv + i) * vi;
      }
      grid_bar(p, g, 5);
      {
        double red[1] = {0.0};
        grid_spmv(L.a, r0, nloc, L.z1, [&](int li, double sum) {
          w[li] = sum;
          red[0] = fma(sum, v0[li], red[0]);
        });
        grid_reduce<1>(s, p, g, red, 6);
        Fin f;
        f.kind = FIN_H;
        f.i = 0;
        f.j = 1;
        proj_fin(st, f, red[0]);
      }
      {
        const double h = ks_h(st)[1];
        double red[1] = {0.0};
        for (int i = i0; i < nloc; i += kTailThreads) {
          const double wi = fma(-h, v0[i], w[i]);
          w[i] = wi;
          red[0] = fma(wi, v1[i], red[0]);
        }
        grid_reduce<1>(s, p, g, red, 7);
        Fin f;
        f.kind = FIN_H;
        f.i = 1;
        f.j = 1;
        proj_fin(st, f, red[0]);
      }
      {
        const double h = ks_h(st)[3];
        double red[1] = {0.0};
        for (int i = i0; i < nloc; i += kTailThreads) {
          const double wi = fma(-h, v1[i], w[i]);
          w[i] = wi;
          red[0] = fma(wi, wi, red[0]);
        }
        grid_reduce<1>(s, p, g, red, 8);
        Fin f;
        f.kind = FIN_ARNOLDI;
        f.j = 1;
        proj_fin(st, f, red[0]);
      }
    }
  }
  proj_backsub(st);
  const int j = st->jeff;
  if (j > 0 || x_zero) {
    const double y0 = ks_y(st)[0], y1 = ks_y(st)[1];
    for (int i = i0; i < nloc; i += kTailThreads) {
      const double di = __ldg(dinv + i);
      double corr = 0.0;
      if (j > 0) corr = fma(y0, di * v0[i], corr);
      if (j > 1) corr = fma(y1, di * v1[i], corr);
      xg[r0 + i] = x_zero ? corr : __ldcg(xg + r0 + i) + corr;
    }
  }
}

// x = V(2,2) b on the scalar hierarchy from x = 0 (amg.cpp:258-296): grid
// levels here, the rest in cluster 0. Ends with x visible grid-wide.
__device__ void proj_vcycle(cg::cluster_group& cl, TailSh& s, double* sm, int cmax,
                            const ProjParams& p, ProjCtx& g, const double* b0, double* x0) {
  const int ngl = p.ngl;
  for (int l = 0; l < ngl; ++l) {
    const ProjLevel& L = p.G[l];
    const double* bg = l == 0 ? b0 : L.b;
    double* xg = l == 0 ? x0 : L.x;
    grid_smooth(s, sm, cmax, p, g, L, bg, xg, true);
    grid_bar(p, g, 9);
    const Rows R = proj_rows(g, L.n, L.chunk);
    grid_spmv(L.a, R.r0, R.nloc, xg, [&](int li, double sum) {
      L.r[R.r0 + li] = __ldcg(bg + R.r0 + li) - sum;
    });
    grid_bar(p, g, 10);
    const Rows C = proj_rows(g, L.nc, L.cchunk);
    double* bc = l + 1 < ngl ? p.G[l + 1].b : const_cast<double*>(p.tail.b0);
    grid_spmv(L.rt, C.r0, C.nloc, L.r,
              [&](int li, double sum) { bc[C.r0 + li] = sum; });
    grid_bar(p, g, 11);
  }
  if (g.wk < 0) {
    proj_trace(p, g, 500);
    TailTrace tr;
    if (p.trace && blockIdx.x == 0) {
      tr.t = p.trace + 2 * (size_t)p.trace_cap;
      tr.cap = p.trace_cap;
      tr.n = &g.nt;
    }
    tail_run(cl, s, sm, p.tail, tr);
    proj_trace(p, g, 501);
  }
  grid_bar(p, g, 12);
  for (int l = ngl - 1; l >= 0; --l) {
    const ProjLevel& L = p.G[l];
    const double* bg = l == 0 ? b0 : L.b;
    double* xg = l == 0 ? x0 : L.x;
    const double* xc = l + 1 < ngl ? p.G[l + 1].x : p.tail.x0;
    const Rows R = proj_rows(g, L.n, L.chunk);
    grid_spmv(L.p, R.r0, R.nloc, xc, [&](int li, double sum) {
      xg[R.r0 + li] = __ldcg(xg + R.r0 + li) + sum;
    });
    grid_bar(p, g, 13);
    grid_smooth(s, sm, cmax, p, g, L, bg, xg, false);
    grid_bar(p, g, 14);
  }
}

__global__ void __launch_bounds__(kTailThreads, 1) sv_project_kernel(ProjParams p) {
  __shared__ TailSh s;
  __shared__ double oks[kProjKsDoubles];
  extern __shared__ double sm[];
  if (p.ngl <= 0) return;  // plan-time probe of the launch configuration
  cg::cluster_group cl = cg::this_cluster();
  ProjCtx g;
  g.target = 0u;
  g.slot = 0;
  g.nt = 0;
  g.seq = 0u;
  g.W = p.workers;
  g.wk = (int)blockIdx.x - (int)cl.num_blocks();  // cluster 0 = the tail
  KState* ost = reinterpret_cast<KState*>(oks);
  const ProjLevel& L0 = p.G[0];
  const int n = p.n, i0 = threadIdx.x;
  int cmax = 0;
  for (int l = 0; l < p.ngl; ++l) cmax = max(cmax, p.G[l].chunk);
  const Rows R = proj_rows(g, n, L0.chunk);
  const int r0 = R.r0, nloc = R.nloc;
  double* sb = sm;                      // the restart residual (own rows)
  double* sw = sm + 3 * (size_t)cmax;   // Arnoldi w (own rows)
  // rhs = M_mix p_dg (transfer.cpp:24), x = 0; ref = ||rhs|| (krylov.cpp:23-24)
  double tot0;
  {
    double red[1] = {0.0};
    grid_spmv(p.mm, r0, nloc, p.p_dg, [&](int li, double sum) {
      p.rhs[r0 + li] = sum;
      p.x[r0 + li] = 0.0;
      red[0] = fma(sum, sum, red[0]);
    });
    grid_reduce<1>(s, p, g, red, 15);
    tot0 = red[0];
    if (threadIdx.x == 0) {
      ost->ref = 1.0;
      ost->tol = p.tol;
      ost->bd = p.bd;
      ost->m = p.restart;
      ost->stop = 0;
      ost->breakdown = 0;
      ost->jeff = 0;
      ost->iterations = 0;
      ost->hist_len = 0;
      ost->hist_cap = 0;
      ost->converged = 0;
      ost->beta = 0.0;
      ost->rnorm = 0.0;
    }
    __syncthreads();
    Fin f;
    f.kind = FIN_REF;
    proj_fin(ost, f, tot0);
    f.kind = FIN_BETA;  // the initial residual b - A 0 = b (krylov.cpp:26-35)
    f.i = 2;
    proj_fin(ost, f, tot0);
  }
  const int m = p.restart;
  bool first = true;
  while (!ost->converged && ost->iterations < p.max_iters) {
    // (re)start from the true residual (krylov.cpp:43-53)
    {
      Fin f;
      f.kind = FIN_BETA;
      f.i = 0;
      if (first) {
        for (int i = i0; i < nloc; i += kTailThreads) sb[i] = __ldcg(p.rhs + r0 + i);
        proj_fin(ost, f, tot0);
      } else {
        double red[1] = {0.0};
        grid_spmv(L0.a, r0, nloc, p.x, [&](int li, double sum) {
          const double ri = __ldcg(p.rhs + r0 + li) - sum;
          sb[li] = ri;
          red[0] = fma(ri, ri, red[0]);
        });
        grid_reduce<1>(s, p, g, red, 16);
        proj_fin(ost, f, red[0]);
      }
    }
    if (ost->stop) break;
    {
      const double beta = ost->beta;
      for (int i = i0; i < nloc; i += kTailThreads) p.V[r0 + i] = sb[i] / beta;
    }
    for (int j = 0; j < m && !ost->stop && ost->iterations < p.max_iters; ++j) {
      double* zj = p.Z + (size_t)j * n;
      proj_vcycle(cl, s, sm, cmax, p, g, p.V + (size_t)j * n, zj);
      // Arnoldi step j (krylov.cpp:61-100): w = A z_j, modified Gram-Schmidt
      {
        double red[1] = {0.0};
        grid_spmv(L0.a, r0, nloc, zj, [&](int li, double sum) {
          sw[li] = sum;
          red[0] = fma(sum, __ldcg(p.V + r0 + li), red[0]);
        });
        grid_reduce<1>(s, p, g, red, 17);
        Fin f;
        f.kind = FIN_H;
        f.i = 0;
        f.j = j;
        proj_fin(ost, f, red[0]);
      }
      for (int i = 1; i <= j; ++i) {
        const double h = ks_h(ost)[(size_t)(i - 1) * m + j];
        const double* vp = p.V + (size_t)(i - 1) * n + r0;
        const double* vn = p.V + (size_t)i * n + r0;
        double red[1] = {0.0};
        for (int k = i0; k < nloc; k += kTailThreads) {
          const double wi = fma(-h, __ldcg(vp + k), sw[k]);
          sw[k] = wi;
          red[0] = fma(wi, __ldcg(vn + k), red[0]);
        }
        grid_reduce<1>(s, p, g, red, 18);
        Fin f;
        f.kind = FIN_H;
        f.i = i;
        f.j = j;
        proj_fin(ost, f, red[0]);
      }
      {
        const double h = ks_h(ost)[(size_t)j * m + j];
        const double* vj = p.V + (size_t)j * n + r0;
        double red[1] = {0.0};
        for (int k = i0; k < nloc; k += kTailThreads) {
          const double wi = fma(-h, __ldcg(vj + k), sw[k]);
          sw[k] = wi;
          red[0] = fma(wi, wi, red[0]);
        }
        grid_reduce<1>(s, p, g, red, 19);
        Fin f;
        f.kind = FIN_ARNOLDI;
        f.j = j;
        proj_fin(ost, f, red[0]);
      }
      if (!ost->stop) {
        const double wn = ost->wnorm;
        double* vq = p.V + (size_t)(j + 1) * n + r0;
        for (int k = i0; k < nloc; k += kTailThreads) vq[k] = sw[k] / wn;
      }
    }
    // back-substitution and x += sum_i y_i z_i (krylov.cpp:102-110)
    proj_backsub(ost);
    {
      const int jj = ost->jeff;
      const double* y = ks_y(ost);
      if (jj > 0) {
        for (int k = i0; k < nloc; k += kTailThreads) {
          double corr = 0.0;
          for (int i = 0; i < jj; ++i) corr = fma(y[i], __ldcg(p.Z + (size_t)i * n + r0 + k), corr);
          p.x[r0 + k] = __ldcg(p.x + r0 + k) + corr;
        }
      }
    }
    first = false;
    grid_bar(p, g, 20);
  }
  proj_trace(p, g, 9999);
  if (blockIdx.x == 0) {
    double* out = reinterpret_cast<double*>(p.st);
    for (int i = i0; i < kProjKsDoubles; i += kTailThreads) out[i] = oks[i];
    __syncthreads();
    if (threadIdx.x == 0 && (!ost->converged || (ld_acquire_u32(p.bar) & 0x80000000u))) {
      *p.fail = 1;
      reinterpret_cast<KState*>(out)->converged = 0;
    }
  }
}

static void proj_launch_cfg(const ProjParams& p, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at,
                            bool coop) {
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = p.smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.tail.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop ? 2 : 1;
}

static bool g_proj_coop = true;

bool sv_project_plan(Ctx& c, ProjParams& p) {
  if (p.ngl < 1 || p.ngl > kProjMaxGl || p.tail.cs <= 0 || p.tail.nlev < 1) return false;
  if (p.restart < 1 || p.restart > kProjMaxRestart) return false;
  constexpr size_t kMaxSmem = 200 * 1024;
  static bool attr[64] = {};
  int dev = 0;
  SAG_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !attr[dev]) {
    if (cudaFuncSetAttribute(sv_project_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess)
      cudaGetLastError();
    if (cudaFuncSetAttribute(sv_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMaxSmem) != cudaSuccess)
      cudaGetLastError();
    attr[dev] = true;
  }
  const int cs = p.tail.cs;
  p.smem = p.tail.smem;
  for (int pass = 0; pass < 3; ++pass) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    p.grid = cs;
    proj_launch_cfg(p, cfg, at, false);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, sv_project_kernel, &cfg) != cudaSuccess || nc < 2) {
      cudaGetLastError();
      return false;
    }
    const char* e = getenv("SAG_PROJ_CLUSTERS");
    if (e && atoi(e) >= 2) nc = std::min(nc, atoi(e));
    p.grid = nc * cs;
    p.workers = p.grid - cs;
    int cmax = 0;
    for (int l = 0; l < p.ngl; ++l) {
      ProjLevel& L = p.G[l];
      L.chunk = ((L.n + p.workers - 1) / p.workers + 31) & ~31;
      L.cchunk = ((L.nc + p.workers - 1) / p.workers + 31) & ~31;
      cmax = std::max(cmax, L.chunk);
    }
    const size_t need = std::max(p.tail.smem, (size_t)4 * cmax * sizeof(double));
    if (need > kMaxSmem) return false;
    if (need == p.smem) break;
    if (pass == 2) return false;
    p.smem = need;
  }
  // probe the launch configuration once (cooperative + cluster); fall back
  // to a plain cluster launch of a grid that is co-resident by construction
  ProjParams probe = p;
  probe.ngl = 0;
  const char* ec = getenv("SAG_PROJ_COOP");
  g_proj_coop = !(ec && std::strcmp(ec, "0") == 0);
  for (int attempt = 0; attempt < 2; ++attempt) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    proj_launch_cfg(p, cfg, at, g_proj_coop);
    cfg.stream = c.stream;
    cudaError_t e = cudaLaunchKernelEx(&cfg, sv_project_kernel, probe);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e == cudaSuccess) return true;
    cudaGetLastError();
    if (!g_proj_coop) return false;
    g_proj_coop = false;
  }
  return false;
}

void launch_sv_project(Ctx& c, const ProjParams& p) {
  SAG_REQUIRE(p.grid > 0 && p.ngl >= 1 && p.p_dg && p.x && p.bar && p.ll, SAG_ERROR,
              "SV mass projection: not planned");
  SAG_CUDA(cudaMemsetAsync(p.bar, 0, p.sync_bytes, c.stream));
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute at[2];
  proj_launch_cfg(p, cfg, at, g_proj_coop);
  cfg.stream = c.stream;
  SAG_CUDA(cudaLaunchKernelEx(&cfg, sv_project_kernel, p));
  SAG_LAUNCHED(c);
}


bool scalar_tail_plan(Ctx& c, TailParams& p) {
  (void)c;
  if (p.nlev < 1 || p.nlev > kTailMaxLev) return false;
  // function attributes are per device
  static bool attr[64] = {};
  int dev = 0;
  SAG_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !attr[dev]) {
    if (cudaFuncSetAttribute(scalar_tail_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess)
      cudaGetLastError();
    if (cudaFuncSetAttribute(scalar_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024) != cudaSuccess)
      cudaGetLastError();
    attr[dev] = true;
  }
  // SAG_TAIL_CS (diagnostic): one cluster size instead of 16, then 8
  const char* ecs = getenv("SAG_TAIL_CS");
  const int force_cs = ecs ? atoi(ecs) : 0;
  for (int cs : {16, 8, 4, 2, 1}) {
    if (force_cs > 0 ? cs != force_cs : cs < 8) continue;
    size_t off = 0;
    for (int l = 0; l < p.nlev; ++l) {
      TailLevel& L = p.L[l];
      L.chunk = (L.n + cs - 1) / cs;
      L.off = (int)off;
      off += (size_t)kTailVecs * L.chunk;
    }
    const size_t bytes = off * sizeof(double);
    if (bytes > 200 * 1024) continue;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, scalar_tail_kernel, &cfg) == cudaSuccess && nc > 0) {
      p.cs = cs;
      p.smem = bytes;
      return true;
    }
    cudaGetLastError();
  }
  return false;
}

void launch_scalar_tail(Ctx& c, const TailParams& p) {
  SAG_REQUIRE(p.cs > 0 && p.nlev >= 1 && p.nlev <= kTailMaxLev && p.b0 && p.x0, SAG_ERROR,
              "scalar V-cycle tail: not planned");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.cs);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SAG_CUDA(cudaLaunchKernelEx(&cfg, scalar_tail_kernel, p));
  SAG_LAUNCHED(c);
}

}  // namespace sag

// =================================================================== C-ABI

using sag::Ctx;

namespace {
thread_local std::string g_last_error;
}
namespace sag {
void set_last_error(const std::string& s) { g_last_error = s; }
}  // namespace sag
using sag::guard;
#define NOTNULL SAG_NOTNULL

extern "C" {

const char* sag_last_error(void) { return g_last_error.c_str(); }

static int create_ctx(int device, cudaStream_t stream, sag_ctx** out);

int sag_create(int device, sag_ctx** out) { return create_ctx(device, nullptr, out); }

int sag_create_on_stream(int device, void* stream, sag_ctx** out) {
  if (!stream) {
    sag::set_last_error("sag_create_on_stream: null stream");
    return SAG_INVALID_ARGUMENT;
  }
  return create_ctx(device, static_cast<cudaStream_t>(stream), out);
}

static int create_ctx(int device, cudaStream_t stream, sag_ctx** out) {
  return guard([&] {
    NOTNULL(out);
    *out = nullptr;
    int ndev = 0;
    SAG_CUDA(cudaGetDeviceCount(&ndev));
    SAG_REQUIRE(device >= 0 && device < ndev, SAG_CUDA_ERROR, "sag_create: no such CUDA device");
    cudaDeviceProp prop;
    SAG_CUDA(cudaGetDeviceProperties(&prop, device));
    SAG_REQUIRE(prop.major == 10, SAG_CUDA_ERROR,
                std::string("sag_create: libsag is built for sm_100a, device is ") + prop.name);
    SAG_CUDA(cudaSetDevice(device));
    auto* h = new sag_ctx;
    h->c.device = device;
    h->c.num_sms = prop.multiProcessorCount;
    if (stream) {
      h->c.stream = stream;
      h->c.own_stream = false;
    } else {
      SAG_CUDA(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking));
    }
    h->c.partials.alloc(sag::kMaxRedGrid * 2);
    h->c.ticket.alloc(64);
    SAG_CUDA(cudaMemset(h->c.ticket.p, 0, sizeof(unsigned) * 64));
    h->c.scal.alloc(64);
    *out = h;
  });
}

int sag_destroy(sag_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.copy_stream) {
      cudaStreamSynchronize(ctx->c.copy_stream);
      cudaStreamDestroy(ctx->c.copy_stream);
      cudaEventDestroy(ctx->c.copy_ev);
    }
    for (cudaStream_t bs : ctx->c.body_streams)
      if (bs) cudaStreamDestroy(bs);
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
  });
}

int sag_synchronize(sag_ctx* ctx) {
  return guard([&] {
    NOTNULL(ctx);
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sag_alloc(sag_ctx* ctx, size_t bytes, void** dptr) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(dptr);
    SAG_CUDA(cudaSetDevice(ctx->c.device));
    SAG_CUDA(cudaMalloc(dptr, bytes ? bytes : 1));
  });
}

int sag_free(sag_ctx* ctx, void* dptr) {
  return guard([&] {
    NOTNULL(ctx);
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    SAG_CUDA(cudaFree(dptr));
  });
}

int sag_memcpy(sag_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    NOTNULL(ctx);
    SAG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->c.stream));
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sag_launch_count(sag_ctx* ctx, long long* out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(out);
    *out = ctx->c.launches;
  });
}

int sag_stream(sag_ctx* ctx, void** stream) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(stream);
    *stream = (void*)ctx->c.stream;
  });
}

int sag_matrix_create(sag_ctx* ctx, int nrows, int ncols, long long nnz, const int* row_offsets,
                      const int* col_indices, const double* values, sag_matrix** out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(out);
    *out = nullptr;
    auto m = sag::matrix_upload(ctx->c, nrows, ncols, nnz, row_offsets, col_indices, values);
    auto* h = new sag_matrix;
    h->m = std::move(*m);
    *out = h;
  });
}

int sag_matrix_destroy(sag_matrix* m) {
  return guard([&] {
    if (m) cudaDeviceSynchronize();  // no kernel or graph still reads it
    delete m;
  });
}

int sag_matrix_shape(const sag_matrix* m, int* nrows, int* ncols, long long* nnz) {
  return guard([&] {
    NOTNULL(m);
    if (nrows) *nrows = m->m.nrows;
    if (ncols) *ncols = m->m.ncols;
    if (nnz) *nnz = m->m.nnz;
  });
}

int sag_spmv(sag_ctx* ctx, const sag_matrix* m, const double* x, double* y) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(m);
    auto& c = ctx->c;
    sag::InVec xi(c, x, m->m.ncols, 0);
    sag::OutVec yo(c, y, m->m.nrows, 1, false);
    sag::launch_spmv(c, m->m, xi.d, yo.d, sag::Epi::Store);
    yo.finish();
  });
}

int sag_spmv_fused(sag_ctx* ctx, const sag_matrix* m, const double* x, double* y,
                   const double* aux, int epilogue) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(m);
    auto& c = ctx->c;
    SAG_REQUIRE(sag::is_device_ptr(x) && sag::is_device_ptr(y) &&
                    (aux == nullptr || sag::is_device_ptr(aux)),
                SAG_INVALID_ARGUMENT, "sag_spmv_fused takes device pointers");
    sag::SpmvArgs a;
    a.b = aux;
    a.dotv = aux;
    sag::Epi e;
    switch (epilogue) {
      case 0: e = sag::Epi::Store; break;
      case 1: e = sag::Epi::Resid; break;
      case 2: e = sag::Epi::Add; break;
      case 3:
        e = sag::Epi::StoreDot;
        a.fin.kind = sag::FIN_STORE;
        a.fin.out = c.scal.p;
        break;
      case 4:
        e = sag::Epi::ResidSsq;
        a.fin.kind = sag::FIN_SQRT;
        a.fin.out = c.scal.p;
        break;
      default: throw sag::Error(SAG_CONFIG_ERROR, "sag_spmv_fused: unknown epilogue");
    }
    SAG_REQUIRE(epilogue == 0 || epilogue == 2 || aux, SAG_INVALID_ARGUMENT, "aux vector needed");
    sag::launch_spmv(c, m->m, x, y, e, a);
  });
}

int sag_norm2(sag_ctx* ctx, int n, const double* v, double* out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(out);
    auto& c = ctx->c;
    sag::InVec vi(c, v, n, 0);
    sag::Fin f;
    f.kind = sag::FIN_SQRT;
    f.out = c.scal.p;
    sag::launch_ssq(c, n, vi.d, f);
    SAG_CUDA(cudaMemcpyAsync(out, c.scal.p, sizeof(double), cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_dot(sag_ctx* ctx, int n, const double* a, const double* b, double* out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(out);
    auto& c = ctx->c;
    sag::InVec ai(c, a, n, 0);
    sag::InVec bi(c, b, n, 1);
    sag::Fin f;
    f.kind = sag::FIN_STORE;
    f.out = c.scal.p;
    sag::launch_dot(c, n, ai.d, bi.d, f);
    SAG_CUDA(cudaMemcpyAsync(out, c.scal.p, sizeof(double), cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

// ---- partitioned-solve primitives (device pointers, no host sync) ----------
static void require_dev(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    SAG_REQUIRE(p == nullptr || sag::is_device_ptr(p), SAG_INVALID_ARGUMENT,
                "partitioned-solve primitives take device pointers");
}

int sag_dot_async(sag_ctx* ctx, int n, const double* a, const double* b,
                  const unsigned char* mask, double* out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(out);
    require_dev({a, b, mask, out});
    auto& c = ctx->c;
    sag::Fin f;
    f.kind = sag::FIN_STORE;
    f.out = out;
    sag::dot_mask_kernel<<<sag::red_grid_fit(c, sag::dot_mask_kernel, n), sag::kRedBlock, 0,
                           c.stream>>>(n, a, b, mask, f, c.partials.p, c.ticket.p);
    SAG_LAUNCHED(c);
  });
}

int sag_axpy_async(sag_ctx* ctx, int n, const double* s, double sign, const double* x, double* y) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({s, x, y});
    auto& c = ctx->c;
    sag::axpy_dev_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, s, sign, x, y);
    SAG_LAUNCHED(c);
  });
}

int sag_div_async(sag_ctx* ctx, int n, const double* x, const double* s, int take_sqrt, double* y) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({x, s, y});
    auto& c = ctx->c;
    sag::div_dev_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, x, s, take_sqrt, y);
    SAG_LAUNCHED(c);
  });
}

int sag_fgmres1_coef_async(sag_ctx* ctx, const double* ssq_r, const double* h00,
                           const double* ssq_w, double* y0) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({ssq_r, h00, ssq_w, y0});
    auto& c = ctx->c;
    sag::fgmres1_coef_kernel<<<1, 1, 0, c.stream>>>(ssq_r, h00, ssq_w, y0);
    SAG_LAUNCHED(c);
  });
}

int sag_sub_mean_async(sag_ctx* ctx, int n, const double* x, const double* sum, double count,
                       double* y) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({x, sum, y});
    auto& c = ctx->c;
    sag::sub_mean_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, x, sum, count, y);
    SAG_LAUNCHED(c);
  });
}

int sag_axpby_async(sag_ctx* ctx, int n, double a, const double* x, double b, double* y) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({x, y});
    auto& c = ctx->c;
    sag::axpby_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, a, x, b, y);
    SAG_LAUNCHED(c);
  });
}

int sag_gather_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* dst) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({idx, src, dst});
    if (n <= 0) return;
    auto& c = ctx->c;
    sag::gather_idx_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, idx, src, dst);
    SAG_LAUNCHED(c);
  });
}

int sag_push_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* peer_dst) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({idx, src, peer_dst});
    if (n <= 0) return;
    auto& c = ctx->c;
    sag::push_idx_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, idx, src, peer_dst);
    SAG_LAUNCHED(c);
  });
}

int sag_scatter_async(sag_ctx* ctx, int n, const int* idx, const double* src, double* dst, int add) {
  return guard([&] {
    NOTNULL(ctx);
    require_dev({idx, src, dst});
    if (n <= 0) return;
    auto& c = ctx->c;
    sag::scatter_idx_kernel<<<sag::ew_grid(c, n), 256, 0, c.stream>>>(n, idx, src, dst, add);
    SAG_LAUNCHED(c);
  });
}

int sag_ipc_get_handle(sag_ctx* ctx, void* dptr, unsigned char* handle) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(dptr);
    NOTNULL(handle);
    cudaIpcMemHandle_t h;
    SAG_CUDA(cudaIpcGetMemHandle(&h, dptr));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, sizeof(h));
  });
}

int sag_ipc_open_handle(sag_ctx* ctx, const unsigned char* handle, void** dptr) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(handle);
    NOTNULL(dptr);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    SAG_CUDA(cudaSetDevice(ctx->c.device));
    SAG_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int sag_ipc_close_handle(sag_ctx* ctx, void* dptr) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(dptr);
    SAG_CUDA(cudaIpcCloseMemHandle(dptr));
  });
}

int sag_matrix_norm_inf(sag_ctx* ctx, const sag_matrix* m, double* out) {
  return guard([&] {
    NOTNULL(ctx);
    NOTNULL(m);
    NOTNULL(out);
    auto& mm = const_cast<sag_matrix*>(m)->m;
    sag::compute_norm_inf(ctx->c, mm);
    *out = mm.norm_inf;
  });
}

}  // extern "C"
