// libsag setup module: the sparse products of the smoothed-aggregation
// hierarchy setup on the device, BITWISE equal to the reference:
//   spgemm            sparse.cpp:113-150
//   galerkin_triple   sparse.cpp:152-156   (spgemm(transpose(P), spgemm(K, P)))
//   smooth_prolongator amg.cpp:226-236     (T - (omega D^-1) (A T), omega from the caller)
//   transpose         sparse.cpp:93-111
// The setup is discrete and rounding-sensitive: entries that cancel
// to exactly 0.0 are dropped, so every product must be summed in the
// reference's order with round-to-nearest multiplies and adds (no FMA
// contraction). spgemm accumulates accum[col] += a_rk * b_kc over the entries
// of A's row in order; each B row holds a column at most once, so every output
// entry is a sequential sum in A-row order. One warp per output row: the warp
// walks A's row entry by entry and its lanes add that entry's B-row products
// into a shared-memory hash table (distinct columns within one step, so no
// two lanes touch one slot); the row's columns are then ranked, zeros dropped,
// and written in ascending order. Two passes: row counts, then the rows.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "internal.cuh"

namespace sag {

// Per-warp tables are sized per launch from the largest row (a pre-pass):
// a power of two >= 2x the row's products, so CTAs hold as many warps as the
// shared memory allows (4096 slots at most).
constexpr int kSetupMaxCap = 4096;
constexpr int kSpgSlot = 4 + 8 + 4 + 8;  // key, value, listed column, listed value
constexpr int kSetupSmem = 200 * 1024;

// upper bound of the distinct columns of each output row (mode 0, spgemm:
// sum of the B-row lengths over A's row) or of a column's 2-step support
// (mode 1, evolution_soc: 1 + deg(j) + sum of its neighbours' degrees); max
__global__ void max_est_kernel(int nrows, const int* __restrict__ arp,
                               const int* __restrict__ aci, const int* __restrict__ brp, int mode,
                               int* __restrict__ out) {
  int best = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    int e = mode ? 1 + arp[r + 1] - arp[r] : 0;
    for (int q = arp[r]; q < arp[r + 1]; ++q) {
      const int j = aci[q];
      e += brp[j + 1] - brp[j];
    }
    best = max(best, e);
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

static int table_cap(Ctx& c, int nrows, const int* arp, const int* aci, const int* brp, int mode) {
  DevBuf<int> m(1);
  SAG_CUDA(cudaMemsetAsync(m.p, 0, sizeof(int), c.stream));
  const int g = std::max(1, std::min((nrows + 255) / 256, c.num_sms * 8));
  max_est_kernel<<<g, 256, 0, c.stream>>>(nrows, arp, aci, brp, mode, m.p);
  SAG_LAUNCHED(c);
  int h = 0;
  SAG_CUDA(cudaMemcpyAsync(&h, m.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  int cap = 64;
  while (cap < 2 * h && cap < kSetupMaxCap) cap <<= 1;
  return cap;
}

// one output row r of C = A B into the warp's table; returns the count of
// distinct columns (cnt) with lc / lv the compacted (column, value) lists
__device__ __forceinline__ int spg_row(int r, const int* __restrict__ arp,
                                       const int* __restrict__ aci, const double* __restrict__ av,
                                       const int* __restrict__ brp, const int* __restrict__ bci,
                                       const double* __restrict__ bv, int capw, int* keys,
                                       double* vals, int* lc, double* lv, int* counter,
                                       int* overflow) {
  const int lane = threadIdx.x & 31;
  // table size: a power of two >= 2x the row's products (at most capw)
  int prod = 0;
  for (int ka = arp[r] + lane; ka < arp[r + 1]; ka += 32) {
    const int j = aci[ka];
    prod += brp[j + 1] - brp[j];
  }
  for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
  int cap = 64;
  while (cap < 2 * prod && cap < capw) cap <<= 1;
  const unsigned mask = cap - 1;
  for (int s = lane; s < cap; s += 32) keys[s] = -1;
  if (lane == 0) *counter = 0;
  __syncwarp();
  bool full = false;
  for (int ka = arp[r]; ka < arp[r + 1]; ++ka) {
    const int j = aci[ka];
    const double a = av[ka];
    for (int kb = brp[j] + lane; kb < brp[j + 1]; kb += 32) {
      const int col = bci[kb];
      unsigned h = ((unsigned)col * 2654435761u) & mask;
      int probes = 0;
      while (true) {
        const int k = atomicCAS(keys + h, -1, col);
        if (k == -1) {
          vals[h] = 0.0;  // accum[col] = 0.0 on first touch (sparse.cpp:128-131)
          break;
        }
        if (k == col) break;
        h = (h + 1) & mask;
        if (++probes >= cap) {
          full = true;
          break;
        }
      }
      if (!full) vals[h] = __dadd_rn(vals[h], __dmul_rn(a, bv[kb]));
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, full)) {
    if (lane == 0) atomicOr(overflow, 1);
    return 0;
  }
  for (int s = lane; s < cap; s += 32) {
    if (keys[s] != -1) {
      const int p = atomicAdd(counter, 1);
      lc[p] = keys[s];
      lv[p] = vals[s];
    }
  }
  __syncwarp();
  return *counter;
}

// pass 0: nonzero count per row; pass 1: the row, columns ascending, exact
// zeros dropped (sparse.cpp:140-146)
__global__ void __launch_bounds__(512) spgemm_kernel(
    int nrows, const int* __restrict__ arp, const int* __restrict__ aci,
    const double* __restrict__ av, const int* __restrict__ brp, const int* __restrict__ bci,
    const double* __restrict__ bv, int capw, int pass, int* __restrict__ row_nnz,
    const int* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv, int* overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  unsigned char* base = smem + (size_t)wib * capw * kSpgSlot;
  double* vals = reinterpret_cast<double*>(base);
  double* lv = vals + capw;
  int* keys = reinterpret_cast<int*>(lv + capw);
  int* lc = keys + capw;
  __shared__ int counters[16];
  const int gw = blockIdx.x * warps + wib, nw = gridDim.x * warps;
  for (int r = gw; r < nrows; r += nw) {
    const int cnt = spg_row(r, arp, aci, av, brp, bci, bv, capw, keys, vals, lc, lv,
                            counters + wib, overflow);
    int nz = 0;
    for (int e = lane; e < cnt; e += 32) nz += lv[e] != 0.0;
    for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    if (pass == 0) {
      if (lane == 0) row_nnz[r] = nz;
    } else {
      const int o0 = crp[r];
      for (int e = lane; e < cnt; e += 32) {
        const double v = lv[e];
        if (v == 0.0) continue;
        const int c = lc[e];
        int rank = 0;
        for (int f = 0; f < cnt; ++f) rank += (lc[f] < c) & (lv[f] != 0.0);
        cci[o0 + rank] = c;
        cv[o0 + rank] = v;
      }
    }
    __syncwarp();
  }
}

// warps per CTA for a per-warp table of `bytes`, and the grid over `rows`
static int setup_warps(int bytes) { return std::max(1, std::min(16, kSetupSmem / bytes)); }
static int setup_grid(Ctx& c, long long rows, int warps) {
  const long long need = (rows + warps - 1) / warps;
  return (int)std::max(1LL, std::min(need, (long long)c.num_sms * 32));
}

// CSR from device row counts + a fill callback on the allocated arrays.
template <class Fill>
static std::unique_ptr<Matrix> csr_from_counts(Ctx& c, int nrows, int ncols, DevBuf<int>& cnt,
                                               Fill fill) {
  DevBuf<int> rp(nrows + 1);
  size_t tmp = 0;
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, rp.p, nrows + 1, c.stream));
  DevBuf<unsigned char> ws(std::max<size_t>(tmp, 1));
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, tmp, cnt.p, rp.p, nrows + 1, c.stream));
  int nnz = 0;
  SAG_CUDA(cudaMemcpyAsync(&nnz, rp.p + nrows, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  DevBuf<int> ci(std::max(nnz, 1));
  DevBuf<double> v(std::max(nnz, 1));
  fill(rp.p, ci.p, v.p);
  return matrix_upload(c, nrows, ncols, nnz, rp.p, ci.p, v.p);
}

std::unique_ptr<Matrix> spgemm_dev(Ctx& c, const Matrix& a, const Matrix& b) {
  SAG_REQUIRE(a.ncols == b.nrows, SAG_DIMENSION_MISMATCH, "spgemm: inner dimensions differ");
  static bool configured = false;
  if (!configured) {
    SAG_CUDA(cudaFuncSetAttribute(spgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSetupSmem));
    configured = true;
  }
  const int capw = table_cap(c, a.nrows, a.rp.p, a.ci.p, b.rp.p, 0);
  const int warps = setup_warps(capw * kSpgSlot), smem = warps * capw * kSpgSlot;
  DevBuf<int> cnt(a.nrows + 1), ovf(1);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (a.nrows + 1), c.stream));
  SAG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c.stream));
  const int grid = setup_grid(c, a.nrows, warps);
  spgemm_kernel<<<grid, warps * 32, smem, c.stream>>>(a.nrows, a.rp.p, a.ci.p, a.v.p, b.rp.p,
                                                      b.ci.p, b.v.p, capw, 0, cnt.p, nullptr,
                                                      nullptr, nullptr, ovf.p);
  SAG_LAUNCHED(c);
  int hov = 0;
  SAG_CUDA(cudaMemcpyAsync(&hov, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  SAG_REQUIRE(!hov, SAG_ERROR, "spgemm: an output row has more than 4096 distinct columns");
  return csr_from_counts(c, a.nrows, b.ncols, cnt, [&](int* rp, int* ci, double* v) {
    spgemm_kernel<<<grid, warps * 32, smem, c.stream>>>(a.nrows, a.rp.p, a.ci.p, a.v.p, b.rp.p,
                                                        b.ci.p, b.v.p, capw, 1, nullptr, rp, ci,
                                                        v, ovf.p);
    SAG_LAUNCHED(c);
  });
}

// ---- smooth_prolongator (amg.cpp:226-236) ------------------------------
// at = A T; at_rq *= omega * d_inv[r]; P = sparse_add(T, at, 1, -1): per row
// the merged column lists, t + (-(at)) where both exist (a sum of two, order
// free), exact zeros dropped (from_triplets, sparse.cpp:44-62).
__global__ void smooth_scale_kernel(int nrows, const int* __restrict__ arp,
                                    const int* __restrict__ aci, const double* __restrict__ av,
                                    const int* __restrict__ rp, double* __restrict__ v, double omega,
                                    int* bad) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    double d = 0.0;  // diagonal_of (sparse.cpp:202-206): A.at(r, r)
    for (int q = arp[r]; q < arp[r + 1]; ++q)
      if (aci[q] == r) d = av[q];
    if (d == 0.0) {
      atomicOr(bad, 1);
      continue;
    }
    const double dinv = 1.0 / d;                    // inv_diagonal (sparse.cpp:208-215)
    const double s = __dmul_rn(omega, dinv);       // omega * d_inv[r]
    for (int q = rp[r]; q < rp[r + 1]; ++q) v[q] = __dmul_rn(v[q], s);
  }
}

__global__ void add_rows_kernel(int nrows, const int* __restrict__ trp, const int* __restrict__ tci,
                                const double* __restrict__ tv, const int* __restrict__ arp,
                                const int* __restrict__ aci, const double* __restrict__ av,
                                int pass, int* __restrict__ cnt, const int* __restrict__ crp,
                                int* __restrict__ cci, double* __restrict__ cv) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    int p = trp[r], q = arp[r], n = 0;
    const int pe = trp[r + 1], qe = arp[r + 1];
    int o = pass ? crp[r] : 0;
    while (p < pe || q < qe) {
      int col;
      double s = 0.0;  // from_triplets: sum = 0.0; sum += ...
      if (q >= qe || (p < pe && tci[p] < aci[q])) {
        col = tci[p];
        s = __dadd_rn(s, tv[p++]);
      } else if (p >= pe || aci[q] < tci[p]) {
        col = aci[q];
        s = __dadd_rn(s, -av[q++]);
      } else {
        col = tci[p];
        s = __dadd_rn(__dadd_rn(s, tv[p++]), -av[q++]);
      }
      if (s != 0.0) {
        if (pass) {
          cci[o] = col;
          cv[o] = s;
          ++o;
        }
        ++n;
      }
    }
    if (!pass) cnt[r] = n;
  }
}

std::unique_ptr<Matrix> smooth_prolongator_dev(Ctx& c, const Matrix& a, const Matrix& t,
                                               double omega) {
  SAG_REQUIRE(a.nrows == a.ncols && a.nrows == t.nrows, SAG_DIMENSION_MISMATCH,
              "smooth_prolongator: shapes differ");
  auto at = spgemm_dev(c, a, t);
  DevBuf<int> bad(1);
  SAG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  const int g = std::max(1, std::min((a.nrows + 255) / 256, c.num_sms * 16));
  smooth_scale_kernel<<<g, 256, 0, c.stream>>>(a.nrows, a.rp.p, a.ci.p, a.v.p, at->rp.p, at->v.p,
                                               omega, bad.p);
  SAG_LAUNCHED(c);
  int hb = 0;
  SAG_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  SAG_REQUIRE(!hb, SAG_ZERO_DIAGONAL, "inv_diagonal: zero diagonal");
  DevBuf<int> cnt(t.nrows + 1);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (t.nrows + 1), c.stream));
  add_rows_kernel<<<g, 256, 0, c.stream>>>(t.nrows, t.rp.p, t.ci.p, t.v.p, at->rp.p, at->ci.p,
                                           at->v.p, 0, cnt.p, nullptr, nullptr, nullptr);
  SAG_LAUNCHED(c);
  return csr_from_counts(c, t.nrows, t.ncols, cnt, [&](int* rp, int* ci, double* v) {
    add_rows_kernel<<<g, 256, 0, c.stream>>>(t.nrows, t.rp.p, t.ci.p, t.v.p, at->rp.p, at->ci.p,
                                             at->v.p, 1, nullptr, rp, ci, v);
    SAG_LAUNCHED(c);
  });
}

// ---- evolution_soc (amg.cpp:45-110) ---------------------------------------
// Column j: z = (I - omega D^-1 A)^k e_j over the sparse "touched" set, in the
// reference's order: each step walks the touched list in order and the rows of
// A^T, accumulating az_i in that order (the lanes of one A^T row add distinct
// i, new entries appended in lane = row order through a ballot prefix), then
// updates z_i = z_i - (omega d_inv_i) az_i over az_touched in order. Edges
// (i, j, s) and (j, i, s) for s = |z_i| / |z_j| >= theta max_m s_m; the
// union is sorted and duplicates keep the stronger weight
// (graph_from_adjacency, amg.cpp:13-42).
constexpr int kSocSlot = 4 + 8 + 8 + 4 + 4 + 1;  // key, z, az, touched, az_touched, flags
static int soc_warp_bytes(int capw) { return (capw * kSocSlot + 15) / 16 * 16; }

struct SocTable {
  int* keys;
  double* z;
  double* az;
  int* touched;
  int* azt;
  unsigned char* fl;  // bit 0 in touched, bit 1 in az (this step)
  unsigned mask;
  __device__ int find_or_insert(int key, bool& overflow) {
    unsigned h = ((unsigned)key * 2654435761u) & mask;
    for (unsigned p = 0; p <= mask; ++p) {
      const int k = atomicCAS(keys + h, -1, key);
      if (k == -1) {
        z[h] = 0.0;
        az[h] = 0.0;
        fl[h] = 0;
        return (int)h;
      }
      if (k == key) return (int)h;
      h = (h + 1) & mask;
    }
    overflow = true;
    return 0;
  }
  __device__ int find(int key) const {
    unsigned h = ((unsigned)key * 2654435761u) & mask;
    while (keys[h] != key) h = (h + 1) & mask;
    return (int)h;
  }
};

__global__ void __launch_bounds__(512) evolution_soc_kernel(
    int n, const int* __restrict__ trp, const int* __restrict__ tci, const double* __restrict__ tv,
    const double* __restrict__ dinv, double omega, double theta, int ksteps, int capw, int pass,
    int* __restrict__ cnt, const long long* __restrict__ eoff, unsigned long long* __restrict__ ekey,
    double* __restrict__ eval, int* overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned char* base = smem + (size_t)wib * ((capw * kSocSlot + 15) / 16 * 16);
  SocTable T;
  T.z = reinterpret_cast<double*>(base);
  T.az = T.z + capw;
  T.keys = reinterpret_cast<int*>(T.az + capw);
  T.touched = T.keys + capw;
  T.azt = T.touched + capw;
  T.fl = reinterpret_cast<unsigned char*>(T.azt + capw);
  __shared__ int wcount[16];
  const int gw = blockIdx.x * warps + wib, nw = gridDim.x * warps;
  for (int j = gw; j < n; j += nw) {
    // table size: >= 2x an upper bound of the touched set (k = 2), <= capw
    int est = 0;
    if (ksteps == 2) {
      for (int q = trp[j] + lane; q < trp[j + 1]; q += 32) {
        const int i = tci[q];
        est += trp[i + 1] - trp[i];
      }
      for (int o = 16; o > 0; o >>= 1) est += __shfl_xor_sync(0xffffffffu, est, o);
      est += 1 + trp[j + 1] - trp[j];
    } else {
      est = capw;
    }
    int cap = 64;
    while (cap < 2 * est && cap < capw) cap <<= 1;
    T.mask = cap - 1;
    for (int s = lane; s < cap; s += 32) T.keys[s] = -1;
    __syncwarp();
    bool ovf = false;
    if (lane == 0) {
      const int sj = T.find_or_insert(j, ovf);
      T.z[sj] = 1.0;
      T.fl[sj] = 1;
      T.touched[0] = j;
    }
    __syncwarp();
    int nt = 1;
    for (int step = 0; step < ksteps; ++step) {
      int naz = 0;
      const int nt0 = nt;
      for (int t = 0; t < nt0; ++t) {
        const int idx = T.touched[t];
        const double v = T.z[T.find(idx)];
        if (v == 0.0) continue;
        const int b = trp[idx], e = trp[idx + 1];
        for (int q0 = b; q0 < e; q0 += 32) {
          const int q = q0 + lane;
          const bool act = q < e;
          int slot = 0;
          bool isnew = false;
          if (act) {
            slot = T.find_or_insert(tci[q], ovf);
            isnew = !(T.fl[slot] & 2);
          }
          const unsigned m = __ballot_sync(0xffffffffu, act && isnew);
          if (act && isnew) {
            const int pos = naz + __popc(m & lt);
            if (pos < capw) T.azt[pos] = tci[q];
            T.fl[slot] |= 2;
            T.az[slot] = 0.0;
          }
          naz += __popc(m);
          if (act) T.az[slot] = __dadd_rn(T.az[slot], __dmul_rn(tv[q], v));
          __syncwarp();
        }
      }
      if (naz > capw) ovf = true;
      for (int u0 = 0; u0 < naz && u0 < capw; u0 += 32) {
        const int u = u0 + lane;
        const bool act = u < naz;
        int slot = 0, i = 0;
        bool newt = false;
        if (act) {
          i = T.azt[u];
          slot = T.find(i);
          newt = !(T.fl[slot] & 1);
        }
        const unsigned m = __ballot_sync(0xffffffffu, act && newt);
        if (act && newt) {
          const int pos = nt + __popc(m & lt);
          if (pos < capw) T.touched[pos] = i;
          T.fl[slot] |= 1;
        }
        nt += __popc(m);
        if (act) {
          T.z[slot] = __dsub_rn(T.z[slot], __dmul_rn(__dmul_rn(omega, dinv[i]), T.az[slot]));
          T.fl[slot] &= ~2;
        }
        __syncwarp();
      }
      if (nt > capw) {
        ovf = true;
        nt = capw;
      }
    }
    // strength over the touched set (amg.cpp:86-101)
    const double zj = fabs(T.z[T.find(j)]);
    int emitted = 0;
    if (zj > 0.0) {
      double smax = 0.0;
      for (int u = lane; u < nt; u += 32) {
        const int i = T.touched[u];
        if (i != j) smax = fmax(smax, fabs(T.z[T.find(i)]) / zj);
      }
      for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
      if (smax > 0.0) {
        const double thr = theta * smax;
        if (lane == 0) wcount[wib] = 0;
        __syncwarp();
        for (int u = lane; u < nt; u += 32) {
          const int i = T.touched[u];
          if (i == j) continue;
          const double sv = fabs(T.z[T.find(i)]) / zj;
          if (sv > 0.0 && sv >= thr) {
            if (pass == 0) {
              ++emitted;
            } else {
              const long long o = eoff[j] + 2LL * atomicAdd(wcount + wib, 1);
              ekey[o] = ((unsigned long long)(unsigned)i << 32) | (unsigned)j;
              eval[o] = sv;
              ekey[o + 1] = ((unsigned long long)(unsigned)j << 32) | (unsigned)i;
              eval[o + 1] = sv;
            }
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(overflow, 1);
    if (pass == 0) {
      for (int o = 16; o > 0; o >>= 1) emitted += __shfl_xor_sync(0xffffffffu, emitted, o);
      if (lane == 0) cnt[j] = 2 * emitted;
    }
    __syncwarp();
  }
}

// sorted (row, col) keys: unique flags, then per unique key the max weight
__global__ void uniq_flag_kernel(long long ne, const unsigned long long* __restrict__ key,
                                 int* __restrict__ flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x)
    flag[e] = (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
}
__global__ void uniq_write_kernel(long long ne, const unsigned long long* __restrict__ key,
                                  const double* __restrict__ val, const int* __restrict__ pos,
                                  int* __restrict__ rowcnt, int* __restrict__ col,
                                  double* __restrict__ w) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x) {
    if (!(e == 0 || key[e] != key[e - 1])) continue;
    double m = val[e];
    for (long long f = e + 1; f < ne && key[f] == key[e]; ++f) m = fmax(m, val[f]);
    const int p = pos[e];
    col[p] = (int)(key[e] & 0xffffffffu);
    w[p] = m;
    atomicAdd(rowcnt + (int)(key[e] >> 32), 1);
  }
}

std::unique_ptr<Matrix> evolution_soc_dev(Ctx& c, const Matrix& a, double omega, double theta,
                                          int ksteps) {
  SAG_REQUIRE(a.nrows == a.ncols, SAG_DIMENSION_MISMATCH, "evolution_soc: A must be square");
  const int n = a.nrows;
  static bool configured = false;
  if (!configured) {
    SAG_CUDA(cudaFuncSetAttribute(evolution_soc_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSetupSmem));
    configured = true;
  }
  auto at = transpose_dev(c, a);
  // d_inv (inv_diagonal, sparse.cpp:208-215): 1 / a_ii
  DevBuf<double> dinv(std::max(n, 1));
  DevBuf<int> bad(1), ovf(1);
  SAG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  SAG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c.stream));
  launch_inv_diag(c, a, dinv.p, bad.p);
  const int capw = ksteps == 2 ? table_cap(c, n, at->rp.p, at->ci.p, at->rp.p, 1) : kSetupMaxCap;
  const int warps = setup_warps(soc_warp_bytes(capw)), smem = warps * soc_warp_bytes(capw);
  DevBuf<int> cnt(n + 1);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (n + 1), c.stream));
  const int grid = setup_grid(c, n, warps);
  evolution_soc_kernel<<<grid, warps * 32, smem, c.stream>>>(
      n, at->rp.p, at->ci.p, at->v.p, dinv.p, omega, theta, ksteps, capw, 0, cnt.p, nullptr,
      nullptr, nullptr, ovf.p);
  SAG_LAUNCHED(c);
  int hb = 0, ho = 0;
  SAG_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaMemcpyAsync(&ho, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  SAG_REQUIRE(!hb, SAG_ZERO_DIAGONAL, "inv_diagonal: zero diagonal");
  SAG_REQUIRE(!ho, SAG_ERROR, "evolution_soc: a column's touched set exceeds the device table");
  // edge offsets (int64), then the edges
  DevBuf<long long> eoff(n + 1);
  {
    DevBuf<long long> cl(n + 1);
    std::vector<int> hc(n + 1);
    SAG_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<long long> ho2(n + 1, 0);
    for (int j = 0; j < n; ++j) ho2[j + 1] = ho2[j] + hc[j];
    SAG_CUDA(cudaMemcpyAsync(eoff.p, ho2.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, c.stream));
    const long long ne = ho2[n];
    SAG_REQUIRE(ne < (1LL << 31), SAG_DIMENSION_MISMATCH, "evolution_soc: too many edges");
    DevBuf<unsigned long long> key(std::max(ne, 1LL)), key2(std::max(ne, 1LL));
    DevBuf<double> val(std::max(ne, 1LL)), val2(std::max(ne, 1LL));
    evolution_soc_kernel<<<grid, warps * 32, smem, c.stream>>>(
        n, at->rp.p, at->ci.p, at->v.p, dinv.p, omega, theta, ksteps, capw, 1, nullptr, eoff.p,
        key.p, val.p, ovf.p);
    SAG_LAUNCHED(c);
    size_t t1 = 0;
    SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, key.p, key2.p, val.p, val2.p, (int)ne, 0,
                                             64, c.stream));
    DevBuf<int> flag(std::max(ne, 1LL) + 1), pos(std::max(ne, 1LL) + 1), rowcnt(n + 1);
    size_t t2 = 0;
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, flag.p, pos.p, (int)ne + 1, c.stream));
    DevBuf<unsigned char> ws(std::max<size_t>(std::max(t1, t2), 1));
    if (ne > 0)
      SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, t1, key.p, key2.p, val.p, val2.p, (int)ne, 0,
                                               64, c.stream));
    SAG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int) * (ne + 1), c.stream));
    const int g = std::max(1, (int)std::min<long long>((ne + 255) / 256, c.num_sms * 16LL));
    uniq_flag_kernel<<<g, 256, 0, c.stream>>>(ne, key2.p, flag.p);
    SAG_LAUNCHED(c);
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, t2, flag.p, pos.p, (int)ne + 1, c.stream));
    int nu = 0;
    SAG_CUDA(cudaMemcpyAsync(&nu, pos.p + ne, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    DevBuf<int> col(std::max(nu, 1));
    DevBuf<double> w(std::max(nu, 1));
    SAG_CUDA(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * (n + 1), c.stream));
    uniq_write_kernel<<<g, 256, 0, c.stream>>>(ne, key2.p, val2.p, pos.p, rowcnt.p, col.p, w.p);
    SAG_LAUNCHED(c);
    DevBuf<int> rp(n + 1);
    size_t t3 = 0;
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, rowcnt.p, rp.p, n + 1, c.stream));
    DevBuf<unsigned char> ws3(std::max<size_t>(t3, 1));
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws3.p, t3, rowcnt.p, rp.p, n + 1, c.stream));
    return matrix_upload(c, n, n, nu, rp.p, col.p, w.p);
  }
}

// ---- assemble_saddle_matrix (fem.cpp:290-306) ------------------------------
// K = [[A, B^T], [B, 0]]: the reference sums the triplets of A, B and B^T in
// from_triplets; the three blocks never share a position and canonical
// A / B hold no zeros, so every entry is the single stored value (0.0 + v)
// and K's rows are the concatenations A row | (B^T row shifted by n_u) for
// velocity rows and B row for pressure rows.
__global__ void saddle_rows_kernel(int nu, int np, const int* __restrict__ arp,
                                   const int* __restrict__ aci, const double* __restrict__ av,
                                   const int* __restrict__ btrp, const int* __restrict__ btci,
                                   const double* __restrict__ btv, const int* __restrict__ brp,
                                   const int* __restrict__ bci, const double* __restrict__ bv,
                                   int pass, int* __restrict__ cnt, const int* __restrict__ krp,
                                   int* __restrict__ kci, double* __restrict__ kv) {
  const int n = nu + np;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int o = pass ? krp[r] : 0, c = 0;
    auto put = [&](int col, double v) {
      const double sum = 0.0 + v;  // from_triplets: sum = 0.0; sum += value
      if (sum == 0.0) return;
      if (pass) {
        kci[o] = col;
        kv[o] = sum;
        ++o;
      }
      ++c;
    };
    if (r < nu) {
      for (int q = arp[r]; q < arp[r + 1]; ++q) put(aci[q], av[q]);
      for (int q = btrp[r]; q < btrp[r + 1]; ++q) put(nu + btci[q], btv[q]);
    } else {
      for (int q = brp[r - nu]; q < brp[r - nu + 1]; ++q) put(bci[q], bv[q]);
    }
    if (!pass) cnt[r] = c;
  }
}

std::unique_ptr<Matrix> saddle_matrix_dev(Ctx& c, const Matrix& a, const Matrix& b) {
  SAG_REQUIRE(a.nrows == a.ncols && b.ncols == a.nrows, SAG_DIMENSION_MISMATCH,
              "assemble_saddle_matrix: A is n_u x n_u and B is n_p x n_u");
  const int nu = a.nrows, np = b.nrows, n = nu + np;
  auto bt = transpose_dev(c, b);
  DevBuf<int> cnt(n + 1);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (n + 1), c.stream));
  const int g = std::max(1, std::min((n + 255) / 256, c.num_sms * 16));
  saddle_rows_kernel<<<g, 256, 0, c.stream>>>(nu, np, a.rp.p, a.ci.p, a.v.p, bt->rp.p, bt->ci.p,
                                              bt->v.p, b.rp.p, b.ci.p, b.v.p, 0, cnt.p, nullptr,
                                              nullptr, nullptr);
  SAG_LAUNCHED(c);
  return csr_from_counts(c, n, n, cnt, [&](int* rp, int* ci, double* v) {
    saddle_rows_kernel<<<g, 256, 0, c.stream>>>(nu, np, a.rp.p, a.ci.p, a.v.p, bt->rp.p,
                                                bt->ci.p, bt->v.p, b.rp.p, b.ci.p, b.v.p, 1,
                                                nullptr, rp, ci, v);
    SAG_LAUNCHED(c);
  });
}

}  // namespace sag

// =================================================================== C-ABI
using namespace sag;


namespace sag {
// ---- tentative prolongator (amg.cpp:184-205) and power_rho_estimate
// (sparse.cpp:239-261), bitwise ---------------------------------------------
// colnorm_c = sqrt(sum over the aggregate's nodes, in node order, of
// nullvec_i^2): a stable sort of the nodes by aggregate keeps node order.
__global__ void agg_norm_kernel(int n, const int* __restrict__ agg_sorted,
                                const int* __restrict__ node_sorted,
                                const double* __restrict__ nullvec, double* colnorm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = agg_sorted[i];
    if (i > 0 && agg_sorted[i - 1] == a) continue;
    double s = 0.0;
    for (int j = i; j < n && agg_sorted[j] == a; ++j) {
      const double v = nullvec[node_sorted[j]];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
    colnorm[a] = sqrt(s);
  }
}
// T_ic = nullvec_i / colnorm_c, one entry per row (from_triplets drops zeros)
__global__ void tentative_count_kernel(int n, const int* __restrict__ agg,
                                       const double* __restrict__ nullvec,
                                       const double* __restrict__ colnorm, int* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = agg[i];
    cnt[i] = (nullvec[i] / colnorm[c]) != 0.0 ? 1 : 0;
  }
}
__global__ void tentative_fill_kernel(int n, const int* __restrict__ agg,
                                      const double* __restrict__ nullvec,
                                      const double* __restrict__ colnorm,
                                      const int* __restrict__ rp, int* ci, double* v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = agg[i];
    const double t = nullvec[i] / colnorm[c];
    if (t != 0.0) {
      ci[rp[i]] = c;
      v[rp[i]] = t;
    }
  }
}
__global__ void empty_agg_kernel(int nc, const double* colnorm, const int* seen, int* bad) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x)
    if (!seen[c] || colnorm[c] == 0.0) atomicMin(bad, c);
}
__global__ void iota_kernel(int n, int* a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}
__global__ void mark_agg_kernel(int n, const int* agg, int* seen) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    seen[agg[i]] = 1;
}

// y = D^-1 (M x), each row summed in order with round-to-nearest operations
// (spmv, sparse.cpp:78-91, then y_i *= d_inv_i, :252)
__global__ void spmv_rn_scale_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                     const double* __restrict__ v, const double* __restrict__ x,
                                     const double* __restrict__ dinv, double* y) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
    y[r] = __dmul_rn(s, dinv[r]);
  }
}
__global__ void scale_div_kernel(int n, const double* y, double ny, double* x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = __ddiv_rn(y[i], ny);
}

}  // namespace sag

namespace {
sag_matrix* wrap(std::unique_ptr<Matrix> m) {
  auto* h = new sag_matrix;
  h->m = std::move(*m);
  return h;
}
}  // namespace

extern "C" {

int sag_spgemm(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* b, sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(b);
    SAG_NOTNULL(out);
    *out = wrap(spgemm_dev(ctx->c, a->m, b->m));
  });
}

int sag_transpose(sag_ctx* ctx, const sag_matrix* a, sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(out);
    *out = wrap(transpose_dev(ctx->c, a->m));
  });
}

int sag_galerkin(sag_ctx* ctx, const sag_matrix* p, const sag_matrix* k, sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(p);
    SAG_NOTNULL(k);
    SAG_NOTNULL(out);
    SAG_REQUIRE(k->m.nrows == k->m.ncols, SAG_DIMENSION_MISMATCH,
                "galerkin_triple: K must be square");
    SAG_REQUIRE(k->m.nrows == p->m.nrows, SAG_DIMENSION_MISMATCH,
                "galerkin_triple: K and P row counts differ");
    auto kp = spgemm_dev(ctx->c, k->m, p->m);
    auto pt = transpose_dev(ctx->c, p->m);
    *out = wrap(spgemm_dev(ctx->c, *pt, *kp));
  });
}

int sag_smooth_prolongator(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* t, double omega,
                           sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(t);
    SAG_NOTNULL(out);
    *out = wrap(smooth_prolongator_dev(ctx->c, a->m, t->m, omega));
  });
}

int sag_evolution_soc(sag_ctx* ctx, const sag_matrix* a, double omega, double theta, int k,
                      sag_matrix** graph) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(graph);
    SAG_REQUIRE(k >= 0, SAG_CONFIG_ERROR, "evolution_soc: k must be non-negative");
    *graph = wrap(evolution_soc_dev(ctx->c, a->m, omega, theta, k));
  });
}

int sag_saddle_matrix(sag_ctx* ctx, const sag_matrix* a, const sag_matrix* b, sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a);
    SAG_NOTNULL(b);
    SAG_NOTNULL(out);
    *out = wrap(saddle_matrix_dev(ctx->c, a->m, b->m));
  });
}

int sag_tentative_prolongator(sag_ctx* ctx, int n, int num_aggregates, const int* node_to_agg,
                              const double* nullvec, sag_matrix** t, double* coarse_nullvec) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(t);
    SAG_REQUIRE(n >= 0 && num_aggregates >= 0, SAG_DIMENSION_MISMATCH,
                "tentative_prolongator: negative size");
    Ctx& c = ctx->c;
    const int nc = num_aggregates;
    DevBuf<int> agg(std::max(n, 1)), agg2(std::max(n, 1)), ids(std::max(n, 1)),
        ids2(std::max(n, 1)), cnt(n + 1), seen(std::max(nc, 1)), bad(1);
    DevBuf<double> nv(std::max(n, 1)), cn(std::max(nc, 1));
    if (n) {
      SAG_NOTNULL(node_to_agg);
      SAG_NOTNULL(nullvec);
      SAG_CUDA(cudaMemcpyAsync(agg.p, node_to_agg, 4 * (size_t)n, cudaMemcpyDefault, c.stream));
      SAG_CUDA(cudaMemcpyAsync(nv.p, nullvec, 8 * (size_t)n, cudaMemcpyDefault, c.stream));
    }
    SAG_CUDA(cudaMemsetAsync(cn.p, 0, 8 * (size_t)std::max(nc, 1), c.stream));
    SAG_CUDA(cudaMemsetAsync(seen.p, 0, 4 * (size_t)std::max(nc, 1), c.stream));
    const int big = 0x7fffffff;
    SAG_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
    const int g = std::max(1, std::min((std::max(n, nc) + 255) / 256, c.num_sms * 16));
    if (n) {
      iota_kernel<<<g, 256, 0, c.stream>>>(n, ids.p);
      SAG_LAUNCHED(c);
      size_t tmp = 0;
      SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, agg.p, agg2.p, ids.p, ids2.p, n, 0,
                                               32, c.stream));
      DevBuf<unsigned char> ws(std::max<size_t>(tmp, 1));
      SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, tmp, agg.p, agg2.p, ids.p, ids2.p, n, 0, 32,
                                               c.stream));
      agg_norm_kernel<<<g, 256, 0, c.stream>>>(n, agg2.p, ids2.p, nv.p, cn.p);
      SAG_LAUNCHED(c);
      mark_agg_kernel<<<g, 256, 0, c.stream>>>(n, agg.p, seen.p);
      SAG_LAUNCHED(c);
    }
    if (nc) {
      empty_agg_kernel<<<g, 256, 0, c.stream>>>(nc, cn.p, seen.p, bad.p);
      SAG_LAUNCHED(c);
    }
    int hb = big;
    SAG_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    SAG_REQUIRE(hb == big, SAG_ERROR,
                "tentative_prolongator: zero near-kernel over aggregate " + std::to_string(hb));
    SAG_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (size_t)(n + 1), c.stream));
    if (n) {
      tentative_count_kernel<<<g, 256, 0, c.stream>>>(n, agg.p, nv.p, cn.p, cnt.p);
      SAG_LAUNCHED(c);
    }
    *t = wrap(csr_from_counts(c, n, nc, cnt, [&](int* rp, int* ci, double* v) {
      if (n) {
        tentative_fill_kernel<<<g, 256, 0, c.stream>>>(n, agg.p, nv.p, cn.p, rp, ci, v);
        SAG_LAUNCHED(c);
      }
    }));
    if (coarse_nullvec && nc)
      SAG_CUDA(cudaMemcpyAsync(coarse_nullvec, cn.p, 8 * (size_t)nc, cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_power_rho(sag_ctx* ctx, const sag_matrix* m, const double* d_inv, const double* x0,
                  int iters, double* rho) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(m);
    SAG_NOTNULL(rho);
    Ctx& c = ctx->c;
    const Matrix& M = m->m;
    SAG_REQUIRE(M.nrows == M.ncols, SAG_DIMENSION_MISMATCH,
                "power_rho_estimate: matrix must be square");
    const int n = M.nrows;
    *rho = 0.0;
    if (n == 0) return;
    SAG_NOTNULL(d_inv);
    SAG_NOTNULL(x0);
    DevBuf<double> x(n), y(n), di(n);
    std::vector<double> hy(n);
    SAG_CUDA(cudaMemcpyAsync(x.p, x0, 8 * (size_t)n, cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaMemcpyAsync(di.p, d_inv, 8 * (size_t)n, cudaMemcpyDefault, c.stream));
    const int g = std::max(1, std::min((n + 255) / 256, c.num_sms * 16));
    for (int it = 0; it < iters; ++it) {
      spmv_rn_scale_kernel<<<g, 256, 0, c.stream>>>(n, M.rp.p, M.ci.p, M.v.p, x.p, di.p, y.p);
      SAG_LAUNCHED(c);
      SAG_CUDA(cudaMemcpyAsync(hy.data(), y.p, 8 * (size_t)n, cudaMemcpyDeviceToHost, c.stream));
      SAG_CUDA(cudaStreamSynchronize(c.stream));
      // norm2 (sparse.cpp:217-221): a sequential sum, on the host
      double s = 0.0;
      for (double v : hy) s += v * v;
      const double ny = std::sqrt(s);
      if (ny == 0.0) {
        *rho = 0.0;
        return;
      }
      *rho = ny;
      scale_div_kernel<<<g, 256, 0, c.stream>>>(n, y.p, ny, x.p);
      SAG_LAUNCHED(c);
    }
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_matrix_export(sag_ctx* ctx, const sag_matrix* m, int* row_offsets, int* col_indices,
                      double* values) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(m);
    auto& c = ctx->c;
    const auto& mm = m->m;
    if (row_offsets)
      SAG_CUDA(cudaMemcpyAsync(row_offsets, mm.rp.p, sizeof(int) * (mm.nrows + 1),
                               cudaMemcpyDefault, c.stream));
    if (col_indices && mm.nnz)
      SAG_CUDA(cudaMemcpyAsync(col_indices, mm.ci.p, sizeof(int) * mm.nnz, cudaMemcpyDefault,
                               c.stream));
    if (values && mm.nnz)
      SAG_CUDA(cudaMemcpyAsync(values, mm.v.p, sizeof(double) * mm.nnz, cudaMemcpyDefault,
                               c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
