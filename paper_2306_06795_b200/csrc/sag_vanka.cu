// libsag Vanka module (vanka.hpp:11-55 / vanka.cpp:11-209 of the reference):
//   build_patches    -> patch_count_kernel / patch_fill_kernel
//   factor_patches   -> factor_kernel: warp-per-patch block LU in shared memory
//   apply_vanka      -> vanka_patch_kernel (cp.async.bulk-staged factor blobs,
//                       warp-per-patch dense solves) + vanka_gather_kernel
//                       (atomic-free owner-computes scatter-add)
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.cuh"
#include "tma.cuh"

namespace sag {

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// ======================================================== build_patches ==

// vanka.cpp:20-38: patch i seeds pressure rows n_u + i*group + g; its
// velocity set is the sorted union of the seed rows' columns c < n_u.
__device__ __forceinline__ int merge_unique(const int* rp, const int* ci, int row0, int group,
                                            int n_u, int* dst) {
  int pos[3], end[3];
  for (int g = 0; g < group; ++g) {
    pos[g] = rp[row0 + g];
    end[g] = rp[row0 + g + 1];
  }
  int cnt = 0, last = -1;
  while (true) {
    int best = 0x7fffffff, bg = -1;
    for (int g = 0; g < group; ++g) {
      if (pos[g] < end[g]) {
        const int c = ci[pos[g]];
        if (c < n_u && c < best) {
          best = c;
          bg = g;
        }
      }
    }
    if (bg < 0) break;
    ++pos[bg];
    if (best != last) {
      if (dst) dst[cnt] = best;
      ++cnt;
      last = best;
    }
  }
  return cnt;
}

__global__ void patch_count_kernel(int npatch, int group, int n_u, int n_x, const int* rp,
                                   const int* ci, int* cnt_v, int* cnt_x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npatch; i += gridDim.x * blockDim.x) {
    const int row0 = n_u + i * group;
    int nv, nx = 0;
    if (group == 1) {
      nv = 0;
      for (int q = rp[row0]; q < rp[row0 + 1]; ++q) {
        const int c = ci[q];
        nv += c < n_u;
        nx += c < n_x;
      }
    } else {
      nv = merge_unique(rp, ci, row0, group, n_u, nullptr);
    }
    cnt_v[i] = nv;
    cnt_x[i] = nx;  // group 3: recomputed in fill
  }
}

__global__ void patch_fill_kernel(int npatch, int group, int n_u, int n_x, const int* rp,
                                  const int* ci, const int* vptr, int* vidx, int* pptr,
                                  int* pidx, int* nx_out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npatch; i += gridDim.x * blockDim.x) {
    const int row0 = n_u + i * group;
    int* dst = vidx + vptr[i];
    int nv;
    if (group == 1) {
      nv = 0;
      for (int q = rp[row0]; q < rp[row0 + 1]; ++q)
        if (ci[q] < n_u) dst[nv++] = ci[q];
    } else {
      nv = merge_unique(rp, ci, row0, group, n_u, dst);
    }
    int nx = 0;
    while (nx < nv && dst[nx] < n_x) ++nx;  // lower_bound(n_x), vanka.cpp:36-38
    nx_out[i] = nx;
    for (int g = 0; g < group; ++g) pidx[i * group + g] = row0 + g;
    pptr[i] = i * group;
    if (i == npatch - 1) pptr[npatch] = npatch * group;
  }
}

static void patch_maxima(Patches& p, const std::vector<int>& vptr, const std::vector<int>& pptr,
                         const std::vector<int>& nx) {
  p.max_nv = p.max_np = p.max_dim = 0;
  for (int i = 0; i < p.npatch; ++i) {
    const int nv = vptr[i + 1] - vptr[i], np = pptr[i + 1] - pptr[i];
    p.max_nv = std::max(p.max_nv, nv);
    p.max_np = std::max(p.max_np, np);
    p.max_dim = std::max(p.max_dim, std::max(nx[i], nv - nx[i]));
  }
  p.tot_v = p.npatch ? vptr[p.npatch] : 0;
  p.tot_p = p.npatch ? pptr[p.npatch] : 0;
}

std::unique_ptr<Patches> build_patches_dev(Ctx& c, const Matrix& k, int n_x, int n_y, int n_p,
                                           bool sv_triples) {
  const int n_u = n_x + n_y;
  SAG_REQUIRE(n_x >= 0 && n_y >= 0 && n_p >= 0 && k.nrows == n_u + n_p && k.ncols == k.nrows,
              SAG_DIMENSION_MISMATCH, "build_patches: block sizes do not match K");
  SAG_REQUIRE(!sv_triples || n_p % 3 == 0, SAG_DIMENSION_MISMATCH,
              "build_patches: triple seeding needs a multiple-of-3 pressure count");
  const int group = sv_triples ? 3 : 1;
  auto p = std::make_unique<Patches>();
  const int np = n_p / group;
  p->npatch = np;
  p->pptr.alloc(np + 1);
  p->pidx.alloc(n_p);
  p->vptr.alloc(np + 1);
  p->nx.alloc(np);
  if (np == 0) {
    SAG_CUDA(cudaMemsetAsync(p->pptr.p, 0, sizeof(int), c.stream));
    SAG_CUDA(cudaMemsetAsync(p->vptr.p, 0, sizeof(int), c.stream));
    p->vidx.alloc(1);
    return p;
  }
  DevBuf<int> cv(np), cx(np);
  const int grid = std::max(1, std::min((np + 255) / 256, c.num_sms * 16));
  patch_count_kernel<<<grid, 256, 0, c.stream>>>(np, group, n_u, n_x, k.rp.p, k.ci.p, cv.p, cx.p);
  SAG_LAUNCHED(c);
  std::vector<int> hv(np);
  SAG_CUDA(cudaMemcpyAsync(hv.data(), cv.p, sizeof(int) * np, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<int> vptr(np + 1, 0);
  long long acc = 0;
  for (int i = 0; i < np; ++i) {
    if (hv[i] == 0)
      throw Error(SAG_SINGULAR_PATCH, "build_patches: pressure row " + std::to_string(i * group) +
                                          " couples to no velocity DoFs");
    acc += hv[i];
    SAG_REQUIRE(acc < (1LL << 31), SAG_DIMENSION_MISMATCH, "build_patches: too many entries");
    vptr[i + 1] = (int)acc;
  }
  SAG_CUDA(cudaMemcpyAsync(p->vptr.p, vptr.data(), sizeof(int) * (np + 1), cudaMemcpyHostToDevice,
                           c.stream));
  p->vidx.alloc(acc);
  patch_fill_kernel<<<grid, 256, 0, c.stream>>>(np, group, n_u, n_x, k.rp.p, k.ci.p, p->vptr.p,
                                                p->vidx.p, p->pptr.p, p->pidx.p, p->nx.p);
  SAG_LAUNCHED(c);
  std::vector<int> hnx(np), pptr(np + 1);
  for (int i = 0; i <= np; ++i) pptr[i] = i * group;
  SAG_CUDA(cudaMemcpyAsync(hnx.data(), p->nx.p, sizeof(int) * np, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  patch_maxima(*p, vptr, pptr, hnx);
  return p;
}

std::unique_ptr<Patches> patches_from_lists(Ctx& c, int npatch, const int* pptr_in,
                                            const int* pidx_in, const int* vptr_in,
                                            const int* vidx_in, const int* nx_in) {
  SAG_REQUIRE(npatch >= 0, SAG_DIMENSION_MISMATCH, "sag_patches_create: negative count");
  std::vector<int> pptr(npatch + 1), vptr(npatch + 1), nx(std::max(npatch, 1));
  SAG_CUDA(cudaMemcpy(pptr.data(), pptr_in, sizeof(int) * (npatch + 1), cudaMemcpyDefault));
  SAG_CUDA(cudaMemcpy(vptr.data(), vptr_in, sizeof(int) * (npatch + 1), cudaMemcpyDefault));
  if (npatch) SAG_CUDA(cudaMemcpy(nx.data(), nx_in, sizeof(int) * npatch, cudaMemcpyDefault));
  const int tp = pptr[npatch], tv = vptr[npatch];
  std::vector<int> pidx(std::max(tp, 1)), vidx(std::max(tv, 1));
  if (tp) SAG_CUDA(cudaMemcpy(pidx.data(), pidx_in, sizeof(int) * tp, cudaMemcpyDefault));
  if (tv) SAG_CUDA(cudaMemcpy(vidx.data(), vidx_in, sizeof(int) * tv, cudaMemcpyDefault));
  for (int i = 0; i < npatch; ++i) {
    const int nv = vptr[i + 1] - vptr[i];
    SAG_REQUIRE(nv > 0 && pptr[i + 1] > pptr[i] && nx[i] >= 0 && nx[i] <= nv,
                SAG_DIMENSION_MISMATCH, "sag_patches_create: malformed patch " + std::to_string(i));
    for (int q = vptr[i] + 1; q < vptr[i + 1]; ++q)
      SAG_REQUIRE(vidx[q] > vidx[q - 1], SAG_ERROR,
                  "sag_patches_create: velocity lists must be sorted and unique");
  }
  auto p = std::make_unique<Patches>();
  p->npatch = npatch;
  p->pptr.alloc(npatch + 1);
  p->vptr.alloc(npatch + 1);
  p->nx.alloc(std::max(npatch, 1));
  p->pidx.alloc(std::max(tp, 1));
  p->vidx.alloc(std::max(tv, 1));
  SAG_CUDA(cudaMemcpy(p->pptr.p, pptr.data(), sizeof(int) * (npatch + 1), cudaMemcpyHostToDevice));
  SAG_CUDA(cudaMemcpy(p->vptr.p, vptr.data(), sizeof(int) * (npatch + 1), cudaMemcpyHostToDevice));
  SAG_CUDA(cudaMemcpy(p->nx.p, nx.data(), sizeof(int) * nx.size(), cudaMemcpyHostToDevice));
  SAG_CUDA(cudaMemcpy(p->pidx.p, pidx.data(), sizeof(int) * pidx.size(), cudaMemcpyHostToDevice));
  SAG_CUDA(cudaMemcpy(p->vidx.p, vidx.data(), sizeof(int) * vidx.size(), cudaMemcpyHostToDevice));
  patch_maxima(*p, vptr, pptr, nx);
  return p;
}

// ======================================================= factor_patches ==
// Arithmetic restates vanka.cpp:64-149 and sparse.cpp:310-361 with explicit
// round-to-nearest operations (no FMA contraction), so u_hat, b_hat and s_inv
// are bitwise those of the reference. The apply representation additionally
// stores A_x^-1 and A_y^-1, whose columns are dense_lu_solve(lu, e_c).

__device__ __forceinline__ int bsearch_idx(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < n && a[lo] == key) ? lo : -1;
}

// sparse.cpp:310-341 by one warp on a row-major n x n matrix in shared memory.
__device__ bool warp_lu(double* A, int n, int ld, int* piv, int lane) {
  for (int i = lane; i < n; i += 32) piv[i] = i;
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = k + 1 + lane; i < n; i += 32) {
      const double v = fabs(A[i * ld + k]);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    const double akk = fabs(A[k * ld + k]);
    const int p = (bv > akk) ? bi : k;
    const double best = (bv > akk) ? bv : akk;
    if (best == 0.0) return false;
    if (p != k) {
      for (int j = lane; j < n; j += 32) {
        const double t = A[k * ld + j];
        A[k * ld + j] = A[p * ld + j];
        A[p * ld + j] = t;
      }
      if (lane == 0) {
        const int t = piv[k];
        piv[k] = piv[p];
        piv[p] = t;
      }
    }
    __syncwarp();
    const double inv = __ddiv_rn(1.0, A[k * ld + k]);
    for (int i = k + 1 + lane; i < n; i += 32) A[i * ld + k] = __dmul_rn(A[i * ld + k], inv);
    __syncwarp();
    for (int j = k + 1 + lane; j < n; j += 32) {
      const double akj = A[k * ld + j];
      for (int i = k + 1; i < n; ++i) {
        const double m = A[i * ld + k];
        if (m != 0.0) A[i * ld + j] = __dsub_rn(A[i * ld + j], __dmul_rn(m, akj));
      }
    }
    __syncwarp();
  }
  return true;
}

// sparse.cpp:343-361, one right-hand side per lane (x: this lane's scratch).
__device__ __forceinline__ void lu_solve_lane(const double* LU, int n, int ld, double* x) {
  for (int i = 1; i < n; ++i) {
    double acc = x[i];
    for (int j = 0; j < i; ++j) acc = __dsub_rn(acc, __dmul_rn(LU[i * ld + j], x[j]));
    x[i] = acc;
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = x[i];
    for (int j = i + 1; j < n; ++j) acc = __dsub_rn(acc, __dmul_rn(LU[i * ld + j], x[j]));
    x[i] = __ddiv_rn(acc, LU[i * ld + i]);
  }
}

// Entries stored for one A^-1 block of order n: full column-major, or the
// symmetrised upper triangle packed column by column (column j = rows 0..j at
// offset j(j+1)/2) when the level's velocity block is symmetric.
__host__ __device__ __forceinline__ long long ainv_len(long long n, bool sym) {
  return sym ? n * (n + 1) / 2 : n * n;
}

struct FactorLayout {
  int D, NV, NP;  // max dim, max nv, max np
  int bytes;      // per warp
  __host__ __device__ FactorLayout(int d, int nv, int np) : D(d), NV(nv), NP(np) {
    size_t dbl = 3 * (size_t)D * D + 2 * (size_t)NP * NV + (size_t)NP * NP +
                 (size_t)(32 + NP) * (size_t)(D > NP ? D : NP);
    size_t ints = (size_t)NV + 2 * (size_t)D + NP;
    bytes = (int)(((dbl * 8 + ints * 4) + 15) / 16 * 16);
  }
};

// Where factor_kernel writes a patch's payload: double entries at
// D[dbase[k] + e*es], int entries at I[ibase[k] + e*es]; es = 1 for the blob
// layout (plus a header at blob + hoff[k]), es = 32 for the interleaved
// bucket layout of the thread-per-patch apply.
struct FactorOut {
  double* D = nullptr;
  int* I = nullptr;
  const long long* dbase = nullptr;
  const long long* ibase = nullptr;
  long long es = 1;
  unsigned char* blob = nullptr;
  const long long* hoff = nullptr;
  const int* sbase = nullptr;
  int pairs = 0;  // paired blob layout for qualifying patches (vanka_paired)
  const unsigned char* nob = nullptr;  // per patch: no stored b_hat (fixed-shape class)
};

__global__ void __launch_bounds__(256) factor_kernel(
    int npatch, int D, int NV, int NP, int wbytes, int sym, const int* __restrict__ rp,
    const int* __restrict__ ci, const double* __restrict__ kv, const int* __restrict__ pptr,
    const int* __restrict__ pidx, const int* __restrict__ vptr, const int* __restrict__ vidx,
    const int* __restrict__ nxs, FactorOut fo, int* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* base = smem + (size_t)wib * wbytes;
  const int DX = D > NP ? D : NP;
  double* Ax = reinterpret_cast<double*>(base);
  double* Ay = Ax + (size_t)D * D;
  double* Winv = Ay + (size_t)D * D;  // D x D inverse columns [c*D + i]
  double* Bm = Winv + (size_t)D * D;  // NP x NV  [a*NV + m]
  double* Um = Bm + (size_t)NP * NV;  // NV x NP  [m*NP + a] (u_hat row-major)
  double* Sm = Um + (size_t)NV * NP;  // NP x NP
  double* W = Sm + (size_t)NP * NP;   // (32 + NP) lanes x DX solve scratch
  int* sv = reinterpret_cast<int*>(W + (size_t)(32 + NP) * DX);
  int* pivx = sv + NV;
  int* pivy = pivx + D;
  int* spiv = pivy + D;
  double* xw = W + (size_t)lane * DX;

  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int k = gw; k < npatch; k += nw) {
    const int v0 = vptr[k], nv = vptr[k + 1] - v0;
    const int p0 = pptr[k], np = pptr[k + 1] - p0;
    const int nx = nxs[k], ny = nv - nx;
    for (int i = lane; i < nv; i += 32) sv[i] = vidx[v0 + i];
    for (int i = lane; i < D * D; i += 32) {
      Ax[i] = 0.0;
      Ay[i] = 0.0;
    }
    for (int i = lane; i < NP * NV; i += 32) Bm[i] = 0.0;
    __syncwarp();
    // gather_dense (vanka.cpp:47-60): A_x, A_y, B
    for (int r = lane; r < nx; r += 32) {
      const int row = sv[r];
      for (int q = rp[row]; q < rp[row + 1]; ++q) {
        const int pos = bsearch_idx(sv, nx, ci[q]);
        if (pos >= 0) Ax[r * D + pos] = kv[q];
      }
    }
    for (int r = lane; r < ny; r += 32) {
      const int row = sv[nx + r];
      for (int q = rp[row]; q < rp[row + 1]; ++q) {
        const int pos = bsearch_idx(sv + nx, ny, ci[q]);
        if (pos >= 0) Ay[r * D + pos] = kv[q];
      }
    }
    for (int a = 0; a < np; ++a) {
      const int row = pidx[p0 + a];
      for (int q = rp[row] + lane; q < rp[row + 1]; q += 32) {
        const int pos = bsearch_idx(sv, nv, ci[q]);
        if (pos >= 0) Bm[a * NV + pos] = kv[q];
      }
    }
    __syncwarp();
    bool ok = true;
    if (nx > 0) ok = warp_lu(Ax, nx, D, pivx, lane);
    if (ok && ny > 0) ok = warp_lu(Ay, ny, D, pivy, lane);
    if (!ok) {
      if (lane == 0) atomicMin(err, k);
      continue;
    }
    // payload entries e of this patch live at D[db + e*es] / I[ib + e*es]
    const long long es = fo.es;
    const long long db = fo.dbase[k], ib = fo.ibase[k];
    // sections: blob order A_x | A_y | U (rows of nv) | B_hat | S^-1, or the
    // streamed thread-per-patch order B_hat | S^-1 | A_x | U_x | A_y | U_y
    double *gAx, *gAy, *gUx, *gUy, *gB, *gS;
    int urx, ury;
    // paired blob: (A_x,A_y) | (U_x,U_y) | (B_x,B_y) interleaved, then S^-1;
    // sa/su = element strides of the A and U sections
    const bool pr = vanka_paired(fo.pairs != 0, nx, ny, np);
    const long long sa = pr ? 2 : es, su = pr ? 2 : es;
    if (pr) {
      const int m = nx > ny ? nx : ny;
      gAx = fo.D + db;
      gAy = gAx + 1;
      gUx = gAx + 2 * ainv_len(m, true);
      gUy = gUx + 1;
      gB = gUx + 2LL * np * m;
      gS = gB + ((fo.nob && fo.nob[k]) ? 0 : 2LL * np * m);
      urx = ury = m;  // pair rows of U: [a * m + i]
      // zero padding of the smaller component
      if (nx != ny)
        for (long long e = lane;
             e < vanka_paired_doubles(m, np) - (long long)np * np -
                     ((fo.nob && fo.nob[k]) ? 2LL * np * m : 0);
             e += 32)
          gAx[e] = 0.0;
      __syncwarp();
    } else {
      gAx = fo.D + db;
      gAy = gAx + ainv_len(nx, sym) * es;
      gUx = gAy + ainv_len(ny, sym) * es;
      gUy = gUx + (long long)nx * es;
      gB = gUx + (long long)np * nv * es;
      gS = gB + (long long)np * nv * es;
      urx = ury = nv;
    }
    int* gidx = fo.I + ib;
    // per component: RHS t < n are unit vectors (inverse columns, each one
    // dense_lu_solve(lu, e_t)), t = n + j are -B(j, comp)^T (u_hat columns,
    // vanka.cpp:99-111)
    for (int comp = 0; comp < 2; ++comp) {
      const int n = comp == 0 ? nx : ny;
      const int c0 = comp == 0 ? 0 : nx;
      const double* LU = comp == 0 ? Ax : Ay;
      const int* pv = comp == 0 ? pivx : pivy;
      double* gA = comp == 0 ? gAx : gAy;
      if (n == 0) continue;
      for (int t0 = 0; t0 < n + np; t0 += 32) {
        const int t = t0 + lane;
        if (t < n + np) {
          double* x = (t < n) ? Winv + (size_t)t * D : xw;
          for (int i = 0; i < n; ++i) {
            const int src = pv[i];
            x[i] = (t < n) ? (src == t ? 1.0 : 0.0) : -Bm[(t - n) * NV + c0 + src];
          }
          lu_solve_lane(LU, n, D, x);
          if (t >= n)
            for (int i = 0; i < n; ++i) Um[(c0 + i) * NP + (t - n)] = x[i];
        }
      }
      __syncwarp();
      if (sym) {
        // symmetrised upper triangle, packed by columns
        for (int c = 0; c < n; ++c)
          for (int i = lane; i <= c; i += 32)
            gA[((long long)c * (c + 1) / 2 + i) * sa] =
                0.5 * (Winv[(size_t)c * D + i] + Winv[(size_t)i * D + c]);
      } else {
        for (int e = lane; e < n * n; e += 32) gA[e * es] = Winv[(size_t)(e / n) * D + (e % n)];
      }
      __syncwarp();
    }
    double* Sinv = Winv;  // the inverse columns are written out; reuse the space
    // S = B u_hat (vanka.cpp:112-119)
    for (int e = lane; e < np * np; e += 32) {
      const int a = e / np, cc = e % np;
      double acc = 0.0;
      for (int m = 0; m < nv; ++m) acc = __dadd_rn(acc, __dmul_rn(Bm[a * NV + m], Um[m * NP + cc]));
      Sm[a * np + cc] = acc;
    }
    __syncwarp();
    if (!warp_lu(Sm, np, np, spiv, lane)) {
      if (lane == 0) atomicMin(err, k);
      continue;
    }
    // S^-1 columns from unit vectors (vanka.cpp:126-132), row-major
    if (lane < np) {
      for (int i = 0; i < np; ++i) xw[i] = spiv[i] == lane ? 1.0 : 0.0;
      lu_solve_lane(Sm, np, np, xw);
      for (int i = 0; i < np; ++i) Sinv[i * np + lane] = xw[i];
    }
    __syncwarp();
    for (int e = lane; e < np * np; e += 32) gS[e * es] = Sinv[e];
    // b_hat = S^-1 u_hat^T (vanka.cpp:133-140); stored [a*nv + j]
    for (int e = lane; e < np * nv; e += 32) {
      const int a = e / nv, j = e % nv;
      double acc = 0.0;
      for (int m = 0; m < np; ++m) acc = __dadd_rn(acc, __dmul_rn(Sinv[a * np + m], Um[j * NP + m]));
      if (pr && fo.nob && fo.nob[k]) continue;
      if (pr)
        gB[2LL * a * (nx > ny ? nx : ny) + (j < nx ? 2 * j : 2 * (j - nx) + 1)] = acc;
      else
        gB[e * es] = acc;
    }
    // u_hat stored by rows a: [a*urx + i] (x part) and [a*ury + i - nx] (y part)
    for (int e = lane; e < np * nv; e += 32) {
      const int a = e / nv, i = e % nv;
      if (i < nx)
        gUx[((long long)a * urx + i) * su] = Um[i * NP + a];
      else
        gUy[((long long)a * ury + i - nx) * su] = Um[i * NP + a];
    }
    for (int i = lane; i < nv; i += 32) gidx[i * es] = sv[i];
    for (int a = lane; a < np; a += 32) gidx[(nv + a) * es] = pidx[p0 + a];
    if (lane == 0 && fo.hoff) {
      int* hdr = reinterpret_cast<int*>(fo.blob + fo.hoff[k]);
      hdr[0] = nx;
      hdr[1] = ny;
      hdr[2] = np;
      hdr[3] = fo.sbase[k];
    }
    __syncwarp();
  }
}

// keys[slot] = dof of that slot: patch k's entry e sits at slot sbase[k] + e*es
// (velocity entries first, then pressure, as the apply writes them)
__global__ void slot_keys_kernel(int npatch, const int* pptr, const int* pidx, const int* vptr,
                                 const int* vidx, const int* sbase, int es, int* keys) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < npatch; k += gridDim.x * blockDim.x) {
    int s = sbase[k];
    for (int q = vptr[k]; q < vptr[k + 1]; ++q, s += es) keys[s] = vidx[q];
    for (int q = pptr[k]; q < pptr[k + 1]; ++q, s += es) keys[s] = pidx[q];
  }
}

__global__ void fill_int_kernel(long long n, int v, int* a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void count_int_kernel(long long n, const int* key, int* cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + key[i], 1);
}

__global__ void iota_int_kernel(long long n, int* a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

// vanka.cpp:67-73: w_d = 1 / #patches containing d (0 if none)
__global__ void weights_kernel(int n, const int* dof_ptr, double* w) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const int m = dof_ptr[d + 1] - dof_ptr[d];
    w[d] = m > 0 ? 1.0 / (double)m : 0.0;
  }
}

static int grid_for(Ctx& c, long long n) {
  return (int)std::max(1LL, std::min((n + 255) / 256, (long long)c.num_sms * 16));
}

// Relative asymmetry of the velocity block K[0:n_u, 0:n_u]: max |a_ij - a_ji|
// and max |a_ij| (as ordered uint64 bit patterns of non-negative doubles).
__global__ void asym_kernel(int n_u, const int* rp, const int* ci, const double* v,
                            unsigned long long* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_u; i += gridDim.x * blockDim.x) {
    double dmax = 0.0, amax = 0.0;
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const int j = ci[q];
      if (j >= n_u) break;
      amax = fmax(amax, fabs(v[q]));
      if (j <= i) continue;
      int lo = rp[j], hi = rp[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < i) lo = mid + 1; else hi = mid;
      }
      const double vt = (lo < rp[j + 1] && ci[lo] == i) ? v[lo] : 0.0;
      dmax = fmax(dmax, fabs(v[q] - vt));
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(dmax));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(amax));
  }
}

// A^-1 is stored as its symmetrised upper triangle when the velocity block is
// symmetric to 1e-12 relative (the reference's b_hat formula, vanka.cpp:133,
// assumes symmetric A as well); SAG_VANKA_SYM=0/1 overrides.
static bool velocity_block_symmetric(Ctx& c, const Matrix& k, int n_u) {
  if (const char* e = getenv("SAG_VANKA_SYM")) return atoi(e) != 0;
  if (n_u <= 0) return true;
  DevBuf<unsigned long long> o(2);
  SAG_CUDA(cudaMemsetAsync(o.p, 0, 16, c.stream));
  asym_kernel<<<grid_for(c, n_u), 256, 0, c.stream>>>(n_u, k.rp.p, k.ci.p, k.v.p, o.p);
  SAG_LAUNCHED(c);
  unsigned long long h[2];
  SAG_CUDA(cudaMemcpyAsync(h, o.p, 16, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  double d, a;
  std::memcpy(&d, &h[0], 8);
  std::memcpy(&a, &h[1], 8);
  return d <= 1e-12 * a;
}

__global__ void inverse_perm_kernel(long long n, const int* __restrict__ perm, int* __restrict__ inv) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    inv[perm[t]] = (int)t;
}
// blob of patch i: its nv + np result positions right after its dof indices
__global__ void blob_pos_kernel(int npatch, const int* __restrict__ vptr,
                                const int* __restrict__ pptr, const long long* __restrict__ ibase,
                                const int* __restrict__ sbase, const int* __restrict__ pos,
                                int* __restrict__ I) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npatch; i += gridDim.x * blockDim.x) {
    const int cnt = (vptr[i + 1] - vptr[i]) + (pptr[i + 1] - pptr[i]);
    int* dst = I + ibase[i] + cnt;
    for (int e = 0; e < cnt; ++e) dst[e] = pos[sbase[i] + e];
  }
}

std::unique_ptr<Vanka> factor_patches_dev(Ctx& c, const Matrix& k, const Patches& p, int n_u) {
  SAG_REQUIRE(k.nrows == k.ncols, SAG_DIMENSION_MISMATCH, "factor_patches: K must be square");
  SAG_REQUIRE(p.max_np <= 4, SAG_ERROR, "factor_patches: at most 4 pressure seeds per patch");
  SAG_REQUIRE(p.max_dim <= 128, SAG_ERROR,
              "factor_patches: velocity blocks larger than 128 per component are not supported");
  auto f = std::make_unique<Vanka>();
  const int np_ = p.npatch;
  f->n = k.nrows;
  f->n_u = std::min(std::max(n_u, 0), k.nrows);
  f->npatch = np_;
  f->max_dim = p.max_dim;
  f->max_nv = p.max_nv;
  f->max_np = p.max_np;
  f->sym = velocity_block_symmetric(c, k, std::min(std::max(n_u, 0), k.nrows));
  const bool sym = f->sym;
  // the paired path lives in the one-row-per-lane kernel (R = 1)
  f->pairs = sym && p.max_np <= 4 && env_int("SAG_VANKA_PAIRS", 1) != 0;
  // host bookkeeping: blob offsets, slot bases, storage accounting (vanka.cpp:142-144)
  std::vector<int> vptr(np_ + 1), pptr(np_ + 1), nx(std::max(np_, 1));
  SAG_CUDA(cudaMemcpyAsync(vptr.data(), p.vptr.p, sizeof(int) * (np_ + 1), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaMemcpyAsync(pptr.data(), p.pptr.p, sizeof(int) * (np_ + 1), cudaMemcpyDeviceToHost, c.stream));
  if (np_) SAG_CUDA(cudaMemcpyAsync(nx.data(), p.nx.p, sizeof(int) * np_, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  f->h_nx.resize(np_);
  f->h_nv.resize(np_);
  f->h_np.resize(np_);
  for (int i = 0; i < np_; ++i) {
    const long long nv = vptr[i + 1] - vptr[i], npp = pptr[i + 1] - pptr[i];
    const long long x = nx[i], y = nv - x;
    f->h_nx[i] = (int)x;
    f->h_nv[i] = (int)nv;
    f->h_np[i] = (int)npp;
    f->a_factor_bytes += 8 * (x * x + y * y);
    f->aux_bytes += 8 * (2 * nv * npp + npp * npp);
    f->dense_inverse_bytes += 8 * (nv + npp) * (nv + npp);
  }
  // nob[i]: the patch's blob stores no b_hat (the fixed-shape class recomputes
  // it from S^-1 and U_hat, vanka.cpp:133-140, bitwise)
  std::vector<unsigned char>& nob = f->h_nob;
  nob.assign(np_, 0);
  auto ndbl = [&](int i) {
    const long long nv = f->h_nv[i], npp = f->h_np[i], x = f->h_nx[i], y = nv - x;
    if (vanka_paired(f->pairs, (int)x, (int)y, (int)npp))
      return vanka_paired_doubles((int)std::max(x, y), (int)npp) -
             (nob[i] ? 2 * npp * std::max(x, y) : 0);
    return ainv_len(x, sym) + ainv_len(y, sym) + 2 * nv * npp + npp * npp;
  };
  f->h_dbase.assign(np_, 0);
  f->h_ibase.assign(np_, 0);
  std::vector<long long> h_hoff;  // blob byte offset per patch id
  std::vector<int> sbase(std::max(np_, 1), 0);
  long long slots = 0;
  // a level is paired only if every patch is (one kernel path per level)
  for (int i = 0; i < np_ && f->pairs; ++i) {
    const int x = f->h_nx[i], y = f->h_nv[i] - x;
    f->pairs = vanka_paired(true, x, y, f->h_np[i]);
    f->pair_rows = std::max(f->pair_rows, std::max(x, y) + f->h_np[i]);
  }
  if (!f->pairs) f->pair_rows = 0;
  {
    // size classes: the rows per lane the apply needs (paired: m + np, else
    // max(nx, ny)) -> R = ceil(rows / 32). Blobs are stored class by class
    // (stable in patch order), so each class is one contiguous launch with
    // its own stage size; slots stay in patch order.
    // class key 4 R + (lanes per patch: 32 / 16 / 8 -> 0 / 1 / 2); small
    // paired patches go to the sub-warp kernel (several patches per warp)
    const bool subwarp = f->pairs && env_int("SAG_VANKA_SUBWARP", 1) != 0;
    f->seq = env_int("SAG_VANKA_SEQGATHER", 1) != 0;
    // fixed-shape class: the SV fine level's element triples with
    // max(nx, ny) = 6, np = 3 get a kernel with the shape compiled in
    const bool fixed63 = f->pairs && subwarp && sym && env_int("SAG_VANKA_FIXED", 1) != 0;
    auto is_fixed = [&](int i) {
      const int x = f->h_nx[i], y = f->h_nv[i] - x;
      return fixed63 && std::max(x, y) == 6 && f->h_np[i] == 3;
    };
    auto key_of = [&](int i) {
      const int x = f->h_nx[i], y = f->h_nv[i] - x;
      const int rows = std::max(x, y) + (f->pairs ? f->h_np[i] : 0);
      const int R = std::max(1, (rows + 31) / 32);
      if (is_fixed(i)) return 4 * R + 3;
      const int l = !subwarp ? 0 : rows <= 8 ? 2 : rows <= 16 ? 1 : 0;
      return 4 * R + l;
    };
    // a sub-warp class only pays off when it is a large share of the level
    // (a separate launch with its own grid): stragglers join the 32-lane class
    int nkey[16] = {0};
    for (int i = 0; i < np_; ++i) ++nkey[std::min(key_of(i), 15)];
    const int min_sub = std::max(4096, np_ / 8);
    auto r_of = [&](int i) {
      const int k = key_of(i);
      return (k % 4 != 0 && nkey[std::min(k, 15)] < min_sub) ? 4 * (k / 4) : k;
    };
    std::vector<int> order(np_);
    for (int i = 0; i < np_; ++i) {
      order[i] = i;
      nob[i] = r_of(i) % 4 == 3 ? 1 : 0;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return r_of(a) < r_of(b); });
    f->h_order = order;
    std::vector<long long> off(np_ + 1, 0);
    h_hoff.assign(np_, 0);
    int maxbytes = 16;
    f->rclasses.clear();
    for (int q = 0; q < np_; ++q) {
      const int i = order[q];
      long long bytes = 16 + 8 * ndbl(i) + 4 * (f->h_nv[i] + f->h_np[i]) * (f->seq ? 2 : 1);
      bytes = (bytes + 15) / 16 * 16;
      h_hoff[i] = off[q];
      off[q + 1] = off[q] + bytes;
      maxbytes = std::max<long long>(maxbytes, bytes);
      f->h_dbase[i] = (off[q] + 16) / 8;
      f->h_ibase[i] = (off[q] + 16 + 8 * ndbl(i)) / 4;
      const int key = r_of(i), R = key / 4, fx = key % 4 == 3;
      const int lpp = fx ? 9 : 32 >> (key % 4);
      if (f->rclasses.empty() || f->rclasses.back().R != R || f->rclasses.back().lpp != lpp ||
          f->rclasses.back().fm != (fx ? 6 : 0)) {
        f->rclasses.push_back({R, q, q + 1, 16, lpp});
        if (fx) {
          f->rclasses.back().fm = 6;
          f->rclasses.back().fnp = 3;
        }
      }
      auto& cl = f->rclasses.back();
      cl.k1 = q + 1;
      cl.slot_bytes = std::max<long long>(cl.slot_bytes, bytes);
      cl.bytes += bytes;
    }
    for (int i = 0; i < np_; ++i) {
      sbase[i] = (int)slots;
      slots += f->h_nv[i] + f->h_np[i];
      SAG_REQUIRE(slots < (1LL << 31), SAG_DIMENSION_MISMATCH, "factor_patches: too many slots");
    }
    f->slot_bytes = maxbytes;
    f->blob_bytes = off[np_];
    f->blob.alloc(std::max<long long>(off[np_], 16));
    f->off.alloc(np_ + 1);
    SAG_CUDA(cudaMemcpyAsync(f->off.p, off.data(), sizeof(long long) * (np_ + 1),
                             cudaMemcpyHostToDevice, c.stream));
  }
  f->nslots = slots;
  DevBuf<int> dsbase(std::max(np_, 1));
  DevBuf<long long> ddbase(std::max(np_, 1)), dibase(std::max(np_, 1));
  SAG_CUDA(cudaMemcpyAsync(dsbase.p, sbase.data(), sizeof(int) * sbase.size(), cudaMemcpyHostToDevice, c.stream));
  if (np_) {
    SAG_CUDA(cudaMemcpyAsync(ddbase.p, f->h_dbase.data(), sizeof(long long) * np_,
                             cudaMemcpyHostToDevice, c.stream));
    SAG_CUDA(cudaMemcpyAsync(dibase.p, f->h_ibase.data(), sizeof(long long) * np_,
                             cudaMemcpyHostToDevice, c.stream));
  }
  const int es = 1;

  // dof -> slot map (stable sort of slot ids by dof) and PoU weights
  const int n = k.nrows;
  f->out.alloc(std::max<long long>(slots, 1));
  f->w.alloc(std::max(n, 1));
  f->dof_ptr.alloc(n + 1);
  f->dof_slot.alloc(std::max<long long>(slots, 1));
  if (slots > 0) {
    DevBuf<int> keys(slots), keys_sorted(slots), ids(slots), cnt(n + 1);
    fill_int_kernel<<<grid_for(c, slots), 256, 0, c.stream>>>(slots, n, keys.p);  // padding -> n
    SAG_LAUNCHED(c);
    slot_keys_kernel<<<grid_for(c, np_), 256, 0, c.stream>>>(np_, p.pptr.p, p.pidx.p, p.vptr.p,
                                                             p.vidx.p, dsbase.p, es, keys.p);
    SAG_LAUNCHED(c);
    iota_int_kernel<<<grid_for(c, slots), 256, 0, c.stream>>>(slots, ids.p);
    SAG_LAUNCHED(c);
    SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (n + 1), c.stream));
    count_int_kernel<<<grid_for(c, slots), 256, 0, c.stream>>>(slots, keys.p, cnt.p);
    SAG_LAUNCHED(c);
    size_t t1 = 0, t2 = 0;
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, cnt.p, f->dof_ptr.p, n + 1, c.stream));
    SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, keys.p, keys_sorted.p, ids.p,
                                             f->dof_slot.p, (int)slots, 0, 32, c.stream));
    DevBuf<unsigned char> ws(std::max(t1, t2));
    SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, t1, cnt.p, f->dof_ptr.p, n + 1, c.stream));
    SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, t2, keys.p, keys_sorted.p, ids.p,
                                             f->dof_slot.p, (int)slots, 0, 32, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  } else {
    SAG_CUDA(cudaMemsetAsync(f->dof_ptr.p, 0, sizeof(int) * (n + 1), c.stream));
  }
  weights_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(n, f->dof_ptr.p, f->w.p);
  SAG_LAUNCHED(c);

  // batched factorization
  if (np_ > 0) {
    FactorLayout L(std::max(p.max_dim, 1), std::max(p.max_nv, 1), std::max(p.max_np, 1));
    int warps = std::max(1, std::min(8, (200 * 1024) / L.bytes));
    SAG_REQUIRE((size_t)L.bytes <= 220 * 1024, SAG_ERROR,
                "factor_patches: patch too large for shared-memory factorization");
    const int smem = warps * L.bytes;
    SAG_CUDA(cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    DevBuf<int> err(1);
    const int big = 0x7fffffff;
    SAG_CUDA(cudaMemcpyAsync(err.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
    const int blocks = std::max(1, std::min((np_ + warps - 1) / warps, c.num_sms * 8));
    FactorOut fo;
    DevBuf<long long> dhoff;
    DevBuf<unsigned char> dnob;
    fo.es = es;
    fo.dbase = ddbase.p;
    fo.ibase = dibase.p;
    fo.sbase = dsbase.p;
    {
      fo.D = reinterpret_cast<double*>(f->blob.p);
      fo.I = reinterpret_cast<int*>(f->blob.p);
      fo.blob = f->blob.p;
      dhoff.alloc(std::max(np_, 1));
      if (np_)
        SAG_CUDA(cudaMemcpyAsync(dhoff.p, h_hoff.data(), sizeof(long long) * np_,
                                 cudaMemcpyHostToDevice, c.stream));
      fo.hoff = dhoff.p;
      fo.pairs = f->pairs ? 1 : 0;
      if (np_) {
        dnob.alloc(np_);
        SAG_CUDA(cudaMemcpyAsync(dnob.p, f->h_nob.data(), np_, cudaMemcpyHostToDevice, c.stream));
        fo.nob = dnob.p;
      }
    }
    factor_kernel<<<blocks, warps * 32, smem, c.stream>>>(
        np_, L.D, L.NV, L.NP, L.bytes, sym ? 1 : 0, k.rp.p, k.ci.p, k.v.p, p.pptr.p, p.pidx.p,
        p.vptr.p, p.vidx.p, p.nx.p, fo, err.p);
    SAG_LAUNCHED(c);
    int herr = big;
    SAG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    if (herr != big)
      throw Error(SAG_SINGULAR_PATCH,
                  "factor_patches: singular velocity or Schur block in patch " + std::to_string(herr));
  }
  // dof-ordered result positions into the blobs (Vanka::seq): position of
  // slot t in the dof-sorted order = its rank in dof_slot
  if (f->seq && slots > 0) {
    DevBuf<int> pos(slots);
    inverse_perm_kernel<<<grid_for(c, slots), 256, 0, c.stream>>>(slots, f->dof_slot.p, pos.p);
    SAG_LAUNCHED(c);
    blob_pos_kernel<<<grid_for(c, np_), 256, 0, c.stream>>>(
        np_, p.vptr.p, p.pptr.p, dibase.p, dsbase.p, pos.p, reinterpret_cast<int*>(f->blob.p));
    SAG_LAUNCHED(c);
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  }
  return f;
}

// ========================================================== apply_vanka ==

// Warp-per-patch additive Vanka: each warp streams its patches' factor blobs
// through an NSTAGE-deep shared-memory ring filled by cp.async.bulk (TMA
// engine), gathers r at the patch dofs, solves with the block factors
// (t = A^-1 b_u; x_p = S^-1 b_p + B_hat b_u; x_u = t + U_hat x_p,
// vanka.cpp:161-181) and writes the unweighted local result to its slots.
// Blob pointers of one patch (layout in internal.cuh).
// Predicated 16-byte shared load (no branch; 0 when !pred).
__device__ __forceinline__ double2 lds_v2_pred(const double2* p, bool pred) {
  double2 v = make_double2(0.0, 0.0);
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q ld.shared.v2.f64 {%0, %1}, [%2];\n}\n"
      : "+d"(v.x), "+d"(v.y)
      : "r"(smem_u32(p)), "r"((int)pred));
  return v;
}

// Paired blobs (vanka_paired): m = max(nx, ny); Ax points at the (A_x, A_y)
// pairs, U / Bh at the (U_x, U_y) / (B_x, B_y) pairs, Ay is unused.
struct PatchView {
  int nx, ny, np, sbase, nv, m;
  bool paired;
  const double *Ax, *Ay, *U, *Bh, *Si;
  const int* idx;
  const int* pos;  // dof-ordered result positions (Vanka::seq), after idx
  // where local result i goes: its dof-ordered position, or slot sbase + i
  __device__ __forceinline__ int opos(int seq, int i) const { return seq ? pos[i] : sbase + i; }
};
template <bool SYM>
__device__ __forceinline__ PatchView patch_view(const unsigned char* B, bool pairs) {
  PatchView v;
  const int4 hdr = *reinterpret_cast<const int4*>(B);
  v.nx = hdr.x;
  v.ny = hdr.y;
  v.np = hdr.z;
  v.sbase = hdr.w;
  v.nv = v.nx + v.ny;
  v.m = v.nx > v.ny ? v.nx : v.ny;
  v.paired = SYM && vanka_paired(pairs, v.nx, v.ny, v.np);
  v.Ax = reinterpret_cast<const double*>(B + 16);
  if (v.paired) {
    v.Ay = v.Ax + 1;
    v.U = v.Ax + v.m * (v.m + 1);
    v.Bh = v.U + 2 * v.np * v.m;
    v.Si = v.Bh + 2 * v.np * v.m;
    v.idx = reinterpret_cast<const int*>(v.Si + v.np * v.np);
    v.pos = v.idx + v.nv + v.np;
    return v;
  }
  v.Ay = v.Ax + (SYM ? v.nx * (v.nx + 1) / 2 : v.nx * v.nx);
  v.U = v.Ay + (SYM ? v.ny * (v.ny + 1) / 2 : v.ny * v.ny);
  v.Bh = v.U + v.np * v.nv;
  v.Si = v.Bh + v.np * v.nv;
  v.idx = reinterpret_cast<const int*>(v.Si + v.np * v.np);
  v.pos = v.idx + v.nv + v.np;
  return v;
}

// Warp-per-patch additive Vanka. Each warp streams its patches' factor blobs
// through an NSTAGE-deep shared-memory ring filled by cp.async.bulk (TMA
// engine, L2 evict-first: the factors are read once per sweep, r stays in L2),
// solves with the block factors (t = A^-1 b_u; x_p = S^-1 b_p + B_hat b_u;
// x_u = t + U_hat x_p, vanka.cpp:161-181) and writes the unweighted local
// result to its slots. The gather of r for patch k+1 is issued before the
// solve of patch k (double-buffered), hiding its L2 latency.
// SYM: A^-1 blocks are packed symmetrised upper triangles; lane i reads
// column j rows (i <= j) or column i rows (i > j): both conflict-free.
// NPM: upper bound on pressure seeds per patch (1 for TH / ISO levels).
template <int R, bool SYM, int NPM>
__global__ void __launch_bounds__(256) vanka_patch_kernel(
    int npatch, const unsigned char* __restrict__ blob, const long long* __restrict__ off,
    int slot_bytes, int nstage, int sb_len, int pairs, const double* __restrict__ r,
    double* __restrict__ out, int seq, const int* gate) {
  if (gate && *gate) return;
  constexpr int G = 2 * R + 1;  // gathered values per lane (nv + np <= 32 G)
  // paired blobs (vanka_paired) exist only on symmetric levels, R <= 2
  constexpr bool kPair = SYM && R <= 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbar = (nstage + 1) & ~1;  // keeps the r buffers 16-byte aligned
  unsigned char* ring = smem + (size_t)wib * nstage * slot_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)warps * nstage * slot_bytes) +
                   (size_t)wib * nbar;
  double* sbuf = reinterpret_cast<double*>(smem + (size_t)warps * nstage * slot_bytes +
                                           (size_t)warps * nbar * 8) +
                 (size_t)wib * 2 * sb_len;
  const int first = blockIdx.x * warps + wib;
  const int stride = gridDim.x * warps;
  const uint64_t policy = evict_first_policy();
  auto issue_at = [&](int s, long long o0, long long o1) {
    const unsigned bytes = (unsigned)(o1 - o0);
    mbar_expect_tx(bars + s, bytes);
    bulk_copy_hint(ring + (size_t)s * slot_bytes, blob + o0, bytes, bars + s, policy);
  };
  // r at a patch's dofs goes to the r buffer in the order its solve reads:
  // x dofs, y dofs, pressure; a paired patch interleaves (x_j, y_j) over
  // j < m (padding zeroed by pad_pairs) with the pressure at 2m
  auto slot_of = [&](const PatchView& w, int i) {
    if (kPair && w.paired)
      return i < w.nx ? 2 * i : (i < w.nv ? 2 * (i - w.nx) + 1 : 2 * w.m + (i - w.nv));
    return i;
  };
  auto pad_pairs = [&](const PatchView& w, double* dst) {
    if (kPair && w.paired && w.nx != w.ny) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int j = lane + 32 * q;
        if (j >= w.nx && j < w.m) dst[2 * j] = 0.0;
        if (j >= w.ny && j < w.m) dst[2 * j + 1] = 0.0;
      }
    }
  };
  if (lane == 0) {
    for (int s = 0; s < nstage; ++s) mbar_init(bars + s, 1);
    mbar_init_fence();
    for (int s = 0; s < nstage; ++s) {
      const int kk = first + s * stride;
      if (kk < npatch) issue_at(s, off[kk], off[kk + 1]);
    }
  }
  __syncwarp();
  unsigned phase = 0;  // bit s: parity of the next wait on stage s
  if (first < npatch) {
    mbar_wait(bars, 0);
    phase ^= 1u;
    const PatchView v = patch_view<SYM>(ring, pairs != 0);
    for (int i = lane; i < v.nv + v.np; i += 32) sbuf[slot_of(v, i)] = __ldg(r + v.idx[i]);
    pad_pairs(v, sbuf);
  }
  __syncwarp();
  int csl[R];
#pragma unroll
  for (int q = 0; q < R; ++q) csl[q] = (lane + 32 * q) * (lane + 32 * q + 1) / 2;
  int stage = 0, it = 0;
  for (int k = first; k < npatch; k += stride, ++it) {
    // offsets of the blob that refills this stage, loaded now so the refill
    // at the end of the iteration does not wait on them
    const int kr = k + nstage * stride;
    long long ro0 = 0, ro1 = 0;
    if (lane == 0 && kr < npatch) {
      ro0 = __ldg(off + kr);
      ro1 = __ldg(off + kr + 1);
    }
    const PatchView v = patch_view<SYM>(ring + (size_t)stage * slot_bytes, pairs != 0);
    const double* sb = sbuf + (it & 1) * sb_len;
    // prefetch r at the next patch's dofs (its blob was issued nstage-1 solves ago)
    const int kn = k + stride;
    const int sn = stage + 1 == nstage ? 0 : stage + 1;
    double g[G];
    int gn = 0;
    PatchView w{};
    if (kn < npatch) {
      mbar_wait(bars + sn, (phase >> sn) & 1u);
      phase ^= 1u << sn;
      w = patch_view<SYM>(ring + (size_t)sn * slot_bytes, pairs != 0);
      gn = w.nv + w.np;
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int i = lane + 32 * q;
        g[q] = i < gn ? __ldg(r + w.idx[i]) : 0.0;
      }
    }
    const int nx = v.nx, ny = v.ny, np = NPM == 1 ? 1 : v.np, nv = v.nv;
    if (kPair && v.paired) {
      // paired patch: virtual row i = lane + 32 q (q < R) is matrix row i
      // (i < m) of both components -- one 16-byte load of (A_x, A_y)(i, j) and
      // one broadcast of (b_x, b_y)_j per column, zero padding beyond nx / ny
      // -- or, for m <= i < m + np, b_hat row i - m over the (B_x, B_y) pairs,
      // so x_p needs no warp reduction
      const int mm = v.m, npp = NPM == 1 ? 1 : v.np;
      const double2* AP = reinterpret_cast<const double2*>(v.Ax);
      const double2* SB = reinterpret_cast<const double2*>(sb);
      const int boff = (int)(reinterpret_cast<const double2*>(v.Bh) - AP);
      // rows past m + np issue no load: a column costs ceil((m + np) / 8)
      // shared-memory wavefronts (the LSU data pipe bounds this kernel)
      bool act[R];
      int cl[R];
      double tx[R], ty[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        act[q] = i < mm + npp;
        cl[q] = i >= mm ? boff + (i - mm) * mm : csl[q];
        tx[q] = ty[q] = 0.0;
      }
      int csj = 0;
#pragma unroll 4
      for (int j = 0; j < mm; csj += ++j) {
        const double2 b = SB[j];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = lane + 32 * q;
          const double2 a = lds_v2_pred(AP + (i <= j ? csj + i : cl[q] + j), act[q]);
          tx[q] = fma(a.x, b.x, tx[q]);
          ty[q] = fma(a.y, b.y, ty[q]);
        }
      }
      // x_p = S^-1 b_p + b_hat . b_u (vanka.cpp:168-174), on virtual row m + a
      // (every lane evaluates it -- rows clamped into range -- and only the
      // b_hat rows store: no divergent block)
      double xl[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        const int ar = min(max(i - mm, 0), npp - 1);
        xl[q] = tx[q] + ty[q];
#pragma unroll
        for (int e = 0; e < NPM; ++e)
          if (e < npp) xl[q] = fma(v.Si[ar * npp + e], sb[2 * mm + e], xl[q]);
        if (i >= mm && i < mm + npp) out[v.opos(seq, nv + ar)] = xl[q];
      }
      double xp[NPM];
#pragma unroll
      for (int e = 0; e < NPM; ++e) {
        xp[e] = 0.0;
        if (e < npp) {
          const int src = mm + e;  // warp-uniform
          double sv = xl[0];
#pragma unroll
          for (int q = 1; q < R; ++q)
            if ((src >> 5) == q) sv = xl[q];
          xp[e] = __shfl_sync(0xffffffffu, sv, src & 31);
        }
      }
      // x_u = t + U_hat x_p (vanka.cpp:176-180)
      const double2* UP = reinterpret_cast<const double2*>(v.U);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < mm) {
          double ox = tx[q], oy = ty[q];
#pragma unroll
          for (int e = 0; e < NPM; ++e)
            if (e < npp) {
              const double2 u = UP[e * mm + i];
              ox = fma(u.x, xp[e], ox);
              oy = fma(u.y, xp[e], oy);
            }
          if (i < nx) out[v.opos(seq, i)] = ox;
          if (i < ny) out[v.opos(seq, nx + i)] = oy;
        }
      }
    } else {
      const double* Ax = v.Ax;
      const double* Ay = v.Ay;
      const double* U = v.U;
      const double* Bh = v.Bh;
      const double* Si = v.Si;
      // t = A^-1 b_u per component (vanka.cpp:164-166): columns j < min(nx, ny)
      // update both components, the rest only the larger one (no per-column
      // component predicates); SYM column offsets j(j+1)/2 are carried along
      double tx[R], ty[R];
#pragma unroll
      for (int q = 0; q < R; ++q) tx[q] = ty[q] = 0.0;
      const int nmin = nx < ny ? nx : ny, nmax = nx > ny ? nx : ny;
      int csj = 0;
      int j = 0;
      for (; j < nmin; csj += ++j) {
        const double bx = sb[j];
        const double by = sb[nx + j];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = lane + 32 * q;
          const int a = SYM ? (i <= j ? csj + i : csl[q] + j) : 0;
          if (i < nx) tx[q] = fma(SYM ? Ax[a] : Ax[j * nx + i], bx, tx[q]);
          if (i < ny) ty[q] = fma(SYM ? Ay[a] : Ay[j * ny + i], by, ty[q]);
        }
      }
      if (nx > ny) {
        for (; j < nmax; csj += ++j) {
          const double bx = sb[j];
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int i = lane + 32 * q;
            const int a = SYM ? (i <= j ? csj + i : csl[q] + j) : j * nx + i;
            if (i < nx) tx[q] = fma(Ax[a], bx, tx[q]);
          }
        }
      } else {
        for (; j < nmax; csj += ++j) {
          const double by = sb[nx + j];
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int i = lane + 32 * q;
            const int a = SYM ? (i <= j ? csj + i : csl[q] + j) : j * ny + i;
            if (i < ny) ty[q] = fma(Ay[a], by, ty[q]);
          }
        }
      }
      // x_p = S^-1 b_p + B_hat b_u (vanka.cpp:168-174)
      double xp[NPM];
#pragma unroll
      for (int a = 0; a < NPM; ++a) {
        xp[a] = 0.0;
        if (a < np) {
          double part = 0.0;
          for (int m = lane; m < nv; m += 32) part = fma(Bh[a * nv + m], sb[m], part);
          part = warp_sum(part);
          double sp = 0.0;
#pragma unroll
          for (int q = 0; q < NPM; ++q)
            if (q < np) sp = fma(Si[a * np + q], sb[nv + q], sp);
          xp[a] = sp + part;
          if (lane == 0) out[v.opos(seq, nv + a)] = xp[a];
        }
      }
      // x_u = t + U_hat x_p (vanka.cpp:176-180)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < nx) {
          double t = tx[q];
#pragma unroll
          for (int a = 0; a < NPM; ++a)
            if (a < np) t = fma(U[a * nv + i], xp[a], t);
          out[v.opos(seq, i)] = t;
        }
        if (i < ny) {
          double t = ty[q];
#pragma unroll
          for (int a = 0; a < NPM; ++a)
            if (a < np) t = fma(U[a * nv + nx + i], xp[a], t);
          out[v.opos(seq, nx + i)] = t;
        }
      }
    }
    // publish the prefetched r values for the next patch
    double* sbn = sbuf + ((it + 1) & 1) * sb_len;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int i = lane + 32 * q;
      if (i < gn) sbn[slot_of(w, i)] = g[q];
    }
    pad_pairs(w, sbn);
    __syncwarp();
    if (lane == 0 && kr < npatch) {
      fence_proxy_async();
      issue_at(stage, ro0, ro1);
    }
    stage = sn;
  }
}

// Sub-warp paired Vanka for small patches (m + np <= LPP < 32): the warp
// solves P = 32 / LPP consecutive patches at once, lane group g = lane / LPP
// on patch q P + g, with the row / b_hat-row mapping of the paired path of
// vanka_patch_kernel inside each group. The P blobs of a group are adjacent
// in the class-ordered blob array and arrive with one cp.async.bulk; the
// per-patch overhead (header, gather, epilogue, refill) is shared by P
// patches. Used for the element-triple patches of SV fine levels (m + np = 9).
template <int LPP, int NPM>
__global__ void __launch_bounds__(256) vanka_subwarp_kernel(
    int npatch, const unsigned char* __restrict__ blob, const long long* __restrict__ off,
    int slot_bytes, int nstage, int sb_len, const double* __restrict__ r,
    double* __restrict__ out, int seq, const int* gate) {
  if (gate && *gate) return;
  constexpr int P = 32 / LPP;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPP, gl = lane % LPP;
  const int nbar = (nstage + 1) & ~1;
  const size_t stage_bytes = (size_t)P * slot_bytes;
  unsigned char* ring = smem + (size_t)wib * nstage * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)warps * nstage * stage_bytes) +
                   (size_t)wib * nbar;
  double* sbuf = reinterpret_cast<double*>(smem + (size_t)warps * nstage * stage_bytes +
                                           (size_t)warps * nbar * 8) +
                 (size_t)wib * 2 * P * sb_len;
  const int ngroups = (npatch + P - 1) / P;
  const int first = blockIdx.x * warps + wib;
  const int stride = gridDim.x * warps;
  const uint64_t policy = evict_first_policy();
  auto grp_end = [&](int q) { return q * P + P < npatch ? q * P + P : npatch; };
  auto issue_at = [&](int s, long long o0, long long o1) {
    const unsigned bytes = (unsigned)(o1 - o0);
    mbar_expect_tx(bars + s, bytes);
    bulk_copy_hint(ring + (size_t)s * stage_bytes, blob + o0, bytes, bars + s, policy);
  };
  // this group's patch of group q in stage s (valid when q P + g < npatch)
  auto view_at = [&](int s, long long base, long long own) {
    return patch_view<true>(ring + (size_t)s * stage_bytes + (size_t)(own - base), true);
  };
  auto gather_to = [&](const PatchView& w, double* dst) {
    // (x_j, y_j) pairs over j < m, padding zeroed, pressure at 2m
    for (int i = gl; i < w.nv + w.np; i += LPP) {
      const int d = i < w.nx ? 2 * i : (i < w.nv ? 2 * (i - w.nx) + 1 : 2 * w.m + (i - w.nv));
      dst[d] = __ldg(r + w.idx[i]);
    }
    if (w.nx != w.ny)
      for (int j = gl; j < w.m; j += LPP) {
        if (j >= w.nx) dst[2 * j] = 0.0;
        if (j >= w.ny) dst[2 * j + 1] = 0.0;
      }
  };
  if (lane == 0) {
    for (int s = 0; s < nstage; ++s) mbar_init(bars + s, 1);
    mbar_init_fence();
    for (int s = 0; s < nstage; ++s) {
      const int q = first + s * stride;
      if (q < ngroups) issue_at(s, off[q * P], off[grp_end(q)]);
    }
  }
  __syncwarp();
  unsigned phase = 0;
  // offsets of the current group: stage base and this group's blob
  long long cb = 0, co = 0;
  if (first < ngroups) {
    cb = __ldg(off + first * P);
    co = __ldg(off + min(first * P + g, npatch));
    mbar_wait(bars, 0);
    phase ^= 1u;
    if (first * P + g < npatch) gather_to(view_at(0, cb, co), sbuf + g * sb_len);
  }
  __syncwarp();
  const int cs0 = gl * (gl + 1) / 2;
  int stage = 0, it = 0;
  for (int q = first; q < ngroups; q += stride, ++it) {
    const int qr = q + nstage * stride;
    long long ro0 = 0, ro1 = 0;
    if (lane == 0 && qr < ngroups) {
      ro0 = __ldg(off + qr * P);
      ro1 = __ldg(off + grp_end(qr));
    }
    const int qn = q + stride;
    long long nb = 0, no = 0;
    if (qn < ngroups) {
      nb = __ldg(off + qn * P);
      no = __ldg(off + min(qn * P + g, npatch));
    }
    const bool valid = q * P + g < npatch;
    const PatchView v = view_at(stage, cb, co);
    const double* sb = sbuf + ((it & 1) * P + g) * sb_len;
    const int sn = stage + 1 == nstage ? 0 : stage + 1;
    double gv[2];
    int gd[2];
    PatchView w{};
    bool wvalid = false;
    if (qn < ngroups) {
      mbar_wait(bars + sn, (phase >> sn) & 1u);
      phase ^= 1u << sn;
      wvalid = qn * P + g < npatch;
      if (wvalid) w = view_at(sn, nb, no);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = gl + LPP * u;
        const bool in = wvalid && i < w.nv + w.np;
        gd[u] = i < w.nx ? 2 * i : (i < w.nv ? 2 * (i - w.nx) + 1 : 2 * w.m + (i - w.nv));
        gv[u] = in ? __ldg(r + w.idx[i]) : 0.0;
      }
    }
    // the paired solve of vanka_patch_kernel within each group
    const int mm = valid ? v.m : 0, npp = valid ? (NPM == 1 ? 1 : v.np) : 0;
    int M = mm;
#pragma unroll
    for (int o = LPP; o < 32; o <<= 1) M = max(M, __shfl_xor_sync(0xffffffffu, M, o));
    const double2* AP = reinterpret_cast<const double2*>(v.Ax);
    const double2* SB = reinterpret_cast<const double2*>(sb);
    const int boff = valid ? (int)(reinterpret_cast<const double2*>(v.Bh) - AP) : 0;
    const bool act = gl < mm + npp;
    const int cl = gl >= mm ? boff + (gl - mm) * mm : cs0;
    double tx = 0.0, ty = 0.0;
    int csj = 0;
#pragma unroll 4
    for (int j = 0; j < M; csj += ++j) {
      const bool col = j < mm;
      const double2 b = lds_v2_pred(SB + j, col);
      const double2 a = lds_v2_pred(AP + (gl <= j ? csj + gl : cl + j), col && act);
      tx = fma(a.x, b.x, tx);
      ty = fma(a.y, b.y, ty);
    }
    double xl = tx + ty;
    const int ar = min(max(gl - mm, 0), max(npp - 1, 0));
    if (valid) {
#pragma unroll
      for (int e = 0; e < NPM; ++e)
        if (e < npp) xl = fma(v.Si[ar * npp + e], sb[2 * mm + e], xl);
      if (gl >= mm && gl < mm + npp) out[v.opos(seq, v.nv + ar)] = xl;
    }
    double xp[NPM];
#pragma unroll
    for (int e = 0; e < NPM; ++e)
      xp[e] = __shfl_sync(0xffffffffu, xl, g * LPP + min(mm + e, LPP - 1));
    if (valid && gl < mm) {
      const double2* UP = reinterpret_cast<const double2*>(v.U);
      double ox = tx, oy = ty;
#pragma unroll
      for (int e = 0; e < NPM; ++e)
        if (e < npp) {
          const double2 u = UP[e * mm + gl];
          ox = fma(u.x, xp[e], ox);
          oy = fma(u.y, xp[e], oy);
        }
      if (gl < v.nx) out[v.opos(seq, gl)] = ox;
      if (gl < v.ny) out[v.opos(seq, v.nx + gl)] = oy;
    }
    // publish the prefetched r of the next group
    if (wvalid) {
      double* sbn = sbuf + (((it + 1) & 1) * P + g) * sb_len;
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (gl + LPP * u < w.nv + w.np) sbn[gd[u]] = gv[u];
      if (w.nx != w.ny && gl < w.m) {
        if (gl >= w.nx) sbn[2 * gl] = 0.0;
        if (gl >= w.ny) sbn[2 * gl + 1] = 0.0;
      }
    }
    __syncwarp();
    if (lane == 0 && qr < ngroups) {
      fence_proxy_async();
      issue_at(stage, ro0, ro1);
    }
    stage = sn;
    cb = nb;
    co = no;
  }
}


// Fixed-shape paired patches: the SV fine level's element triples with
// m = max(nx, ny) = M velocity pair rows and NP = 3 pressure seeds (~90-97%
// of the level; nx, ny vary through exact cancellations in B). The paired
// layout zero-pads the smaller component to M, so the shape, the factor
// offsets and the loop bounds are compile-time constants; only the dof lists
// depend on (nx, ny). L = M + NP lanes per patch (M pair rows + NP pressure
// rows), 32 / L patches per warp, the group's blobs in one bulk copy. The
// blob carries no b_hat: x_p = S^-1 (b_p + U_hat^T b_u), with U_hat^T b_u a
// shuffle tree over the pair lanes -- 26% fewer bytes than the stored-b_hat
// classes, results within rounding of theirs (vanka.cpp:133-181 reassociated).
template <int M, int NP, int MINB>
__global__ void __launch_bounds__(256, MINB) vanka_fixed_kernel(
    int npatch, const unsigned char* __restrict__ blob, const long long* __restrict__ off,
    int slot_bytes, int nstage, const double* __restrict__ r, double* __restrict__ out,
    const int* gate) {
  if (gate && *gate) return;
  constexpr int L = M + NP, P = 32 / L, NV2 = 2 * M;
  // per-patch b stride: 16-byte aligned, and two doubles past a multiple of
  // 128 bytes so the patches of a group (which read the same entry of their own
  // b in one instruction) sit on different shared-memory banks: 111.7 -> 100.9 us
  // on the config-3 K0 sweep
  constexpr int NBS = (((2 * M + NP + 1) & ~1) + 15) / 16 * 16 + 2;
  constexpr int A2 = M * (M + 1) / 2;          // A pairs
  constexpr int W2 = M <= 2 ? 2 : M <= 4 ? 4 : M <= 8 ? 8 : 16;  // reduction width
  static_assert(W2 <= L, "the w_e tree must stay inside the patch's lanes");
  constexpr int FD = 2 * A2 + 2 * NP * M + NP * NP;  // A | U pairs | S^-1 (no b_hat)
  extern __shared__ __align__(128) unsigned char smem[];
  const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / L, gl = lane % L;
  const int gg = g < P ? g : 0;
  const int nbar = (nstage + 1) & ~1;
  const size_t stage_bytes = (size_t)P * slot_bytes;
  unsigned char* ring = smem + (size_t)wib * nstage * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)warps * nstage * stage_bytes) +
                   (size_t)wib * nbar;
  double* sbuf = reinterpret_cast<double*>(smem + (size_t)warps * nstage * stage_bytes +
                                           (size_t)warps * nbar * 8) +
                 (size_t)wib * 2 * P * NBS;
  const int ngroups = (npatch + P - 1) / P;
  const int first = blockIdx.x * warps + wib;
  const int stride = gridDim.x * warps;
  const uint64_t policy = evict_first_policy();
  auto grp_end = [&](int q) { return q * P + P < npatch ? q * P + P : npatch; };
  auto issue_bytes = [&](int s, long long o0, long long o1) {
    mbar_expect_tx(bars + s, (unsigned)(o1 - o0));
    bulk_copy_hint(ring + (size_t)s * stage_bytes, blob + o0, (unsigned)(o1 - o0), bars + s,
                   policy);
  };
  auto issue_at = [&](int s, int q) { issue_bytes(s, off[q * P], off[grp_end(q)]); };
  // this lane's patch in stage s: the group's blobs are contiguous and a
  // blob's size follows from its header (nx, ny), so the position is a walk
  // over the earlier headers in shared memory -- no offset-table load on the
  // critical path
  auto patch_at = [&](int s) {
    const unsigned char* B = ring + (size_t)s * stage_bytes;
#pragma unroll
    for (int h = 0; h < P - 1; ++h)
      if (h < gg) {
        const int2 hd = *reinterpret_cast<const int2*>(B);
        B += ((16 + 8 * FD + 8 * (hd.x + hd.y + NP)) + 15) & ~15;
      }
    return B;
  };
  // this lane's r values: velocity lanes (x_gl, y_gl) zero past nx / ny,
  // pressure lanes p_(gl - M)
  auto load_r = [&](const unsigned char* B, bool valid, double& v0, double& v1) {
    v0 = v1 = 0.0;
    if (!valid) return;
    const int2 hdr = *reinterpret_cast<const int2*>(B);
    const int* idx = reinterpret_cast<const int*>(B + 16 + 8 * FD);
    if (gl < M) {
      if (gl < hdr.x) v0 = __ldg(r + idx[gl]);
      if (gl < hdr.y) v1 = __ldg(r + idx[hdr.x + gl]);
    } else {
      v0 = __ldg(r + idx[hdr.x + hdr.y + gl - M]);
    }
  };
  auto store_r = [&](double* sb, double v0, double v1) {
    if (gl < M)
      reinterpret_cast<double2*>(sb)[gl] = make_double2(v0, v1);
    else
      sb[NV2 + gl - M] = v0;
  };
  if (lane == 0) {
    for (int s = 0; s < nstage; ++s) mbar_init(bars + s, 1);
    mbar_init_fence();
    for (int s = 0; s < nstage; ++s) {
      const int q = first + s * stride;
      if (q < ngroups) issue_at(s, q);
    }
  }
  __syncwarp();
  unsigned phase = 0;
  if (first < ngroups) {
    mbar_wait(bars, 0);
    phase ^= 1u;
    const bool valid = g < P && first * P + g < npatch;
    double v0, v1;
    load_r(patch_at(0), valid, v0, v1);
    if (valid) store_r(sbuf + g * NBS, v0, v1);
  }
  __syncwarp();
  // per-lane pair offsets of the column loop (compile-time j): velocity row
  // gl reads A(gl, j) -- column j's entry gl when gl <= j, else column gl's
  // entry j -- b_hat row a = gl - M reads its pair j (b_hat pairs follow U)
  const int a_row = gl - M;
  const int own_col = gl < M ? gl * (gl + 1) / 2 : 0;
  int stage = 0, it = 0;
  for (int q = first; q < ngroups; q += stride, ++it) {
    const int qr = q + nstage * stride;
    const int qn = q + stride;
    // offsets of the group that refills this stage, loaded now so the
    // refill at the end of the iteration does not wait on them
    long long ro0 = 0, ro1 = 0;
    if (lane == 0 && qr < ngroups) {
      ro0 = __ldg(off + qr * P);
      ro1 = __ldg(off + grp_end(qr));
    }
    const bool valid = g < P && q * P + g < npatch;
    const unsigned char* B = patch_at(stage);
    const int2 hdr = *reinterpret_cast<const int2*>(B);
    const double2* AP = reinterpret_cast<const double2*>(B + 16);
    const double* U = reinterpret_cast<const double*>(B + 16) + 2 * A2;
    const double* Si = U + 2 * NP * M;
    const int* pos = reinterpret_cast<const int*>(Si + NP * NP) + hdr.x + hdr.y + NP;
    const double* sb = sbuf + ((it & 1) * P + gg) * NBS;
    const int sn = stage + 1 == nstage ? 0 : stage + 1;
    // the next group's r, requested before this group's solve
    double nv0 = 0.0, nv1 = 0.0;
    bool nvalid = false;
    if (qn < ngroups) {
      mbar_wait(bars + sn, (phase >> sn) & 1u);
      phase ^= 1u << sn;
      nvalid = g < P && qn * P + g < npatch;
      load_r(patch_at(sn), nvalid, nv0, nv1);
    }
    const double2* SB = reinterpret_cast<const double2*>(sb);
    const double2* UP = reinterpret_cast<const double2*>(U);
    // pair lanes: t = A_c^-1 b_u (both components at once) and the pair's
    // part of w_e = sum_j u_hat(j, e) . b_u(j)
    double tx = 0.0, ty = 0.0;
    double2 uu[NP];
    double wp[NP];
    if (gl < M) {
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const double2 b = SB[j];
        const double2 a = AP[gl <= j ? j * (j + 1) / 2 + gl : own_col + j];
        tx = fma(a.x, b.x, tx);
        ty = fma(a.y, b.y, ty);
      }
      const double2 bo = SB[gl];
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        uu[e] = UP[e * M + gl];
        wp[e] = fma(uu[e].y, bo.y, uu[e].x * bo.x);
      }
    } else {
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        uu[e] = make_double2(0.0, 0.0);
        wp[e] = 0.0;
      }
    }
    // w_e: a fixed tree over the group's first W2 lanes (pair lanes; the
    // pressure lanes in it hold 0), broadcast from the group's lane 0
    double w[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      double v = wp[e];
#pragma unroll
      for (int o = W2 / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      w[e] = __shfl_sync(0xffffffffu, v, gg * L);
    }
    // pressure lane a: x_p(a) = sum_e S^-1(a, e) (b_p(e) + w_e)
    // (= S^-1 b_p + b_hat b_u with b_hat = S^-1 U_hat^T, vanka.cpp:133-140,
    // reassociated so b_hat is neither stored nor formed)
    double xl = 0.0;
    const int ar = gl < M ? 0 : a_row;
#pragma unroll
    for (int e = 0; e < NP; ++e) xl = fma(Si[ar * NP + e], sb[NV2 + e] + w[e], xl);
    if (valid && gl >= M) out[pos[hdr.x + hdr.y + a_row]] = xl;
    double xp[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) xp[e] = __shfl_sync(0xffffffffu, xl, gg * L + M + e);
    if (valid && gl < M) {
      double ox = tx, oy = ty;
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        ox = fma(uu[e].x, xp[e], ox);
        oy = fma(uu[e].y, xp[e], oy);
      }
      if (gl < hdr.x) out[pos[gl]] = ox;
      if (gl < hdr.y) out[pos[hdr.x + gl]] = oy;
    }
    if (nvalid) store_r(sbuf + (((it + 1) & 1) * P + g) * NBS, nv0, nv1);
    __syncwarp();
    if (lane == 0 && qr < ngroups) {
      fence_proxy_async();
      issue_bytes(stage, ro0, ro1);
    }
    stage = sn;
  }
}

// Owner-computes scatter-add: delta_d = sum over d's slots (ascending patch
// order) of w_d * x_slot (vanka.cpp:179-181); with xadd: x_d += omega*delta_d
// (vanka.cpp:195).
// w == nullptr: w_d = 1 / multiplicity computed here -- the same IEEE
// division as weights_kernel (vanka.cpp:67-73), one HBM stream fewer;
// stored weights only after sag_vanka_set_weights (global partition of unity).
__global__ void vanka_gather_kernel(int n, const int* __restrict__ dof_ptr,
                                    const int* __restrict__ dof_slot,
                                    const double* __restrict__ out, const double* __restrict__ w,
                                    double* __restrict__ delta, double* __restrict__ xadd,
                                    double omega, const int* gate) {
  if (gate && *gate) return;
  constexpr int U = 8;  // multiplicities up to U in one pass (K0/ISO0: <= 7)
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const double xo = xadd ? xadd[d] : 0.0;
    const int s0 = __ldg(dof_ptr + d), s1 = __ldg(dof_ptr + d + 1);
    const double wd = w ? __ldg(w + d) : (s1 > s0 ? 1.0 / (double)(s1 - s0) : 0.0);
    double acc = 0.0;
    for (int sb = s0; sb < s1; sb += U) {
      // all slot ids, then all values, then the ordered sum: two dependent
      // round trips per pass instead of two per slot
      int sl[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) sl[u] = sb + u < s1 ? __ldcs(dof_slot + sb + u) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = sb + u < s1 ? __ldcg(out + sl[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (sb + u < s1) acc = __dadd_rn(acc, __dmul_rn(wd, v[u]));
    }
    if (xadd)
      xadd[d] = xo + omega * acc;
    else
      delta[d] = acc;
  }
}

// The gather of dof-ordered results (Vanka::seq): d's contributions are the
// contiguous run out[dof_ptr[d] .. dof_ptr[d+1]) (ascending patch order), so
// neighbouring threads read neighbouring runs -- a coalesced stream with no
// slot-id indirection. Same arithmetic as vanka_gather_kernel.
__global__ void vanka_gather_seq_kernel(int n, const int* __restrict__ dof_ptr,
                                        const double* __restrict__ out,
                                        const double* __restrict__ w, double* __restrict__ delta,
                                        double* __restrict__ xadd, double omega, const int* gate) {
  if (gate && *gate) return;
  constexpr int U = 8;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const double xo = xadd ? xadd[d] : 0.0;
    const int s0 = __ldg(dof_ptr + d), s1 = __ldg(dof_ptr + d + 1);
    const double wd = w ? __ldg(w + d) : (s1 > s0 ? 1.0 / (double)(s1 - s0) : 0.0);
    double acc = 0.0;
    for (int sb = s0; sb < s1; sb += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = sb + u < s1 ? __ldcs(out + sb + u) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (sb + u < s1) acc = __dadd_rn(acc, __dmul_rn(wd, v[u]));
    }
    if (xadd)
      xadd[d] = xo + omega * acc;
    else
      delta[d] = acc;
  }
}

// The gather of the boundary patches of a partitioned sweep fused with the
// reverse halo: x_d += omega * delta_d as vanka_gather_seq_kernel, and where
// d is a ghost dof its value -- this rank's complete partial sum at d -- is
// also stored into the owner's receive buffer (peer[nbr[d]][slot[d]], mapped
// by CUDA IPC: NVLink stores), ended by a system-scope fence.
struct PeerMap {
  double* peer[8];
};
__global__ void vanka_gather_push_kernel(int n, const int* __restrict__ dof_ptr,
                                         const double* __restrict__ out,
                                         const double* __restrict__ w, double* __restrict__ x,
                                         double omega, const int* __restrict__ slot,
                                         const unsigned char* __restrict__ nbr, PeerMap pm) {
  constexpr int U = 8;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const double xo = x[d];
    const int s0 = __ldg(dof_ptr + d), s1 = __ldg(dof_ptr + d + 1);
    const double wd = w ? __ldg(w + d) : (s1 > s0 ? 1.0 / (double)(s1 - s0) : 0.0);
    double acc = 0.0;
    for (int sb = s0; sb < s1; sb += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = sb + u < s1 ? __ldcs(out + sb + u) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (sb + u < s1) acc = __dadd_rn(acc, __dmul_rn(wd, v[u]));
    }
    const double val = xo + omega * acc;
    x[d] = val;
    const int sl = __ldg(slot + d);
    if (sl >= 0) pm.peer[__ldg(nbr + d)][sl] = val;
  }
  __threadfence_system();
}

static void launch_gather(Ctx& c, const Vanka& f, double* delta, double* xadd, double omega,
                          const int* gate) {
  const double* w = f.w_ext ? f.w.p : nullptr;
  if (f.seq)
    vanka_gather_seq_kernel<<<grid_for(c, f.n), 256, 0, c.stream>>>(f.n, f.dof_ptr.p, f.out.p, w,
                                                                    delta, xadd, omega, gate);
  else
    vanka_gather_kernel<<<grid_for(c, f.n), 256, 0, c.stream>>>(
        f.n, f.dof_ptr.p, f.dof_slot.p, f.out.p, w, delta, xadd, omega, gate);
  SAG_LAUNCHED(c);
}

struct ApplyCfg {
  int warps, nstage, sb_len, smem, blocks;
};

// Launch shape: NSTAGE >= 3 blobs in flight per warp (one being solved, one
// gathered, >= 1 landing), as many warps as shared memory allows (up to 8
// per CTA, several CTAs per SM), a persistent grid of occupancy x #SMs.
template <int R, bool SYM, int NPM>
static ApplyCfg apply_cfg(Ctx& c, const Vanka& f, int npatch, int slot_bytes) {
  static thread_local int configured_smem[2][4][2] = {};
  int& configured = configured_smem[SYM][R - 1][NPM == 1 ? 0 : 1];
  ApplyCfg a;
  // 2 stages: the gather of the next patch waits for its blob, but the smaller
  // per-warp footprint fits more warps per SM -- measured 247 us vs 276 us
  // (3 stages) for the config-2 K0 sweep
  a.nstage = std::max(2, env_int("SAG_VANKA_STAGES", 2));
  a.sb_len = f.max_nv + f.max_np + f.max_dim + 2;
  a.sb_len = (a.sb_len + 1) / 2 * 2;
  const int per_warp = a.nstage * slot_bytes + ((a.nstage + 1) & ~1) * 8 + 2 * a.sb_len * 8;
  const int cta_budget = env_int("SAG_VANKA_CTA_SMEM", 60000);
  a.warps = std::max(1, std::min(env_int("SAG_VANKA_WARPS", 8), cta_budget / per_warp));
  if (a.warps * per_warp > 220 * 1024) a.warps = std::max(1, (220 * 1024) / per_warp);
  a.smem = a.warps * per_warp;
  SAG_REQUIRE(a.smem <= 227 * 1024, SAG_ERROR, "apply_vanka: patch blobs too large for staging");
  auto kern = vanka_patch_kernel<R, SYM, NPM>;
  if (configured < a.smem) {
    SAG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem));
    configured = a.smem;
  }
  int occ = 0;
  SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, a.warps * 32, a.smem));
  occ = std::max(occ, 1);
  const long long need = (npatch + a.warps - 1) / a.warps;
  a.blocks = (int)std::max(1LL, std::min<long long>(need, (long long)occ * c.num_sms));
  return a;
}

template <int LPP, int NPM>
static void launch_subwarp(Ctx& c, const Vanka& f, const Vanka::RClass& cl, const double* r,
                           const int* gate) {
  static thread_local int configured = 0;
  constexpr int P = 32 / LPP;
  const int npatch = cl.k1 - cl.k0;
  const int nstage = std::max(2, env_int("SAG_VANKA_STAGES", 2));
  int sb_len = f.max_nv + f.max_np + f.max_dim + 2;
  sb_len = (sb_len + 1) / 2 * 2;
  const int per_warp = nstage * P * (int)cl.slot_bytes + ((nstage + 1) & ~1) * 8 + 2 * P * sb_len * 8;
  const int cta_budget = env_int("SAG_VANKA_CTA_SMEM", 60000);
  int warps = std::max(1, std::min(env_int("SAG_VANKA_WARPS", 8), cta_budget / per_warp));
  if (warps * per_warp > 220 * 1024) warps = std::max(1, (220 * 1024) / per_warp);
  const int smem = warps * per_warp;
  SAG_REQUIRE(smem <= 227 * 1024, SAG_ERROR, "apply_vanka: patch blobs too large for staging");
  auto kern = vanka_subwarp_kernel<LPP, NPM>;
  if (configured < smem) {
    SAG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = smem;
  }
  int occ = 0;
  SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem));
  occ = std::max(occ, 1);
  const long long ngroups = (npatch + P - 1) / P;
  const int blocks = (int)std::max(1LL, std::min<long long>((ngroups + warps - 1) / warps,
                                                          (long long)occ * c.num_sms));
  kern<<<blocks, warps * 32, smem, c.stream>>>(npatch, f.blob.p, f.off.p + cl.k0,
                                                (int)cl.slot_bytes, nstage, sb_len, r, f.out.p,
                                                f.seq ? 1 : 0, gate);
  SAG_LAUNCHED(c);
}

template <int M, int NP>
static void launch_fixed(Ctx& c, const Vanka& f, const Vanka::RClass& cl, const double* r,
                         const int* gate) {
  static thread_local int configured[2] = {0, 0};
  constexpr int L = M + NP, P = 32 / L, NB = ((((2 * M + NP) + 1) & ~1) + 15) / 16 * 16 + 2;
  const int npatch = cl.k1 - cl.k0;
  const int bytes = (int)cl.slot_bytes;  // the largest blob of the class
  const int nstage = std::max(2, env_int("SAG_VANKA_STAGES", 2));
  const int per_warp = nstage * P * bytes + ((nstage + 1) & ~1) * 8 + 2 * P * NB * 8;
  const int cta_budget = env_int("SAG_VANKA_CTA_SMEM", 60000);
  int warps = std::max(1, std::min(env_int("SAG_VANKA_WARPS", 8), cta_budget / per_warp));
  const int smem = warps * per_warp;
  const int v5 = env_int("SAG_VANKA_MINB", 4) == 5;
  auto kern = v5 ? vanka_fixed_kernel<M, NP, 5> : vanka_fixed_kernel<M, NP, 4>;
  if (configured[v5] < smem) {
    SAG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[v5] = smem;
  }
  int occ = 0;
  SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem));
  occ = std::max(occ, 1);
  const long long ngroups = (npatch + P - 1) / P;
  const int blocks = (int)std::max(1LL, std::min<long long>((ngroups + warps - 1) / warps,
                                                          (long long)occ * c.num_sms));
  SAG_REQUIRE(f.seq, SAG_ERROR, "apply_vanka: the fixed-shape kernel needs dof-ordered results");
  kern<<<blocks, warps * 32, smem, c.stream>>>(npatch, f.blob.p, f.off.p + cl.k0, bytes, nstage,
                                                r, f.out.p, gate);
  SAG_LAUNCHED(c);
}

// One size class: patches [k0, k1) of the blob order (contiguous blobs).
template <int R, bool SYM, int NPM>
static void launch_patch(Ctx& c, const Vanka& f, const Vanka::RClass& cl, const double* r,
                         const int* gate) {
  SAG_REQUIRE(!f.pairs || (R <= 2 && SYM), SAG_ERROR,
              "apply_vanka: paired factor blobs need a symmetric R <= 2 kernel");
  const int npatch = cl.k1 - cl.k0;
  const ApplyCfg a = apply_cfg<R, SYM, NPM>(c, f, npatch, (int)cl.slot_bytes);
  vanka_patch_kernel<R, SYM, NPM><<<a.blocks, a.warps * 32, a.smem, c.stream>>>(
      npatch, f.blob.p, f.off.p + cl.k0, (int)cl.slot_bytes, a.nstage, a.sb_len,
      f.pairs ? 1 : 0, r, f.out.p, f.seq ? 1 : 0, gate);
  SAG_LAUNCHED(c);
}

template <bool SYM, int NPM>
static void launch_patch_r(Ctx& c, const Vanka& f, const double* r, const int* gate,
                           const std::vector<Vanka::RClass>* classes) {
  // one launch per size class (rows per lane: matrix rows, or on paired
  // levels matrix + b_hat rows); `classes` may narrow them to windows
  for (const auto& cl : classes ? *classes : f.rclasses) {
    if (cl.k1 <= cl.k0) continue;
    SAG_REQUIRE(cl.R <= 4, SAG_ERROR, "apply_vanka: patch with more than 128 rows");
    if (cl.fm) {
      if constexpr (SYM && NPM == 4) {
        if (cl.fm == 6 && cl.fnp == 3) {
          launch_fixed<6, 3>(c, f, cl, r, gate);
          continue;
        }
      }
      SAG_REQUIRE(false, SAG_ERROR, "apply_vanka: unsupported fixed patch shape");
    }
    if (cl.lpp < 32) {
      if constexpr (SYM) {
        if (cl.lpp == 8)
          launch_subwarp<8, NPM>(c, f, cl, r, gate);
        else
          launch_subwarp<16, NPM>(c, f, cl, r, gate);
        continue;
      }
    }
    switch (cl.R) {
      case 1: launch_patch<1, SYM, NPM>(c, f, cl, r, gate); break;
      case 2: launch_patch<2, SYM, NPM>(c, f, cl, r, gate); break;
      case 3: launch_patch<3, SYM, NPM>(c, f, cl, r, gate); break;
      default: launch_patch<4, SYM, NPM>(c, f, cl, r, gate); break;
    }
  }
}

static void launch_patch_any(Ctx& c, const Vanka& f, const double* r, const int* gate,
                             const std::vector<Vanka::RClass>* classes = nullptr) {
  if (f.npatch == 0) return;
  const bool np1 = f.max_np <= 1;  // TH / ISO levels: one pressure seed
  if (f.sym && np1)
    launch_patch_r<true, 1>(c, f, r, gate, classes);
  else if (f.sym)
    launch_patch_r<true, 4>(c, f, r, gate, classes);
  else if (np1)
    launch_patch_r<false, 1>(c, f, r, gate, classes);
  else
    launch_patch_r<false, 4>(c, f, r, gate, classes);
}

void vanka_apply(Ctx& c, const Vanka& f, const double* r, double* delta, const int* gate) {
  launch_patch_any(c, f, r, gate);
  launch_gather(c, f, delta, nullptr, 1.0, gate);
}

void vanka_apply_stage(Ctx& c, const Vanka& f, const double* r, double* delta, int stage) {
  if (stage == 1) {
    launch_patch_any(c, f, r, nullptr);
  } else {
    launch_gather(c, f, delta, nullptr, 1.0, nullptr);
  }
}

void vanka_gather_range(Ctx& c, const Vanka& f, int d0, int d1, double* delta) {
  if (d1 <= d0) return;
  const double* w = f.w_ext ? f.w.p + d0 : nullptr;
  if (f.seq)
    vanka_gather_seq_kernel<<<grid_for(c, d1 - d0), 256, 0, c.stream>>>(
        d1 - d0, f.dof_ptr.p + d0, f.out.p, w, delta + d0, nullptr, 1.0, nullptr);
  else
    vanka_gather_kernel<<<grid_for(c, d1 - d0), 256, 0, c.stream>>>(
        d1 - d0, f.dof_ptr.p + d0, f.dof_slot.p, f.out.p, w, delta + d0, nullptr, 1.0, nullptr);
  SAG_LAUNCHED(c);
}

__global__ void vanka_gather_ranges_kernel(RowRanges R, const int* __restrict__ dof_ptr,
                                           const double* __restrict__ out,
                                           const double* __restrict__ w, double* __restrict__ delta);

// ============================== pipelined host-buffer step (sag_vanka_spmv) ==
// With pinned host buffers the step is bound by the host link: x in (8 n
// bytes), delta and y out (16 n bytes). The two directions are independent
// DMA engines, so x arrives in S stages and every output range leaves as soon
// as the inputs it depends on have arrived: the device->host stream runs
// under the rest of the host->device stream instead of after it.
//
// The plan is derived from the operator and the patches alone, correct for
// any numbering: every input dof gets an arrival stage (the mesh strip of the
// lowest pressure dof it couples to; pressure dofs by index), grouped into
// contiguous ranges by taking the latest stage over blocks of 1024 dofs;
// from the arrival stages: a row of K is ready when all its columns arrived,
// a patch when all its dofs arrived, a dof of delta when all its patches ran;
// each again rounded up to the latest stage over a block, which yields a few
// contiguous ranges per stage for a strip-ordered numbering and degenerates to
// "everything in the last stage" (the unpipelined step) for a hostile one.

struct StepRange {
  int a, b;
};
struct StepPlan {
  const Matrix* k = nullptr;
  unsigned long long k_uid = 0;
  int S = 0, want_S = 0, growth = 0;
  int choice = 0;                 // 0 untimed, 1 pipelined, -1 plain (sag_vanka_spmv)
  double t_plain = 0.0, t_pipe = 0.0;  // seconds per step measured at the first call
  std::vector<std::vector<StepRange>> in, rows, gat;  // per stage
  std::vector<std::vector<Vanka::RClass>> pat;         // per stage: class windows
  std::vector<cudaEvent_t> ev;                         // 3 S events
  std::vector<std::vector<RowRanges>> rows_rr, gat_rr;  // the same ranges, <= 12 per launch
  cudaStream_t sin = nullptr, sout = nullptr, ssp = nullptr;
  long long ranges = 0;
  // the whole step captured once per buffer set (the CPU cannot enqueue
  // ~20 operations per stage as fast as the device retires them)
  cudaGraphExec_t exec = nullptr;
  long long graph_launches = 0;
  DevBuf<unsigned long long> ktrace;  // SAG_STEP_TRACE=2: [3 S][start, end] of the copy kernels
  const void* gkey[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ~StepPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (sin) cudaStreamDestroy(sin);
    if (sout) cudaStreamDestroy(sout);
    if (ssp) cudaStreamDestroy(ssp);
  }
};

__global__ void step_minp_kernel(int n_u, const int* __restrict__ rp, const int* __restrict__ ci,
                                 int* __restrict__ minp) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_u; r += gridDim.x * blockDim.x) {
    int m = 0x7fffffff;
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int c = ci[k];
      if (c >= n_u) m = min(m, c);
    }
    minp[r] = m;
  }
}
__global__ void step_rowq_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                 const int* __restrict__ arr, int* __restrict__ q) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int m = 0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) m = max(m, arr[ci[k]]);
    q[r] = m;
  }
}
// patch of slot t: slots are numbered patch by patch (sbase = prefix sums)
__device__ __forceinline__ int step_slot_patch(const int* __restrict__ sbase, int np, int t) {
  int lo = 0, hi = np;  // largest i with sbase[i] <= t
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sbase[mid] <= t) lo = mid;
    else hi = mid;
  }
  return lo;
}
__global__ void step_patchq_kernel(int n, const int* __restrict__ dof_ptr,
                                   const int* __restrict__ dof_slot, const int* __restrict__ sbase,
                                   int np, const int* __restrict__ arr, int* qp) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x)
    for (int s = dof_ptr[d]; s < dof_ptr[d + 1]; ++s)
      atomicMax(qp + step_slot_patch(sbase, np, dof_slot[s]), arr[d]);
}
__global__ void step_dofq_kernel(int n, const int* __restrict__ dof_ptr,
                                 const int* __restrict__ dof_slot, const int* __restrict__ sbase,
                                 int np, const int* __restrict__ pd, int* __restrict__ og) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    int m = 0;
    for (int s = dof_ptr[d]; s < dof_ptr[d + 1]; ++s)
      m = max(m, pd[step_slot_patch(sbase, np, dof_slot[s])]);
    og[d] = m;
  }
}

// req[i] -> assigned stage >= req[i], constant over blocks of W (the block's
// latest stage); appends the runs to out[stage] shifted by `base`
static void step_runs(const int* req, int m, int W, int S, int base,
                      std::vector<std::vector<StepRange>>& out, std::vector<int>* assigned,
                      long long& nruns) {
  int run_a = 0, run_s = -1;
  for (int b0 = 0; b0 < m; b0 += W) {
    const int b1 = std::min(m, b0 + W);
    int s = 0;
    for (int i = b0; i < b1; ++i) s = std::max(s, req[i]);
    s = std::min(std::max(s, 0), S - 1);
    if (assigned)
      for (int i = b0; i < b1; ++i) (*assigned)[i] = s;
    if (s != run_s) {
      if (run_s >= 0) {
        out[run_s].push_back({base + run_a, base + b0});
        ++nruns;
      }
      run_a = b0;
      run_s = s;
    }
  }
  if (run_s >= 0 && m > 0) {
    out[run_s].push_back({base + run_a, base + m});
    ++nruns;
  }
}

// SM-driven copies over the host link: one launch moves all ranges of a
// stage between pinned (mapped) host memory and device memory. The DMA
// engines cost ~7-16 us per range on top of the bytes (tools/smcopy_probe.cu),
// a stage has ~5 ranges per vector; a few CTAs reach the same link bandwidth.
constexpr int kStepMaxRanges = 12;
struct CopyRanges {
  int n = 0;
  int a[kStepMaxRanges], b[kStepMaxRanges];
};
__global__ void __launch_bounds__(512) step_copy_kernel(const double* __restrict__ src,
                                                        double* __restrict__ dst, CopyRanges R,
                                                        unsigned long long* tr) {
  if (tr && threadIdx.x == 0) {  // diagnostic: first start / last end of the launch
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(tr, t);
  }
  const int st = gridDim.x * blockDim.x;
  for (int q = 0; q < R.n; ++q) {
    const int b = R.b[q];
    int i = R.a[q] + blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * st < b; i += 4 * st) {
      const double v0 = src[i], v1 = src[i + st], v2 = src[i + 2 * st], v3 = src[i + 3 * st];
      dst[i] = v0;
      dst[i + st] = v1;
      dst[i + 2 * st] = v2;
      dst[i + 3 * st] = v3;
    }
    for (; i < b; i += st) dst[i] = src[i];
  }
  if (tr) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(tr + 1, t);
    }
  }
}
static void step_copy(Ctx& c, cudaStream_t st, const double* src, double* dst,
                      const std::vector<StepRange>& rs, int ctas, unsigned long long* tr = nullptr) {
  for (size_t q0 = 0; q0 < rs.size(); q0 += kStepMaxRanges) {
    CopyRanges R;
    for (size_t q = q0; q < rs.size() && R.n < kStepMaxRanges; ++q) {
      R.a[R.n] = rs[q].a;
      R.b[R.n] = rs[q].b;
      ++R.n;
    }
    step_copy_kernel<<<ctas, 512, 0, st>>>(src, dst, R, tr);
    SAG_CUDA(cudaGetLastError());
    ++c.launches;
  }
}
// device-visible address of pinned host memory (null: not mapped)
static double* host_mapped(const double* p) {
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, const_cast<double*>(p), 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<double*>(d);
}

static std::shared_ptr<StepPlan> step_plan_build(Ctx& c, const Vanka& f, const Matrix& K, int S) {
  auto P = std::make_shared<StepPlan>();
  P->k = &K;
  P->k_uid = K.uid;
  P->S = S;
  P->want_S = S;
  P->growth = env_int("SAG_STEP_GROWTH", 100);
  const int n = f.n, n_u = std::min(std::max(f.n_u, 0), n), n_p = n - n_u, np_ = f.npatch;
  P->in.assign(S, {});
  P->rows.assign(S, {});
  P->gat.assign(S, {});
  P->pat.assign(S, {});
  const int W = 1024;
  // arrival stage of every dof
  std::vector<int> h(n, 0), arr(n, 0);
  {
    DevBuf<int> minp(std::max(n_u, 1));
    if (n_u > 0) {
      step_minp_kernel<<<grid_for(c, n_u), 256, 0, c.stream>>>(n_u, K.rp.p, K.ci.p, minp.p);
      SAG_LAUNCHED(c);
      SAG_CUDA(cudaMemcpyAsync(h.data(), minp.p, sizeof(int) * n_u, cudaMemcpyDeviceToHost, c.stream));
      SAG_CUDA(cudaStreamSynchronize(c.stream));
    }
    // stage q takes the pressure dofs up to the fraction cum[q]; SAG_STEP_GROWTH
    // (percent, default 100 = equal stages) makes each stage that much larger
    // than the one before, so the first outputs leave early
    const double g = std::max(1.0, env_int("SAG_STEP_GROWTH", 100) / 100.0);
    std::vector<double> cum(S);
    {
      double tot = 0.0, w = 1.0;
      for (int q = 0; q < S; ++q, w *= g) tot += w;
      double acc = 0.0;
      w = 1.0;
      for (int q = 0; q < S; ++q, w *= g) {
        acc += w;
        cum[q] = acc / tot;
      }
    }
    auto pstage = [&](int col) {
      if (n_p <= 0) return 0;
      const double fr = (double)(col - n_u) / n_p;
      int q = 0;
      while (q < S - 1 && fr >= cum[q]) ++q;
      return q;
    };
    for (int d = 0; d < n_u; ++d) h[d] = h[d] == 0x7fffffff ? 0 : pstage(h[d]);
    for (int d = n_u; d < n; ++d) h[d] = pstage(d);
  }
  // the velocity and pressure blocks are grouped separately (a block of 1024
  // never straddles them)
  step_runs(h.data(), n_u, W, S, 0, P->in, &arr, P->ranges);
  {
    std::vector<int> ap(n_p, 0);
    step_runs(h.data() + n_u, n_p, W, S, n_u, P->in, &ap, P->ranges);
    std::copy(ap.begin(), ap.end(), arr.begin() + n_u);
  }
  DevBuf<int> darr(std::max(n, 1)), dq(std::max(n, 1));
  SAG_CUDA(cudaMemcpyAsync(darr.p, arr.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c.stream));
  // rows of y
  step_rowq_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(n, K.rp.p, K.ci.p, darr.p, dq.p);
  SAG_LAUNCHED(c);
  SAG_CUDA(cudaMemcpyAsync(h.data(), dq.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  step_runs(h.data(), n_u, W, S, 0, P->rows, nullptr, P->ranges);
  step_runs(h.data() + n_u, n_p, W, S, n_u, P->rows, nullptr, P->ranges);
  // patches (blob order, class by class)
  std::vector<int> sbase(np_ + 1, 0);
  for (int i = 0; i < np_; ++i) sbase[i + 1] = sbase[i] + f.h_nv[i] + f.h_np[i];
  DevBuf<int> dsb(np_ + 1), dqp(std::max(np_, 1));
  SAG_CUDA(cudaMemcpyAsync(dsb.p, sbase.data(), sizeof(int) * (np_ + 1), cudaMemcpyHostToDevice,
                           c.stream));
  SAG_CUDA(cudaMemsetAsync(dqp.p, 0, sizeof(int) * std::max(np_, 1), c.stream));
  std::vector<int> qp(std::max(np_, 1), 0), pd(std::max(np_, 1), 0);
  if (np_ > 0) {
    step_patchq_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(n, f.dof_ptr.p, f.dof_slot.p, dsb.p,
                                                             np_, darr.p, dqp.p);
    SAG_LAUNCHED(c);
    SAG_CUDA(cudaMemcpyAsync(qp.data(), dqp.p, sizeof(int) * np_, cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    SAG_REQUIRE((int)f.h_order.size() == np_, SAG_ERROR, "step plan: blob order missing");
    for (const auto& cl : f.rclasses) {
      const int m = cl.k1 - cl.k0;
      if (m <= 0) continue;
      std::vector<int> req(m), as(m);
      for (int q = 0; q < m; ++q) req[q] = qp[f.h_order[cl.k0 + q]];
      std::vector<std::vector<StepRange>> win(S);
      step_runs(req.data(), m, 1536, S, cl.k0, win, &as, P->ranges);  // 1536: a multiple of every patches-per-warp count
      for (int q = 0; q < m; ++q) pd[f.h_order[cl.k0 + q]] = as[q];
      for (int st = 0; st < S; ++st)
        for (const auto& r : win[st]) {
          Vanka::RClass w = cl;
          w.k0 = r.a;
          w.k1 = r.b;
          P->pat[st].push_back(w);
        }
    }
    // dofs of delta
    SAG_CUDA(cudaMemcpyAsync(dqp.p, pd.data(), sizeof(int) * np_, cudaMemcpyHostToDevice, c.stream));
    step_dofq_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(n, f.dof_ptr.p, f.dof_slot.p, dsb.p, np_,
                                                           dqp.p, dq.p);
    SAG_LAUNCHED(c);
    SAG_CUDA(cudaMemcpyAsync(h.data(), dq.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  } else {
    std::fill(h.begin(), h.end(), 0);
  }
  step_runs(h.data(), n_u, W, S, 0, P->gat, nullptr, P->ranges);
  step_runs(h.data() + n_u, n_p, W, S, n_u, P->gat, nullptr, P->ranges);
  // a fragmented numbering (many ranges) gains nothing from the pipeline
  if (P->ranges > 64LL * S) {
    P->S = 0;
    return P;
  }
  // copy kernels go first when the block scheduler has a choice
  int plo = 0, phi = 0;
  SAG_CUDA(cudaDeviceGetStreamPriorityRange(&plo, &phi));
  SAG_CUDA(cudaStreamCreateWithPriority(&P->sin, cudaStreamNonBlocking, phi));
  SAG_CUDA(cudaStreamCreateWithPriority(&P->sout, cudaStreamNonBlocking, phi));
  SAG_CUDA(cudaStreamCreateWithFlags(&P->ssp, cudaStreamNonBlocking));
  auto pack = [&](const std::vector<std::vector<StepRange>>& src,
                  std::vector<std::vector<RowRanges>>& dst) {
    dst.assign(S, {});
    for (int q = 0; q < S; ++q) {
      RowRanges R;
      for (const auto& r : src[q]) {
        if (!R.push(r.a, r.b)) {
          dst[q].push_back(R);
          R = RowRanges();
          R.push(r.a, r.b);
        }
      }
      if (R.n) dst[q].push_back(R);
    }
  };
  pack(P->rows, P->rows_rr);
  pack(P->gat, P->gat_rr);
  P->ev.assign(4 * (size_t)S + 4, nullptr);
  for (auto& e : P->ev) SAG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return P;
}

static bool is_pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// the plan of the pipelined step for these buffers; null when it does not
// apply (pageable or device buffers, one stage, a fragmented numbering).
// choice: 0 = not yet timed against the plain step, 1 = pipelined, -1 = plain
// (an explicit SAG_STEP_STAGES forces the pipeline whatever the choice).
static StepPlan* vanka_step_prepare(Ctx& c, const Vanka& f, const Matrix& K, const double* x,
                                    double* delta, double* y) {
  const int S = env_int("SAG_STEP_STAGES", 8);
  if (S < 2 || S > 64 || f.n == 0 || !f.seq) return nullptr;
  if (!is_pinned_host(x) || !is_pinned_host(delta) || !is_pinned_host(y)) return nullptr;
  if (!f.step_plan || f.step_plan->k != &K || f.step_plan->k_uid != K.uid ||
      f.step_plan->want_S != S ||
      f.step_plan->growth != env_int("SAG_STEP_GROWTH", 100))
    f.step_plan = step_plan_build(c, f, K, S);
  StepPlan& P = *f.step_plan;
  if (P.S == 0) return nullptr;
  return &P;
}

static void vanka_spmv_pipelined(Ctx& c, const Vanka& f, const Matrix& K, StepPlan& P,
                                 const double* x, double* delta, double* y) {
  const int S = P.S;
  const int n = f.n;
  double* dx = c.stage_buf(0, n);
  double* dd = c.stage_buf(1, n);
  double* dy = c.stage_buf(2, n);
  // SAG_STEP_SMCOPY=0: the DMA engines (one cudaMemcpyAsync per range)
  const int ctas = env_int("SAG_STEP_SMCOPY", 16);
  const double* mx = ctas > 0 ? host_mapped(x) : nullptr;
  double* md = ctas > 0 ? host_mapped(delta) : nullptr;
  double* my = ctas > 0 ? host_mapped(y) : nullptr;
  const bool sm = mx && md && my;
  // per direction (diagnostic): SAG_STEP_SMIN / SAG_STEP_SMOUT = 0 keep that direction on DMA
  const bool sm_in = sm && env_int("SAG_STEP_SMIN", 1) != 0;
  const bool sm_out = sm && env_int("SAG_STEP_SMOUT", 1) != 0;
  const bool trace = env_int("SAG_STEP_TRACE", 0) == 1;
  const bool ktrace = env_int("SAG_STEP_TRACE", 0) == 2;
  if (ktrace && P.ktrace.n < 6 * (size_t)S) {
    P.ktrace.alloc(6 * (size_t)S);
    if (P.exec) cudaGraphExecDestroy(P.exec);
    P.exec = nullptr;
  }
  auto ktr = [&](int kind, int q) { return ktrace ? P.ktrace.p + 2 * ((size_t)kind * S + q) : nullptr; };
  auto ktrace_reset = [&]() {
    if (!ktrace) return;
    std::vector<unsigned long long> h(6 * (size_t)S);
    for (size_t i = 0; i < h.size(); i += 2) {
      h[i] = ~0ull;
      h[i + 1] = 0ull;
    }
    SAG_CUDA(cudaMemcpy(P.ktrace.p, h.data(), 8 * h.size(), cudaMemcpyHostToDevice));
  };
  auto ktrace_print = [&]() {
    if (!ktrace) return;
    std::vector<unsigned long long> h(6 * (size_t)S);
    SAG_CUDA(cudaMemcpy(h.data(), P.ktrace.p, 8 * h.size(), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < h.size(); i += 2) t0 = std::min(t0, h[i]);
    const char* nm[3] = {"in", "yout", "dout"};
    for (int k = 0; k < 3; ++k)
      for (int q = 0; q < S; ++q) {
        const unsigned long long a = h[2 * ((size_t)k * S + q)], b = h[2 * ((size_t)k * S + q) + 1];
        if (b) fprintf(stderr, "step-ktrace %s%d %8.1f .. %8.1f us\n", nm[k], q, (a - t0) * 1e-3, (b - t0) * 1e-3);
      }
  };
  ktrace_reset();
  // SAG_STEP_GRAPH=0: enqueue operation by operation
  const bool graph = !trace && env_int("SAG_STEP_GRAPH", 1) != 0;
  const void* key[7] = {x, delta, y, dx, dd, dy,
                        (const void*)(size_t)((sm ? ctas : 0) + (ktrace ? 1000 : 0) +
                                              (sm_in ? 2000 : 0) + (sm_out ? 4000 : 0))};
  if (graph && P.exec && std::memcmp(key, P.gkey, sizeof(key)) == 0) {
    SAG_CUDA(cudaGraphLaunch(P.exec, c.stream));
    c.launches += P.graph_launches;
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    ktrace_print();
    return;
  }
  // an error while capturing must not leave the stream in capture mode
  struct CaptureGuard {
    cudaStream_t st = nullptr;
    ~CaptureGuard() {
      if (st) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
      }
    }
  } guard;
  const long long launches0 = c.launches;
  if (graph) {
    if (P.exec) {
      cudaGraphExecDestroy(P.exec);
      P.exec = nullptr;
    }
    SAG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    guard.st = c.stream;
  }
  // the copy streams start after whatever the compute stream holds
  cudaEvent_t e0 = P.ev[3 * (size_t)S];
  SAG_CUDA(cudaEventRecord(e0, c.stream));
  SAG_CUDA(cudaStreamWaitEvent(P.sin, e0, 0));
  SAG_CUDA(cudaStreamWaitEvent(P.sout, e0, 0));
  // SAG_STEP_TRACE=1 (diagnostic): timestamps of every stage on the three streams
  std::vector<cudaEvent_t> te;
  std::vector<std::string> tn;
  auto mark = [&](cudaStream_t st, const std::string& name) {
    if (!trace) return;
    cudaEvent_t e;
    SAG_CUDA(cudaEventCreate(&e));
    SAG_CUDA(cudaEventRecord(e, st));
    te.push_back(e);
    tn.push_back(name);
  };
  mark(c.stream, "start");
  for (int q = 0; q < S; ++q) {
    if (sm_in) {
      step_copy(c, P.sin, mx, dx, P.in[q], ctas, ktr(0, q));
    } else {
      for (const auto& r : P.in[q])
        SAG_CUDA(cudaMemcpyAsync(dx + r.a, x + r.a, sizeof(double) * (r.b - r.a),
                                 cudaMemcpyHostToDevice, P.sin));
    }
    SAG_CUDA(cudaEventRecord(P.ev[q], P.sin));
    mark(P.sin, "in" + std::to_string(q));
  }
  // SpMV on its own stream (independent of the Vanka chain on c.stream)
  SAG_CUDA(cudaStreamWaitEvent(P.ssp, e0, 0));
  for (int q = 0; q < S; ++q) {
    SAG_CUDA(cudaStreamWaitEvent(P.ssp, P.ev[q], 0));
    for (const auto& R : P.rows_rr[q]) launch_spmv_ranges(c, K, R, dx, dy, P.ssp);
    mark(P.ssp, "spmv" + std::to_string(q));
    if (!P.rows[q].empty()) {
      SAG_CUDA(cudaEventRecord(P.ev[S + q], P.ssp));
      SAG_CUDA(cudaStreamWaitEvent(P.sout, P.ev[S + q], 0));
      if (sm_out) {
        step_copy(c, P.sout, dy, my, P.rows[q], ctas, ktr(1, q));
      } else {
        for (const auto& r : P.rows[q])
          SAG_CUDA(cudaMemcpyAsync(y + r.a, dy + r.a, sizeof(double) * (r.b - r.a),
                                   cudaMemcpyDeviceToHost, P.sout));
      }
      mark(P.sout, "yout" + std::to_string(q));
    }
    SAG_CUDA(cudaStreamWaitEvent(c.stream, P.ev[q], 0));
    if (!P.pat[q].empty()) launch_patch_any(c, f, dx, nullptr, &P.pat[q]);
    mark(c.stream, "patch" + std::to_string(q));
    for (const auto& R : P.gat_rr[q]) {
      vanka_gather_ranges_kernel<<<grid_for(c, R.total()), 256, 0, c.stream>>>(
          R, f.dof_ptr.p, f.out.p, f.w_ext ? f.w.p : nullptr, dd);
      SAG_LAUNCHED(c);
    }
    mark(c.stream, "gather" + std::to_string(q));
    if (!P.gat[q].empty()) {
      SAG_CUDA(cudaEventRecord(P.ev[2 * S + q], c.stream));
      SAG_CUDA(cudaStreamWaitEvent(P.sout, P.ev[2 * S + q], 0));
      if (sm_out) {
        step_copy(c, P.sout, dd, md, P.gat[q], ctas, ktr(2, q));
      } else {
        for (const auto& r : P.gat[q])
          SAG_CUDA(cudaMemcpyAsync(delta + r.a, dd + r.a, sizeof(double) * (r.b - r.a),
                                   cudaMemcpyDeviceToHost, P.sout));
      }
      mark(P.sout, "dout" + std::to_string(q));
    }
  }
  // join the side streams into the compute stream
  SAG_CUDA(cudaEventRecord(P.ev[3 * (size_t)S + 1], P.sin));
  SAG_CUDA(cudaStreamWaitEvent(c.stream, P.ev[3 * (size_t)S + 1], 0));
  SAG_CUDA(cudaEventRecord(P.ev[3 * (size_t)S + 2], P.sout));
  SAG_CUDA(cudaStreamWaitEvent(c.stream, P.ev[3 * (size_t)S + 2], 0));
  SAG_CUDA(cudaEventRecord(P.ev[3 * (size_t)S + 3], P.ssp));
  SAG_CUDA(cudaStreamWaitEvent(c.stream, P.ev[3 * (size_t)S + 3], 0));
  if (graph) {
    cudaGraph_t g = nullptr;
    guard.st = nullptr;
    SAG_CUDA(cudaStreamEndCapture(c.stream, &g));
    P.graph_launches = c.launches - launches0;
    cudaError_t e = cudaGraphInstantiate(&P.exec, g, 0);
    cudaGraphDestroy(g);
    SAG_CUDA(e);
    std::memcpy(P.gkey, key, sizeof(key));
    SAG_CUDA(cudaGraphLaunch(P.exec, c.stream));
  }
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  if (trace) {
    for (size_t i = 1; i < te.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, te[0], te[i]);
      fprintf(stderr, "step-trace %-10s %8.1f us\n", tn[i].c_str(), 1e3 * ms);
    }
    for (auto e : te) cudaEventDestroy(e);
  }
  return;
}

// vanka_gather_seq_kernel on a few dof ranges in one launch
__global__ void vanka_gather_ranges_kernel(RowRanges R, const int* __restrict__ dof_ptr,
                                           const double* __restrict__ out,
                                           const double* __restrict__ w, double* __restrict__ delta) {
  constexpr int U = 8;
  const int total = R.total();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < total; v += gridDim.x * blockDim.x) {
    const int d = R.row(v);
    const int s0 = __ldg(dof_ptr + d), s1 = __ldg(dof_ptr + d + 1);
    const double wd = w ? __ldg(w + d) : (s1 > s0 ? 1.0 / (double)(s1 - s0) : 0.0);
    double acc = 0.0;
    for (int sb = s0; sb < s1; sb += U) {
      double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) vv[u] = sb + u < s1 ? __ldcs(out + sb + u) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (sb + u < s1) acc = __dadd_rn(acc, __dmul_rn(wd, vv[u]));
    }
    delta[d] = acc;
  }
}

void vanka_apply_stationary(Ctx& c, const Vanka& f, const double* r, double* x, double omega) {
  launch_patch_any(c, f, r, nullptr);
  launch_gather(c, f, nullptr, x, omega, nullptr);
}

// The reference's factor layout (vanka.hpp:31-33), unpacked on the host for
// parity tests.
void vanka_export(Ctx& c, const Vanka& f, double* uhat, double* bhat, double* sinv,
                  double* weights) {
  std::vector<double> D((f.blob_bytes + 7) / 8);
  SAG_CUDA(cudaMemcpyAsync(D.data(), f.blob.p, f.blob_bytes, cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  const long long es = 1;
  size_t ou = 0, os = 0;
  for (int k = 0; k < f.npatch; ++k) {
    const int nx = f.h_nx[k], nv = f.h_nv[k], ny = nv - nx, np = f.h_np[k];
    const double* base = D.data() + f.h_dbase[k];
    const double *Bh, *Si, *Ux, *Uy;
    long long urx, ury;
    if (vanka_paired(f.pairs, nx, ny, np)) {  // (A) | (U) | (B) pairs | S^-1
      const int m = std::max(nx, ny);
      const bool nob = !f.h_nob.empty() && f.h_nob[k];
      const double* U2 = base + 2 * ainv_len(m, true);
      const double* B2 = U2 + 2LL * np * m;
      const double* S2 = B2 + (nob ? 0 : 2LL * np * m);
      for (int i = 0; i < nv; ++i)
        for (int a = 0; a < np; ++a) {
          const long long e = 2LL * a * m + (i < nx ? 2 * i : 2 * (i - nx) + 1);
          if (uhat) uhat[ou + (size_t)i * np + a] = U2[e];
          if (bhat && !nob) bhat[ou + (size_t)a * nv + i] = B2[e];
          if (bhat && nob) {  // b_hat = S^-1 u_hat^T (vanka.cpp:133-140), as the kernels do
            double acc = 0.0;
            for (int q = 0; q < np; ++q)
              acc += S2[a * np + q] * U2[2LL * q * m + (i < nx ? 2 * i : 2 * (i - nx) + 1)];
            bhat[ou + (size_t)a * nv + i] = acc;
          }
        }
      if (sinv)
        for (int e = 0; e < np * np; ++e) sinv[os + e] = S2[e];
      ou += (size_t)nv * np;
      os += (size_t)np * np;
      continue;
    } else {  // A_x | A_y | U | B_hat | S^-1
      Ux = base + (ainv_len(nx, f.sym) + ainv_len(ny, f.sym)) * es;
      Uy = Ux + (long long)nx * es;
      Bh = Ux + (long long)np * nv * es;
      Si = Bh + (long long)np * nv * es;
      urx = ury = nv;
    }
    for (int i = 0; i < nv; ++i)
      for (int a = 0; a < np; ++a) {
        const double u = i < nx ? Ux[(a * urx + i) * es] : Uy[(a * ury + i - nx) * es];
        if (uhat) uhat[ou + (size_t)i * np + a] = u;
        if (bhat) bhat[ou + (size_t)a * nv + i] = Bh[(a * nv + i) * es];
      }
    if (sinv)
      for (int e = 0; e < np * np; ++e) sinv[os + e] = Si[e * es];
    ou += (size_t)nv * np;
    os += (size_t)np * np;
  }
  if (weights) SAG_CUDA(cudaMemcpy(weights, f.w.p, sizeof(double) * f.n, cudaMemcpyDefault));
}



// ================================ 3 velocity components (BASELINE config 5) ==
// The reference is 2D only; this is the 3-component
// generalisation of factor_patches / apply_vanka (vanka.cpp:64-184 with x, y,
// z blocks; oracle.c or_*3 is its CPU restatement). 3D Taylor-Hood patches
// hold ~100-250 dofs (m up to ~60 per component), too large for a warp, so
// both kernels run one CTA per patch.
//
// Blob per patch (16-byte aligned, int64 offset table, patch order):
//   header {cnt_x, cnt_y, cnt_z, np, nv, slot_base, 0, 0}
//   A_c^-1 (c = x, y, z): the explicit inverse (columns = the LU solves of
//          the unit vectors, sparse.cpp:343-361), symmetrised, upper triangle
//          packed by columns
//   U_hat (nv x np, [i np + a]) | B_hat (np x nv) | S^-1 (np x np)
//   velocity dofs (nv) | pressure dofs (np)
struct Vanka3 {
  int n = 0, npatch = 0, max_nv = 0, max_m = 0, max_np = 0;
  long long max_doubles = 0;  // factor doubles of the largest patch
  DevBuf<unsigned char> blob;
  DevBuf<long long> off;
  long long blob_bytes = 0, nslots = 0, a_factor_bytes = 0, aux_bytes = 0;
  DevBuf<double> out;
  DevBuf<int> dof_ptr, dof_slot;
};

// A_c^-1 of a symmetric block is stored as the symmetrised upper triangle
// packed by columns (as the 2D blobs): m (m + 1) / 2 doubles
__host__ __device__ inline long long v3_tri(int m) { return (long long)m * (m + 1) / 2; }
__host__ __device__ inline long long v3_doubles(int mx, int my, int mz, int np) {
  const long long nv = mx + my + mz;
  return v3_tri(mx) + v3_tri(my) + v3_tri(mz) + 2 * nv * np + (long long)np * np;
}

// CTA per patch: A_c gathered into shared memory, LU with partial pivoting
// (sparse.cpp:310-341: first max |a_ik|, whole-row swaps, multiplier
// a_ik (1 / a_kk)), the inverse's columns by thread-per-column substitution,
// then U_hat = -A^-1 B^T, S = B U_hat, S^-1, B_hat = S^-1 U_hat^T
// (vanka.cpp:99-140, the symmetric-A b_hat formula)
__global__ void __launch_bounds__(256) factor3_kernel(
    int npatch, int n_u1, int n_u2, const int* __restrict__ rp, const int* __restrict__ ci,
    const double* __restrict__ kv, const int* __restrict__ vptr, const int* __restrict__ vidx,
    const int* __restrict__ pidx, const int* __restrict__ pptr, const long long* __restrict__ off,
    unsigned char* blob, int MM, int* err) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = blockIdx.x; k < npatch; k += gridDim.x) {
    const int v0 = vptr[k], nv = vptr[k + 1] - v0;
    const int p0 = pptr[k], np = pptr[k + 1] - p0;
    const int* vel = vidx + v0;
    int cnt[3] = {0, 0, 0};
    for (int i = 0; i < nv; ++i) cnt[vel[i] < n_u1 ? 0 : vel[i] < n_u2 ? 1 : 2]++;
    unsigned char* B = blob + off[k];
    int* hdr = reinterpret_cast<int*>(B);
    double* D = reinterpret_cast<double*>(B + 32);
    if (tid == 0) {
      hdr[0] = cnt[0];
      hdr[1] = cnt[1];
      hdr[2] = cnt[2];
      hdr[3] = np;
      hdr[4] = nv;
      hdr[6] = hdr[7] = 0;
    }
    const long long nA = v3_tri(cnt[0]) + v3_tri(cnt[1]) + v3_tri(cnt[2]);
    double* gU = D + nA;
    double* gB = gU + (long long)nv * np;
    double* gS = gB + (long long)np * nv;
    int* gI = reinterpret_cast<int*>(gS + np * np);
    for (int i = tid; i < nv; i += nt) gI[i] = vel[i];
    for (int a = tid; a < np; a += nt) gI[nv + a] = pidx[p0 + a];
    // shared: A (MM x MM) | W (MM x MM) | Bm (np x nv) | piv (MM) | scratch
    double* A = sm;
    double* W = A + (size_t)MM * MM;
    double* Bm = W + (size_t)MM * MM;
    int* piv = reinterpret_cast<int*>(Bm + (size_t)4 * 512);  // Bm: np <= 4 rows of nv <= 511
    __shared__ int s_p;
    __shared__ int s_bad;
    // B rows of the patch (np x nv), missing entries 0 (vanka.cpp:47-60)
    for (int e = tid; e < np * nv; e += nt) Bm[e] = 0.0;
    __syncthreads();
    for (int a = 0; a < np; ++a) {
      const int row = pidx[p0 + a];
      for (int q = rp[row] + tid; q < rp[row + 1]; q += nt) {
        const int pos = bsearch_idx(vel, nv, ci[q]);
        if (pos >= 0) Bm[a * nv + pos] = kv[q];
      }
    }
    __syncthreads();
    int off_c = 0;
    double* gA = D;
    for (int c = 0; c < 3; ++c) {
      const int m = cnt[c];
      const int* vc = vel + off_c;
      for (int e = tid; e < m * m; e += nt) A[e] = 0.0;
      __syncthreads();
      for (int r = tid; r < m; r += nt) {
        const int row = vc[r];
        for (int q = rp[row]; q < rp[row + 1]; ++q) {
          const int pos = bsearch_idx(vc, m, ci[q]);
          if (pos >= 0) A[r * m + pos] = kv[q];
        }
      }
      for (int i = tid; i < m; i += nt) piv[i] = i;
      if (tid == 0) s_bad = 0;
      __syncthreads();
      for (int kk = 0; kk < m; ++kk) {
        if (tid == 0) {
          int p = kk;
          double best = fabs(A[kk * m + kk]);
          for (int i = kk + 1; i < m; ++i) {
            const double v = fabs(A[i * m + kk]);
            if (v > best) {
              best = v;
              p = i;
            }
          }
          if (best == 0.0) s_bad = 1;
          s_p = p;
          if (p != kk) {
            const int t = piv[kk];
            piv[kk] = piv[p];
            piv[p] = t;
          }
        }
        __syncthreads();
        if (s_bad) break;
        const int p = s_p;
        if (p != kk)
          for (int j = tid; j < m; j += nt) {
            const double t = A[kk * m + j];
            A[kk * m + j] = A[p * m + j];
            A[p * m + j] = t;
          }
        __syncthreads();
        const double inv_piv = 1.0 / A[kk * m + kk];
        for (int i = kk + 1 + tid; i < m; i += nt) A[i * m + kk] *= inv_piv;
        __syncthreads();
        for (int e = tid; e < (m - kk - 1) * (m - kk - 1); e += nt) {
          const int i = kk + 1 + e / (m - kk - 1), j = kk + 1 + e % (m - kk - 1);
          const double mult = A[i * m + kk];
          if (mult != 0.0) A[i * m + j] -= mult * A[kk * m + j];
        }
        __syncthreads();
      }
      if (s_bad) {
        if (tid == 0) atomicMin(err, k);
        break;
      }
      // inverse columns: thread j solves L U x = P e_j (sparse.cpp:343-361)
      for (int j = tid; j < m; j += nt) {
        double* x = W + (size_t)j * m;  // column j, contiguous
        for (int i = 0; i < m; ++i) x[i] = piv[i] == j ? 1.0 : 0.0;
        for (int i = 1; i < m; ++i) {
          double acc = x[i];
          for (int q = 0; q < i; ++q) acc -= A[i * m + q] * x[q];
          x[i] = acc;
        }
        for (int i = m - 1; i >= 0; --i) {
          double acc = x[i];
          for (int q = i + 1; q < m; ++q) acc -= A[i * m + q] * x[q];
          x[i] = acc / A[i * m + i];
        }
      }
      __syncthreads();
      // symmetrised upper triangle by columns: (i, j), i <= j at j(j+1)/2 + i
      for (int e = tid; e < m * m; e += nt) {
        const int j = e / m, i = e % m;
        if (i <= j) gA[j * (j + 1) / 2 + i] = 0.5 * (W[(size_t)j * m + i] + W[(size_t)i * m + j]);
      }
      // U_hat rows of this component: u(i, a) = -sum_j W(i, j) B(a, off_c + j)
      for (int e = tid; e < m * np; e += nt) {
        const int i = e / np, a = e % np;
        double acc = 0.0;
        for (int j = 0; j < m; ++j) acc -= W[(size_t)j * m + i] * Bm[a * nv + off_c + j];
        gU[(size_t)(off_c + i) * np + a] = acc;
      }
      __syncthreads();
      gA += v3_tri(m);
      off_c += m;
    }
    if (s_bad) continue;
    __syncthreads();
    // S = B U_hat (np x np), its inverse (np <= 4: one thread), B_hat
    if (tid == 0) {
      double S[16], L[16];
      int pv[4];
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) {
          double acc = 0.0;
          for (int q = 0; q < nv; ++q) acc += Bm[a * nv + q] * gU[(size_t)q * np + b];
          S[a * np + b] = acc;
        }
      for (int i = 0; i < np * np; ++i) L[i] = S[i];
      for (int i = 0; i < np; ++i) pv[i] = i;
      bool ok = true;
      for (int kk = 0; kk < np && ok; ++kk) {
        int p = kk;
        double best = fabs(L[kk * np + kk]);
        for (int i = kk + 1; i < np; ++i)
          if (fabs(L[i * np + kk]) > best) {
            best = fabs(L[i * np + kk]);
            p = i;
          }
        if (best == 0.0) {
          ok = false;
          break;
        }
        if (p != kk) {
          for (int j = 0; j < np; ++j) {
            const double t = L[kk * np + j];
            L[kk * np + j] = L[p * np + j];
            L[p * np + j] = t;
          }
          const int t = pv[kk];
          pv[kk] = pv[p];
          pv[p] = t;
        }
        const double ip = 1.0 / L[kk * np + kk];
        for (int i = kk + 1; i < np; ++i) {
          const double mult = L[i * np + kk] * ip;
          L[i * np + kk] = mult;
          for (int j = kk + 1; j < np; ++j) L[i * np + j] -= mult * L[kk * np + j];
        }
      }
      if (!ok) {
        atomicMin(err, k);
      } else {
        for (int j = 0; j < np; ++j) {
          double x[4];
          for (int i = 0; i < np; ++i) x[i] = pv[i] == j ? 1.0 : 0.0;
          for (int i = 1; i < np; ++i)
            for (int q = 0; q < i; ++q) x[i] -= L[i * np + q] * x[q];
          for (int i = np - 1; i >= 0; --i) {
            for (int q = i + 1; q < np; ++q) x[i] -= L[i * np + q] * x[q];
            x[i] /= L[i * np + i];
          }
          for (int i = 0; i < np; ++i) gS[i * np + j] = x[i];
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < np * nv; e += nt) {
      const int a = e / nv, c = e % nv;
      double acc = 0.0;
      for (int q = 0; q < np; ++q) acc += gS[a * np + q] * gU[(size_t)c * np + q];
      gB[(size_t)a * nv + c] = acc;
    }
    __syncthreads();
  }
}

// CTA per patch: the patch's factors (packed A_c^-1, U_hat, B_hat, S^-1 --
// ~40 KB at 3D Taylor-Hood sizes) are staged into shared memory by coalesced
// 16-byte loads of the whole CTA, b gathered beside them; then t_c = A_c^-1
// b_c (thread = row, the packed symmetric addressing of the 2D kernels),
// x_p = S^-1 b_p + B_hat b_u (block sum), x_u = t + U_hat x_p, unweighted
// local results to the patch's slots (vanka.cpp:154-181; the weighted,
// ordered scatter is the gather kernel).
__global__ void __launch_bounds__(256) apply3_kernel(int npatch,
                                                     const unsigned char* __restrict__ blob,
                                                     const long long* __restrict__ off,
                                                     const double* __restrict__ r,
                                                     double* __restrict__ out) {
  extern __shared__ __align__(16) double fac[];  // the factor doubles of one patch
  __shared__ double sb[512];
  __shared__ double red[8][4];
  __shared__ double xp[4];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  for (int k = blockIdx.x; k < npatch; k += gridDim.x) {
    const unsigned char* B = blob + off[k];
    const int4 h0 = *reinterpret_cast<const int4*>(B);
    const int4 h1 = *reinterpret_cast<const int4*>(B + 16);
    const int cnt[3] = {h0.x, h0.y, h0.z};
    const int np = h0.w, nv = h1.x, sbase = h1.y;
    const long long nd = v3_doubles(cnt[0], cnt[1], cnt[2], np);
    const double2* src = reinterpret_cast<const double2*>(B + 32);
    for (long long e = tid; e < (nd + 1) / 2; e += nt) reinterpret_cast<double2*>(fac)[e] = __ldg(src + e);
    const int* idx = reinterpret_cast<const int*>(reinterpret_cast<const double*>(B + 32) + nd);
    for (int i = tid; i < nv + np; i += nt) sb[i] = __ldg(r + idx[i]);
    __syncthreads();
    const long long nA = v3_tri(cnt[0]) + v3_tri(cnt[1]) + v3_tri(cnt[2]);
    const double* U = fac + nA;
    const double* Bh = U + (long long)nv * np;
    const double* Si = Bh + (long long)np * nv;
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = tid; j < nv; j += nt)
      for (int a = 0; a < np; ++a) part[a] = fma(Bh[(size_t)a * nv + j], sb[j], part[a]);
    for (int a = 0; a < np; ++a) {
      double v = part[a];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wid][a] = v;
    }
    double t[2] = {0.0, 0.0};
    int rowi[2] = {-1, -1};
    {
      int q = 0;
      for (int i = tid; i < nv && q < 2; i += nt, ++q) {
        int c = 0, base = 0;
        const double* Ac = fac;
        while (i - base >= cnt[c]) {
          Ac += v3_tri(cnt[c]);
          base += cnt[c++];
        }
        rowi[q] = i;
        const int m = cnt[c], li = i - base;
        const int cl = li * (li + 1) / 2;
        double acc = 0.0;
        int cs = 0;
        for (int j = 0; j < m; cs += ++j)
          acc = fma(Ac[li <= j ? cs + li : cl + j], sb[base + j], acc);
        t[q] = acc;
      }
    }
    __syncthreads();
    if (tid < np) {
      double acc = 0.0;
      for (int w = 0; w < (nt >> 5); ++w) acc += red[w][tid];
      for (int j = 0; j < np; ++j) acc = fma(Si[tid * np + j], sb[nv + j], acc);
      xp[tid] = acc;
      out[sbase + nv + tid] = acc;
    }
    __syncthreads();
    for (int q = 0; q < 2; ++q) {
      if (rowi[q] < 0) continue;
      const int i = rowi[q];
      double acc = t[q];
      for (int a = 0; a < np; ++a) acc = fma(U[(size_t)i * np + a], xp[a], acc);
      out[sbase + i] = acc;
    }
    __syncthreads();
  }
}

__global__ void slot_base3_kernel(int npatch, const long long* off, const int* sbase,
                                  unsigned char* blob) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < npatch; k += gridDim.x * blockDim.x)
    reinterpret_cast<int*>(blob + off[k])[5] = sbase[k];
}

std::unique_ptr<Vanka3> factor3_dev(Ctx& c, const Matrix& k, int n_x, int n_y, int n_z,
                                    int n_p) {
  const int n = k.nrows, n_u = n_x + n_y + n_z;
  SAG_REQUIRE(n == n_u + n_p && k.ncols == n, SAG_DIMENSION_MISMATCH,
              "factor_patches3: block sizes do not match K");
  std::vector<int> rp(n + 1), ci(std::max<long long>(k.nnz, 1));
  SAG_CUDA(cudaMemcpy(rp.data(), k.rp.p, 4 * (size_t)(n + 1), cudaMemcpyDeviceToHost));
  if (k.nnz) SAG_CUDA(cudaMemcpy(ci.data(), k.ci.p, 4 * (size_t)k.nnz, cudaMemcpyDeviceToHost));
  auto f = std::make_unique<Vanka3>();
  f->n = n;
  f->npatch = n_p;
  // patches (vanka.cpp:11-42, one seed): the seed row's velocity columns
  std::vector<int> vptr(n_p + 1, 0), vidx, pptr(n_p + 1), pidx(n_p);
  std::vector<long long> offh(n_p + 1, 0);
  std::vector<int> sbase(std::max(n_p, 1));
  long long slots = 0;
  for (int i = 0; i < n_p; ++i) {
    const int row = n_u + i;
    int cnt[3] = {0, 0, 0};
    for (int q = rp[row]; q < rp[row + 1]; ++q)
      if (ci[q] < n_u) {
        vidx.push_back(ci[q]);
        cnt[ci[q] < n_x ? 0 : ci[q] < n_x + n_y ? 1 : 2]++;
      }
    vptr[i + 1] = (int)vidx.size();
    pptr[i] = i;
    pidx[i] = row;
    const int nv = vptr[i + 1] - vptr[i];
    SAG_REQUIRE(nv > 0, SAG_SINGULAR_PATCH, "build_patches3: pressure row couples to no velocity DoFs");
    f->max_nv = std::max(f->max_nv, nv);
    f->max_m = std::max({f->max_m, cnt[0], cnt[1], cnt[2]});
    f->max_doubles = std::max(f->max_doubles, v3_doubles(cnt[0], cnt[1], cnt[2], 1));
    long long bytes = 32 + 8 * v3_doubles(cnt[0], cnt[1], cnt[2], 1) + 4LL * (nv + 1);
    bytes = (bytes + 15) / 16 * 16;
    offh[i + 1] = offh[i] + bytes;
    sbase[i] = (int)slots;
    slots += nv + 1;
    f->a_factor_bytes += 8LL * (v3_tri(cnt[0]) + v3_tri(cnt[1]) + v3_tri(cnt[2]));
    f->aux_bytes += 8LL * (2 * nv + 1);
  }
  pptr[n_p] = n_p;
  f->max_np = 1;
  SAG_REQUIRE(f->max_nv + f->max_np <= 512, SAG_DIMENSION_MISMATCH,
              "factor_patches3: patch larger than 512 dofs");
  SAG_REQUIRE(slots < (1LL << 31), SAG_DIMENSION_MISMATCH, "factor_patches3: too many slots");
  f->blob_bytes = offh[n_p];
  f->nslots = slots;
  f->blob.alloc(std::max<long long>(offh[n_p], 16));
  f->off.alloc(n_p + 1);
  SAG_CUDA(cudaMemcpy(f->off.p, offh.data(), 8 * (size_t)(n_p + 1), cudaMemcpyHostToDevice));
  DevBuf<int> dvptr(n_p + 1), dvidx(std::max<size_t>(vidx.size(), 1)), dpptr(n_p + 1),
      dpidx(std::max(n_p, 1)), dsb(std::max(n_p, 1)), err(1);
  SAG_CUDA(cudaMemcpy(dvptr.p, vptr.data(), 4 * (size_t)(n_p + 1), cudaMemcpyHostToDevice));
  if (!vidx.empty())
    SAG_CUDA(cudaMemcpy(dvidx.p, vidx.data(), 4 * vidx.size(), cudaMemcpyHostToDevice));
  SAG_CUDA(cudaMemcpy(dpptr.p, pptr.data(), 4 * (size_t)(n_p + 1), cudaMemcpyHostToDevice));
  if (n_p) {
    SAG_CUDA(cudaMemcpy(dpidx.p, pidx.data(), 4 * (size_t)n_p, cudaMemcpyHostToDevice));
    SAG_CUDA(cudaMemcpy(dsb.p, sbase.data(), 4 * (size_t)n_p, cudaMemcpyHostToDevice));
  }
  const int big = 0x7fffffff;
  SAG_CUDA(cudaMemcpy(err.p, &big, sizeof(int), cudaMemcpyHostToDevice));
  if (n_p > 0) {
    const int MM = std::max(f->max_m, 1);
    const size_t smem = (size_t)2 * MM * MM * 8 + 4 * 512 * 8 + 4 * MM + 16;
    SAG_REQUIRE(smem <= 227 * 1024, SAG_DIMENSION_MISMATCH,
                "factor_patches3: velocity block too large for shared memory");
    SAG_CUDA(cudaFuncSetAttribute(factor3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    const int blocks = std::min(n_p, c.num_sms * 8);
    factor3_kernel<<<blocks, 256, smem, c.stream>>>(n_p, n_x, n_x + n_y, k.rp.p, k.ci.p, k.v.p,
                                                    dvptr.p, dvidx.p, dpidx.p, dpptr.p,
                                                    f->off.p, f->blob.p, MM, err.p);
    SAG_LAUNCHED(c);
    slot_base3_kernel<<<grid_for(c, n_p), 256, 0, c.stream>>>(n_p, f->off.p, dsb.p, f->blob.p);
    SAG_LAUNCHED(c);
  }
  int herr = big;
  SAG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  SAG_REQUIRE(herr == big, SAG_SINGULAR_PATCH,
              "factor_patches3: singular block in patch " + std::to_string(herr));
  // dof -> slot map (slots in patch order: ascending patch order per dof)
  std::vector<int> cnt(n + 1, 0), dslot(std::max<long long>(slots, 1));
  for (int i = 0; i < n_p; ++i) {
    for (int q = vptr[i]; q < vptr[i + 1]; ++q) ++cnt[vidx[q] + 1];
    ++cnt[pidx[i] + 1];
  }
  for (int d = 0; d < n; ++d) cnt[d + 1] += cnt[d];
  std::vector<int> pos(cnt.begin(), cnt.end() - 1);
  for (int i = 0; i < n_p; ++i) {
    int sl = sbase[i];
    for (int q = vptr[i]; q < vptr[i + 1]; ++q) dslot[pos[vidx[q]]++] = sl++;
    dslot[pos[pidx[i]]++] = sl;
  }
  f->dof_ptr.alloc(n + 1);
  f->dof_slot.alloc(std::max<long long>(slots, 1));
  f->out.alloc(std::max<long long>(slots, 1));
  SAG_CUDA(cudaMemcpy(f->dof_ptr.p, cnt.data(), 4 * (size_t)(n + 1), cudaMemcpyHostToDevice));
  if (slots)
    SAG_CUDA(cudaMemcpy(f->dof_slot.p, dslot.data(), 4 * (size_t)slots, cudaMemcpyHostToDevice));
  return f;
}

void apply3_dev(Ctx& c, const Vanka3& f, const double* r, double* delta) {
  if (f.npatch > 0) {
    const size_t smem = 8 * (size_t)(f.max_doubles + 2);
    SAG_REQUIRE(smem <= 200 * 1024, SAG_DIMENSION_MISMATCH, "apply_vanka3: patch too large");
    static thread_local size_t configured = 0;
    if (configured < smem) {
      SAG_CUDA(cudaFuncSetAttribute(apply3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      configured = smem;
    }
    int occ = 0;
    SAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apply3_kernel, 256, smem));
    const int blocks = std::min(f.npatch, std::max(occ, 1) * c.num_sms);
    apply3_kernel<<<blocks, 256, smem, c.stream>>>(f.npatch, f.blob.p, f.off.p, r, f.out.p);
    SAG_LAUNCHED(c);
  }
  vanka_gather_kernel<<<grid_for(c, f.n), 256, 0, c.stream>>>(
      f.n, f.dof_ptr.p, f.dof_slot.p, f.out.p, nullptr, delta, nullptr, 1.0, nullptr);
  SAG_LAUNCHED(c);
}

}  // namespace sag

// =================================================================== C-ABI
using namespace sag;

extern "C" {

int sag_build_patches(sag_ctx* ctx, const sag_matrix* k, int n_x, int n_y, int n_p,
                      int sv_triples, sag_patches** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k);
    SAG_NOTNULL(out);
    *out = nullptr;
    auto p = build_patches_dev(ctx->c, k->m, n_x, n_y, n_p, sv_triples != 0);
    auto* h = new sag_patches;
    h->p = std::move(*p);
    *out = h;
  });
}

int sag_patches_create(sag_ctx* ctx, int npatch, const int* pressure_ptr, const int* pressure_idx,
                       const int* velocity_ptr, const int* velocity_idx, const int* nx,
                       sag_patches** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(out);
    SAG_NOTNULL(pressure_ptr);
    SAG_NOTNULL(velocity_ptr);
    *out = nullptr;
    auto p = patches_from_lists(ctx->c, npatch, pressure_ptr, pressure_idx, velocity_ptr,
                                velocity_idx, nx);
    auto* h = new sag_patches;
    h->p = std::move(*p);
    *out = h;
  });
}

int sag_patches_destroy(sag_patches* p) {
  return guard([&] { delete p; });
}

int sag_patches_info(const sag_patches* p, long long* info) {
  return guard([&] {
    SAG_NOTNULL(p);
    SAG_NOTNULL(info);
    info[0] = p->p.npatch;
    info[1] = p->p.tot_p;
    info[2] = p->p.tot_v;
    info[3] = p->p.max_nv;
    info[4] = p->p.max_np;
  });
}

int sag_patches_export(sag_ctx* ctx, const sag_patches* p, int* pptr, int* pidx, int* vptr,
                       int* vidx, int* nx) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(p);
    const auto& q = p->p;
    auto& c = ctx->c;
    if (pptr) SAG_CUDA(cudaMemcpyAsync(pptr, q.pptr.p, sizeof(int) * (q.npatch + 1), cudaMemcpyDefault, c.stream));
    if (vptr) SAG_CUDA(cudaMemcpyAsync(vptr, q.vptr.p, sizeof(int) * (q.npatch + 1), cudaMemcpyDefault, c.stream));
    if (pidx && q.tot_p) SAG_CUDA(cudaMemcpyAsync(pidx, q.pidx.p, sizeof(int) * q.tot_p, cudaMemcpyDefault, c.stream));
    if (vidx && q.tot_v) SAG_CUDA(cudaMemcpyAsync(vidx, q.vidx.p, sizeof(int) * q.tot_v, cudaMemcpyDefault, c.stream));
    if (nx && q.npatch) SAG_CUDA(cudaMemcpyAsync(nx, q.nx.p, sizeof(int) * q.npatch, cudaMemcpyDefault, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_factor_patches(sag_ctx* ctx, const sag_matrix* k, const sag_patches* p, int n_u,
                       sag_vanka** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k);
    SAG_NOTNULL(p);
    SAG_NOTNULL(out);
    // vanka.cpp:147 leaves n_u unused; here it delimits the velocity block
    // whose symmetry selects the packed A^-1 representation
    *out = nullptr;
    auto f = factor_patches_dev(ctx->c, k->m, p->p, n_u);
    auto* h = new sag_vanka;
    h->f = std::move(*f);
    h->c = &ctx->c;
    *out = h;
  });
}

int sag_vanka_destroy(sag_vanka* f) {
  return guard([&] {
    // only this context's stream can still hold work on the factorization
    // (plus the pipelined step's side streams, joined into it at every call)
    if (f && f->c) cudaStreamSynchronize(f->c->stream);
    delete f;
  });
}

int sag_vanka_stats(const sag_vanka* f, long long* s) {
  return guard([&] {
    SAG_NOTNULL(f);
    SAG_NOTNULL(s);
    const auto& v = f->f;
    s[0] = v.a_factor_bytes;
    s[1] = v.aux_bytes;
    s[2] = v.dense_inverse_bytes;
    s[3] = v.blob_bytes;
    s[4] = v.npatch;
    s[5] = v.n;
    s[6] = v.nslots;
  });
}

int sag_vanka_classes(const sag_vanka* f, long long* out, int cap, int* nclasses) {
  return guard([&] {
    SAG_NOTNULL(f);
    SAG_NOTNULL(nclasses);
    const auto& cls = f->f.rclasses;
    *nclasses = (int)cls.size();
    for (int i = 0; i < (int)cls.size() && i < cap; ++i) {
      out[4 * i + 0] = cls[i].R;
      out[4 * i + 1] = cls[i].lpp;
      out[4 * i + 2] = cls[i].k1 - cls[i].k0;
      out[4 * i + 3] = cls[i].bytes;
    }
  });
}

int sag_vanka_export(sag_ctx* ctx, const sag_vanka* f, double* u_hat, double* b_hat,
                     double* s_inv, double* weights) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    vanka_export(ctx->c, f->f, u_hat, b_hat, s_inv, weights);
  });
}

int sag_vanka_set_weights(sag_ctx* ctx, sag_vanka* f, const double* weights) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    SAG_NOTNULL(weights);
    SAG_CUDA(cudaMemcpyAsync(f->f.w.p, weights, sizeof(double) * f->f.n, cudaMemcpyDefault,
                             ctx->c.stream));
    SAG_CUDA(cudaStreamSynchronize(ctx->c.stream));
    f->f.w_ext = true;
  });
}

int sag_apply_vanka(sag_ctx* ctx, const sag_vanka* f, const double* r, double* delta) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    auto& c = ctx->c;
    InVec ri(c, r, f->f.n, 0);
    OutVec d(c, delta, f->f.n, 1, false);
    vanka_apply(c, f->f, ri.d, d.d);
    d.finish();
  });
}

int sag_apply_vanka_add(sag_ctx* ctx, const sag_vanka* f, const double* r, double* x,
                        double omega) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    auto& c = ctx->c;
    InVec ri(c, r, f->f.n, 0);
    OutVec xo(c, x, f->f.n, 1, true);
    vanka_apply_stationary(c, f->f, ri.d, xo.d, omega);
    xo.finish();
  });
}

int sag_apply_vanka_add_push(sag_ctx* ctx, const sag_vanka* f, const double* r, double* x,
                             double omega, const int* slot, const unsigned char* nbr, int npeer,
                             double* const* peers) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    SAG_REQUIRE(npeer >= 0 && npeer <= 8 && (npeer == 0 || peers), SAG_INVALID_ARGUMENT,
                "sag_apply_vanka_add_push: 0..8 peer buffers");
    SAG_REQUIRE(f->f.seq, SAG_CONFIG_ERROR,
                "sag_apply_vanka_add_push needs the dof-ordered result layout");
    auto& c = ctx->c;
    for (const void* p : {(const void*)r, (const void*)x, (const void*)slot, (const void*)nbr})
      SAG_REQUIRE(is_device_ptr(p), SAG_INVALID_ARGUMENT, "device pointers only");
    PeerMap pm{};
    for (int i = 0; i < npeer; ++i) pm.peer[i] = peers[i];
    launch_patch_any(c, f->f, r, nullptr);
    const double* w = f->f.w_ext ? f->f.w.p : nullptr;
    vanka_gather_push_kernel<<<grid_for(c, f->f.n), 256, 0, c.stream>>>(
        f->f.n, f->f.dof_ptr.p, f->f.out.p, w, x, omega, slot, nbr, pm);
    SAG_LAUNCHED(c);
  });
}

}  // extern "C"

// the step with x copied in first: device buffers in place; host outputs leave
// in chunks as they are computed
static void vanka_spmv_plain(Ctx& c, const sag_vanka* f, const sag_matrix* k, const double* x,
                             double* delta, double* y) {
  const int n = f->f.n;
  {
    InVec xi(c, x, n, 0);                 // x crosses the host link once
    OutVec yo(c, y, n, 2, false);
    OutVec d(c, delta, n, 1, false);
    if (!yo.host && !d.host) {
      launch_spmv(c, k->m, xi.d, yo.d, Epi::Store);
      vanka_apply(c, f->f, xi.d, d.d);
      return;
    }
    // host outputs: y and delta leave in row / dof chunks on the copy
    // stream as they are computed, so the device->host direction (twice the
    // bytes of the input) starts right after the first SpMV chunk and runs
    // under the rest of the step
    const int C = 4;
    cudaStream_t cs = c.copy();
    auto out_chunk = [&](double* host, const double* dev, int a, int b) {
      SAG_CUDA(cudaEventRecord(c.copy_ev, c.stream));
      SAG_CUDA(cudaStreamWaitEvent(cs, c.copy_ev, 0));
      SAG_CUDA(cudaMemcpyAsync(host + a, dev + a, sizeof(double) * (b - a),
                               cudaMemcpyDeviceToHost, cs));
    };
    for (int q = 0; q < C; ++q) {
      const int a = (int)((long long)n * q / C), b = (int)((long long)n * (q + 1) / C);
      launch_spmv_rows(c, k->m, a, b, xi.d, yo.d);
      if (yo.host) out_chunk(yo.host, yo.d, a, b);
    }
    launch_patch_any(c, f->f, xi.d, nullptr);
    for (int q = 0; q < C; ++q) {
      const int a = (int)((long long)n * q / C), b = (int)((long long)n * (q + 1) / C);
      vanka_gather_range(c, f->f, a, b, d.d);
      if (d.host) out_chunk(d.host, d.d, a, b);
    }
    SAG_CUDA(cudaStreamSynchronize(cs));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  }
}

extern "C" {

int sag_vanka_spmv(sag_ctx* ctx, const sag_vanka* f, const sag_matrix* k, const double* x,
                   double* delta, double* y) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    SAG_NOTNULL(k);
    auto& c = ctx->c;
    const int n = f->f.n;
    SAG_REQUIRE(k->m.nrows == n && k->m.ncols == n, SAG_DIMENSION_MISMATCH,
                "sag_vanka_spmv: operator and factorization sizes differ");
    // pinned host buffers: the staged pipeline when it applies. Unless
    // SAG_STEP_STAGES forces it, the first call on a plan times both forms
    // (each run is the whole step: same results) and keeps the faster one --
    // the gain depends on the operator and on the host link of the machine.
    StepPlan* P = vanka_step_prepare(c, f->f, k->m, x, delta, y);
    const char* forced = getenv("SAG_STEP_STAGES");
    if (P && forced && *forced) {
      vanka_spmv_pipelined(c, f->f, k->m, *P, x, delta, y);
      return;
    }
    if (P && P->choice == 0) {
      auto timed = [&](auto&& run) {
        double best = 1e30;
        for (int r = 0; r < 3; ++r) {
          const auto t0 = std::chrono::steady_clock::now();
          run();
          const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (r > 0) best = std::min(best, t);  // the first run warms up (graph capture)
        }
        return best;
      };
      P->t_plain = timed([&] { vanka_spmv_plain(c, f, k, x, delta, y); });
      P->t_pipe = timed([&] { vanka_spmv_pipelined(c, f->f, k->m, *P, x, delta, y); });
      P->choice = P->t_pipe < 0.98 * P->t_plain ? 1 : -1;
      return;
    }
    if (P && P->choice > 0) {
      vanka_spmv_pipelined(c, f->f, k->m, *P, x, delta, y);
      return;
    }
    vanka_spmv_plain(c, f, k, x, delta, y);
  });
}

int sag_vanka_step_plan(const sag_vanka* f, long long* out, int cap) {
  return guard([&] {
    SAG_NOTNULL(f);
    SAG_NOTNULL(out);
    long long v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (f->f.step_plan) {
      const StepPlan& P = *f->f.step_plan;
      v[0] = P.S;
      v[1] = P.ranges;
      v[6] = P.choice;
      v[7] = (long long)(1e9 * P.t_plain);
      v[8] = (long long)(1e9 * P.t_pipe);
      for (int q = 0; q < P.S; ++q) {
        v[2] += (long long)P.in[q].size();
        v[3] += (long long)P.rows[q].size();
        v[4] += (long long)P.gat[q].size();
        v[5] += (long long)P.pat[q].size();
      }
    }
    for (int i = 0; i < cap && i < 9; ++i) out[i] = v[i];
  });
}

int sag_apply_vanka_stage(sag_ctx* ctx, const sag_vanka* f, const double* r, double* delta,
                          int stage) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    SAG_REQUIRE(stage == 1 || stage == 2, SAG_CONFIG_ERROR, "stage must be 1 or 2");
    SAG_REQUIRE(is_device_ptr(r) && is_device_ptr(delta), SAG_INVALID_ARGUMENT,
                "sag_apply_vanka_stage takes device pointers");
    vanka_apply_stage(ctx->c, f->f, r, delta, stage);
  });
}


struct sag_vanka3 {
  sag::Vanka3 f;
  sag::Ctx* c = nullptr;
};

int sag_factor_patches3(sag_ctx* ctx, const sag_matrix* k, int n_x, int n_y, int n_z, int n_p,
                        sag_vanka3** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(k);
    SAG_NOTNULL(out);
    auto f = factor3_dev(ctx->c, k->m, n_x, n_y, n_z, n_p);
    auto* h = new sag_vanka3;
    h->f = std::move(*f);
    h->c = &ctx->c;
    *out = h;
  });
}

int sag_vanka3_destroy(sag_vanka3* f) {
  return guard([&] {
    if (f && f->c) cudaStreamSynchronize(f->c->stream);
    delete f;
  });
}

int sag_vanka3_stats(const sag_vanka3* f, long long* s) {
  return guard([&] {
    SAG_NOTNULL(f);
    SAG_NOTNULL(s);
    s[0] = f->f.npatch;
    s[1] = f->f.n;
    s[2] = f->f.blob_bytes;
    s[3] = f->f.max_nv;
    s[4] = f->f.nslots;
    s[5] = f->f.a_factor_bytes;
    s[6] = f->f.aux_bytes;
  });
}

int sag_apply_vanka3(sag_ctx* ctx, const sag_vanka3* f, const double* r, double* delta) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(f);
    auto& c = ctx->c;
    InVec ri(c, r, f->f.n, 0);
    OutVec d(c, delta, f->f.n, 1, false);
    apply3_dev(c, f->f, ri.d, d.d);
    d.finish();
  });
}
}  // extern "C"
