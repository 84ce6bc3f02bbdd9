// libsag FEM module: element assembly and Dirichlet elimination on the
// device, BITWISE equal to the reference:
//   from_triplets               sparse.cpp:43-66
//   assemble_taylor_hood        fem.cpp:354-450     (element loop :361-389)
//   assemble_scott_vogelius     fem.cpp:452-566     (element loop :464-498)
//   assemble_iso                fem.cpp:568-662     (element loop :578-605)
//   assemble_p1_stiffness/mass  fem.cpp:310-335
//   reduce_scalar/divergence    fem.cpp:207-266
//
// This translation unit is compiled with --fmad=false: every expression below
// rounds operation by operation, like the reference built with
// -ffp-contract=off (oracle/Makefile), so element values are the reference's
// bits.
//
// from_triplets sums duplicate (row, col) entries in the order std::sort
// leaves them, and std::sort is not stable. Its permutation is, however, a
// deterministic function of the key sequence alone (the comparator reads only
// (row, col)), so the device reproduces it: libstdc++'s introsort
// (__introsort_loop: median-of-three to the front, unguarded Hoare
// partition, recursion while a range holds > 16 elements, heapsort at the
// depth limit 2 floor(log2 n)) is run level by level over all open ranges at
// once -- a Hoare partition is data-parallel: the k-th element >= pivot from
// the left trades places with the k-th element <= pivot from the right while
// the first stays left of the second -- and the final insertion sort, which
// is stable, becomes a stable radix sort. Ranges that reach the depth limit
// (never seen on FEM key sequences) are heap-sorted by the host's own
// std::partial_sort. Each (row, col) run is then summed sequentially from 0.0
// in that order and exact zeros are dropped (sparse.cpp:51-61).
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <vector>

#include "internal.cuh"

namespace sag {

namespace {

constexpr int kIntroThreshold = 16;  // libstdc++ _S_threshold

__global__ void iota_kernel(long long n, int* a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

inline int grid_n(Ctx& c, long long n, int per = 256) {
  const long long g = (n + per - 1) / per;
  return (int)std::max(1LL, std::min(g, (long long)c.num_sms * 32));
}

struct Seg {
  int F, E, depth;
};

// __move_median_to_first(first, first+1, mid, last-1) and the pivot key; a
// range at the depth limit is set aside for the heap sort instead.
__global__ void seg_median_kernel(int S, Seg* segs, unsigned long long* K, int* I,
                                  unsigned long long* piv, int* headpos, int* seg_at, Seg* heap,
                                  int* nheap) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  Seg g = segs[s];
  if (g.depth == 0) {
    heap[atomicAdd(nheap, 1)] = g;
    segs[s].F = -1;  // inactive
    return;
  }
  const int F = g.F, E = g.E;
  const int a = F + 1, b = F + (E - F) / 2, c = E - 1;
  const unsigned long long ka = K[a], kb = K[b], kc = K[c];
  int m;
  if (ka < kb) {
    if (kb < kc) m = b;
    else if (ka < kc) m = c;
    else m = a;
  } else if (ka < kc) {
    m = a;
  } else if (kb < kc) {
    m = c;
  } else {
    m = b;
  }
  const unsigned long long kf = K[F], km = K[m];
  const int i_f = I[F], i_m = I[m];
  K[F] = km;
  K[m] = kf;
  I[F] = i_m;
  I[m] = i_f;
  piv[s] = km;
  headpos[F] = F + 1;
  seg_at[F] = s;
}

// per position: its open range (the nearest range start at or left of it)
// and the two candidate flags of the partition
__global__ void seg_flags_kernel(long long n, const int* __restrict__ mx,
                                 const int* __restrict__ seg_at, const Seg* __restrict__ segs,
                                 const unsigned long long* __restrict__ K,
                                 const unsigned long long* __restrict__ piv, int* fl, int* fr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int l = 0, r = 0;
    const int h = mx[i];
    if (h > 0) {
      const int s = seg_at[h - 1];
      const Seg g = segs[s];
      if (g.F >= 0 && i < g.E) {
        const unsigned long long p = piv[s], k = K[i];
        l = (i > g.F && k >= p) ? 1 : 0;  // stops `while (*first < pivot) ++first`
        r = (k <= p) ? 1 : 0;             // stops `while (pivot < *last) --last`
      }
    }
    fl[i] = l;
    fr[i] = r;
  }
}

struct SegCounts {
  int cl, cr;
};
__device__ __forceinline__ SegCounts seg_counts(const Seg& g, const int* sl, const int* sr) {
  SegCounts c;
  c.cl = sl[g.E - 1] - sl[g.F];
  c.cr = sr[g.E - 1] - (g.F > 0 ? sr[g.F - 1] : 0);
  return c;
}

// k-th left candidate (ascending) -> posl[F + k]; k-th right candidate
// (descending) -> posr[F + k]
__global__ void seg_pos_kernel(long long n, const int* __restrict__ mx,
                               const int* __restrict__ seg_at, const Seg* __restrict__ segs,
                               const int* __restrict__ fl, const int* __restrict__ fr,
                               const int* __restrict__ sl, const int* __restrict__ sr, int* posl,
                               int* posr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int h = mx[i];
    if (h <= 0) continue;
    const Seg g = segs[seg_at[h - 1]];
    if (g.F < 0 || i >= g.E) continue;
    if (fl[i]) posl[g.F + (sl[i] - 1 - sl[g.F])] = (int)i;
    if (fr[i]) posr[g.F + (sr[g.E - 1] - sr[i])] = (int)i;
  }
}

// pair k trades places when l_k < r_k; the pairs that do are a prefix, and
// the thread at its end records how many
__global__ void seg_swap_kernel(long long n, const int* __restrict__ mx,
                                const int* __restrict__ seg_at, const Seg* __restrict__ segs,
                                const int* __restrict__ sl, const int* __restrict__ sr,
                                const int* __restrict__ posl, const int* __restrict__ posr,
                                unsigned long long* K, int* I, int* nswap) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int h = mx[i];
    if (h <= 0) continue;
    const int s = seg_at[h - 1];
    const Seg g = segs[s];
    if (g.F < 0 || i >= g.E) continue;
    const SegCounts c = seg_counts(g, sl, sr);
    const int lim = min(c.cl, c.cr);
    const int k = (int)i - g.F;
    const bool v0 = k < lim && posl[g.F + k] < posr[g.F + k];
    const bool v1 = k + 1 < lim && posl[g.F + k + 1] < posr[g.F + k + 1];
    if (v0) {
      const int a = posl[g.F + k], b = posr[g.F + k];
      const unsigned long long ka = K[a];
      const int ia = I[a];
      K[a] = K[b];
      I[a] = I[b];
      K[b] = ka;
      I[b] = ia;
      if (!v1) nswap[s] = k + 1;
    } else if (k == 0) {
      nswap[s] = 0;
    }
  }
}

// the cut (the left scan's stop at the K-th step: min(l_K, r_{K-1})), the
// two sub-ranges with depth - 1, those longer than the threshold reopened
__global__ void seg_cut_kernel(int S, const Seg* segs, const int* sl, const int* sr,
                               const int* posl, const int* posr, const int* nswap, int* headpos,
                               Seg* next, int* nnext, int* bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const Seg g = segs[s];
  if (g.F < 0) return;
  headpos[g.F] = 0;
  const SegCounts c = seg_counts(g, sl, sr);
  const int Kp = nswap[s];
  int cut;
  if (Kp < c.cl) {
    cut = posl[g.F + Kp];
    if (Kp > 0) cut = min(cut, posr[g.F + Kp - 1]);
  } else if (Kp > 0) {
    cut = posr[g.F + Kp - 1];
  } else {
    *bad = 1;  // no element >= pivot right of it: impossible after median-of-three
    return;
  }
  if (cut - g.F > kIntroThreshold) next[atomicAdd(nnext, 1)] = Seg{g.F, cut, g.depth - 1};
  if (g.E - cut > kIntroThreshold) next[atomicAdd(nnext, 1)] = Seg{cut, g.E, g.depth - 1};
}

template <class T>
struct HostPair {
  unsigned long long k;
  T i;
};

}  // namespace

// std::sort's permutation of the key sequence K (in place): on return K is
// sorted and I holds, for each position, the original index of the element
// libstdc++'s std::sort (with a comparator reading only the key) puts there.
int sort_like_std(Ctx& c, long long n, unsigned long long* K, int* I) {
  SAG_REQUIRE(n < (1LL << 31) - 1, SAG_DIMENSION_MISMATCH, "from_triplets: too many triplets");
  if (n <= 1) return 0;
  int nh = 0;
  int depth0 = 0;
  for (long long v = n; v > 1; v >>= 1) ++depth0;  // std::__lg(n)
  depth0 *= 2;
  if (n > kIntroThreshold) {
    const long long segcap = 2 * (n / (kIntroThreshold + 1)) + 4;
    DevBuf<Seg> sa(segcap), sb(segcap), heap(segcap);
    DevBuf<unsigned long long> piv(segcap);
    DevBuf<int> nswap(segcap), cnt(4);
    DevBuf<int> headpos(n), mx(n), seg_at(n), fl(n), fr(n), sl(n), sr(n), posl(n), posr(n);
    SAG_CUDA(cudaMemsetAsync(headpos.p, 0, sizeof(int) * n, c.stream));
    SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * 4, c.stream));  // [nnext, nheap, bad]
    Seg root{0, (int)n, depth0};
    SAG_CUDA(cudaMemcpyAsync(sa.p, &root, sizeof(Seg), cudaMemcpyHostToDevice, c.stream));
    size_t t1 = 0, t2 = 0;
    SAG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, t1, headpos.p, mx.p, cub::Max(), (int)n,
                                            c.stream));
    SAG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t2, fl.p, sl.p, (int)n, c.stream));
    DevBuf<unsigned char> ws(std::max(t1, t2));
    int S = 1;
    Seg* cur = sa.p;
    Seg* nxt = sb.p;
    const int g = grid_n(c, n);
    while (S > 0) {
      SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), c.stream));
      seg_median_kernel<<<(S + 255) / 256, 256, 0, c.stream>>>(S, cur, K, I, piv.p, headpos.p,
                                                               seg_at.p, heap.p, cnt.p + 1);
      SAG_LAUNCHED(c);
      SAG_CUDA(cub::DeviceScan::InclusiveScan(ws.p, t1, headpos.p, mx.p, cub::Max(), (int)n,
                                              c.stream));
      seg_flags_kernel<<<g, 256, 0, c.stream>>>(n, mx.p, seg_at.p, cur, K, piv.p, fl.p, fr.p);
      SAG_LAUNCHED(c);
      SAG_CUDA(cub::DeviceScan::InclusiveSum(ws.p, t2, fl.p, sl.p, (int)n, c.stream));
      SAG_CUDA(cub::DeviceScan::InclusiveSum(ws.p, t2, fr.p, sr.p, (int)n, c.stream));
      seg_pos_kernel<<<g, 256, 0, c.stream>>>(n, mx.p, seg_at.p, cur, fl.p, fr.p, sl.p, sr.p,
                                              posl.p, posr.p);
      SAG_LAUNCHED(c);
      seg_swap_kernel<<<g, 256, 0, c.stream>>>(n, mx.p, seg_at.p, cur, sl.p, sr.p, posl.p,
                                               posr.p, K, I, nswap.p);
      SAG_LAUNCHED(c);
      seg_cut_kernel<<<(S + 255) / 256, 256, 0, c.stream>>>(S, cur, sl.p, sr.p, posl.p, posr.p,
                                                            nswap.p, headpos.p, nxt, cnt.p,
                                                            cnt.p + 2);
      SAG_LAUNCHED(c);
      int h[3];
      SAG_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(int) * 3, cudaMemcpyDeviceToHost, c.stream));
      SAG_CUDA(cudaStreamSynchronize(c.stream));
      SAG_REQUIRE(h[2] == 0, SAG_ERROR, "from_triplets: partition without a right sentinel");
      S = h[0];
      std::swap(cur, nxt);
    }
    // ranges at the depth limit: std::partial_sort(first, last, last) (the
    // heap sort of __introsort_loop) by the host's own libstdc++
    SAG_CUDA(cudaMemcpyAsync(&nh, cnt.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
    if (nh > 0) {
      std::vector<Seg> hs(nh);
      SAG_CUDA(cudaMemcpy(hs.data(), heap.p, sizeof(Seg) * nh, cudaMemcpyDeviceToHost));
      for (const Seg& s : hs) {
        const int len = s.E - s.F;
        std::vector<unsigned long long> k(len);
        std::vector<int> ix(len);
        SAG_CUDA(cudaMemcpy(k.data(), K + s.F, 8 * len, cudaMemcpyDeviceToHost));
        SAG_CUDA(cudaMemcpy(ix.data(), I + s.F, 4 * len, cudaMemcpyDeviceToHost));
        std::vector<HostPair<int>> v(len);
        for (int q = 0; q < len; ++q) v[q] = {k[q], ix[q]};
        std::partial_sort(v.begin(), v.end(), v.end(),
                          [](const HostPair<int>& a, const HostPair<int>& b) { return a.k < b.k; });
        for (int q = 0; q < len; ++q) {
          k[q] = v[q].k;
          ix[q] = v[q].i;
        }
        SAG_CUDA(cudaMemcpy(K + s.F, k.data(), 8 * len, cudaMemcpyHostToDevice));
        SAG_CUDA(cudaMemcpy(I + s.F, ix.data(), 4 * len, cudaMemcpyHostToDevice));
      }
    }
  }
  // __final_insertion_sort: stable, so = a stable sort of what the loop left
  DevBuf<unsigned long long> K2(n);
  DevBuf<int> I2(n);
  size_t t = 0;
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t, K, K2.p, I, I2.p, (int)n, 0, 64, c.stream));
  DevBuf<unsigned char> ws(std::max<size_t>(t, 1));
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, t, K, K2.p, I, I2.p, (int)n, 0, 64, c.stream));
  SAG_CUDA(cudaMemcpyAsync(K, K2.p, 8 * n, cudaMemcpyDeviceToDevice, c.stream));
  SAG_CUDA(cudaMemcpyAsync(I, I2.p, 4 * n, cudaMemcpyDeviceToDevice, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  return nh;
}

namespace {

__global__ void run_head_kernel(long long n, const unsigned long long* __restrict__ K,
                                int* head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || K[i] != K[i - 1]) ? 1 : 0;
}

// one (row, col) run: sum = 0.0; sum += value in the sorted order
// (sparse.cpp:50-55); kept when sum != 0.0 (:56-60)
__global__ void run_sum_kernel(int R, long long n, const int* __restrict__ starts,
                               const unsigned long long* __restrict__ K,
                               const int* __restrict__ I, const double* __restrict__ val,
                               int* keep, double* sum_out, int* rows, int* cols, int* rowcnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const long long s = starts[r], e = r + 1 < R ? starts[r + 1] : n;
    double sum = 0.0;
    for (long long j = s; j < e; ++j) sum += val[I[j]];
    const unsigned long long k = K[s];
    const int row = (int)(k >> 32), col = (int)(k & 0xffffffffu);
    keep[r] = sum != 0.0 ? 1 : 0;
    sum_out[r] = sum;
    rows[r] = row;
    cols[r] = col;
    if (sum != 0.0) atomicAdd(rowcnt + row, 1);
  }
}

}  // namespace

// from_triplets (sparse.cpp:43-66) of n triplets given by their keys
// (row << 32 | col) and values in generation order.
std::unique_ptr<Matrix> from_triplets_dev(Ctx& c, int nrows, int ncols, long long n,
                                          const unsigned long long* keys, const double* vals) {
  DevBuf<int> rowcnt(nrows + 1);
  SAG_CUDA(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * (nrows + 1), c.stream));
  if (n == 0) {
    std::vector<int> rp(nrows + 1, 0);
    return matrix_upload(c, nrows, ncols, 0, rp.data(), nullptr, nullptr);
  }
  DevBuf<unsigned long long> K(n);
  DevBuf<int> I(n);
  SAG_CUDA(cudaMemcpyAsync(K.p, keys, 8 * n, cudaMemcpyDeviceToDevice, c.stream));
  iota_kernel<<<grid_n(c, n), 256, 0, c.stream>>>(n, I.p);
  SAG_LAUNCHED(c);
  sort_like_std(c, n, K.p, I.p);
  // runs of equal keys
  DevBuf<int> head(n), idx(n), starts(n), nrun(1);
  run_head_kernel<<<grid_n(c, n), 256, 0, c.stream>>>(n, K.p, head.p);
  SAG_LAUNCHED(c);
  iota_kernel<<<grid_n(c, n), 256, 0, c.stream>>>(n, idx.p);
  SAG_LAUNCHED(c);
  size_t t = 0;
  SAG_CUDA(cub::DeviceSelect::Flagged(nullptr, t, idx.p, head.p, starts.p, nrun.p, (int)n,
                                      c.stream));
  DevBuf<unsigned char> ws(std::max<size_t>(t, 1));
  SAG_CUDA(cub::DeviceSelect::Flagged(ws.p, t, idx.p, head.p, starts.p, nrun.p, (int)n,
                                      c.stream));
  int R = 0;
  SAG_CUDA(cudaMemcpyAsync(&R, nrun.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  DevBuf<int> keep(R), rows(R), cols(R), ci(R), nkeep(1);
  DevBuf<double> sums(R), v(R);
  run_sum_kernel<<<grid_n(c, R), 256, 0, c.stream>>>(R, n, starts.p, K.p, I.p, vals, keep.p,
                                                     sums.p, rows.p, cols.p, rowcnt.p);
  SAG_LAUNCHED(c);
  // the kept runs in sorted order are the CSR entries
  size_t t2 = 0, t3 = 0, t4 = 0;
  SAG_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, cols.p, keep.p, ci.p, nkeep.p, R, c.stream));
  SAG_CUDA(cub::DeviceSelect::Flagged(nullptr, t4, sums.p, keep.p, v.p, nkeep.p, R, c.stream));
  DevBuf<int> rp(nrows + 1);
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, rowcnt.p, rp.p, nrows + 1, c.stream));
  DevBuf<unsigned char> ws2(std::max<size_t>(std::max(std::max(t2, t3), t4), 1));
  SAG_CUDA(cub::DeviceSelect::Flagged(ws2.p, t2, cols.p, keep.p, ci.p, nkeep.p, R, c.stream));
  SAG_CUDA(cub::DeviceSelect::Flagged(ws2.p, t4, sums.p, keep.p, v.p, nkeep.p, R, c.stream));
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws2.p, t3, rowcnt.p, rp.p, nrows + 1, c.stream));
  int nnz = 0;
  SAG_CUDA(cudaMemcpyAsync(&nnz, nkeep.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  return matrix_upload(c, nrows, ncols, nnz, rp.p, ci.p, v.p);
}

// ---------------------------------------------------------------- elements --
namespace {

// tri_quadrature (fem.cpp:21-36): degree-4 rule, barycentric points
struct Quad6 {
  double l[6][3];
  double w[6];
};
__device__ __forceinline__ Quad6 tri_quad() {
  const double a1 = 0.445948490915965;
  const double w1 = 0.223381589678011;
  const double a2 = 0.091576213509771;
  const double w2 = 0.109951743655322;
  const double b1 = 1 - 2 * a1, b2 = 1 - 2 * a2;
  Quad6 q = {{{a1, a1, b1}, {a1, b1, a1}, {b1, a1, a1}, {a2, a2, b2}, {a2, b2, a2}, {b2, a2, a2}},
             {w1, w1, w1, w2, w2, w2}};
  return q;
}

// tri_geometry (fem.cpp:57-71)
struct Geo {
  double area;
  double gl[3][2];
};
__device__ __forceinline__ Geo tri_geo(const double* __restrict__ vx, const int* tri) {
  const double ax = vx[2 * tri[0]], ay = vx[2 * tri[0] + 1];
  const double bx = vx[2 * tri[1]], by = vx[2 * tri[1] + 1];
  const double cx = vx[2 * tri[2]], cy = vx[2 * tri[2] + 1];
  const double twoA = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  Geo g;
  g.area = 0.5 * twoA;
  g.gl[0][0] = (by - cy) / twoA;
  g.gl[0][1] = (cx - bx) / twoA;
  g.gl[1][0] = (cy - ay) / twoA;
  g.gl[1][1] = (ax - cx) / twoA;
  g.gl[2][0] = (ay - by) / twoA;
  g.gl[2][1] = (bx - ax) / twoA;
  return g;
}

__device__ __forceinline__ unsigned long long key_of(int r, int c) {
  return ((unsigned long long)(unsigned)r << 32) | (unsigned)c;
}

// One (triangle, quadrature point) of the P2 element loop (fem.cpp:361-389 TH,
// :464-487 SV): 36 A triplets, 36 B triplets (x then y per (k, j)) and the
// load contributions, each at its position in the reference's push order.
__global__ void p2_element_kernel(int nt, int nv, int n_s, int sv, const double* __restrict__ vx,
                                  const int* __restrict__ tris, const int* __restrict__ tedges,
                                  const double* __restrict__ fq, unsigned long long* akey,
                                  double* aval, unsigned long long* bkey, double* bval,
                                  int* fdof, double* fxv, double* fyv) {
  const long long total = (long long)nt * 6;
  for (long long tq = blockIdx.x * (long long)blockDim.x + threadIdx.x; tq < total;
       tq += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(tq / 6), qi = (int)(tq % 6);
    const int* tri = tris + 3 * t;
    const Geo g = tri_geo(vx, tri);
    int dofs[6];
    for (int k = 0; k < 3; ++k) dofs[k] = tri[k];
    for (int k = 0; k < 3; ++k) dofs[3 + k] = nv + tedges[3 * t + k];
    const Quad6 Q = tri_quad();
    const double* l = Q.l[qi];
    const double w = Q.w[qi] * g.area;
    // p2_gradients (fem.cpp:92-104)
    double dn[6][2];
    for (int i = 0; i < 3; ++i) {
      dn[i][0] = (4 * l[i] - 1) * g.gl[i][0];
      dn[i][1] = (4 * l[i] - 1) * g.gl[i][1];
    }
    for (int i = 0; i < 3; ++i) {
      const int p = (i + 1) % 3, q = (i + 2) % 3;
      dn[3 + i][0] = 4 * (l[p] * g.gl[q][0] + l[q] * g.gl[p][0]);
      dn[3 + i][1] = 4 * (l[p] * g.gl[q][1] + l[q] * g.gl[p][1]);
    }
    const long long ab = tq * 36;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        akey[ab + i * 6 + j] = key_of(dofs[i], dofs[j]);
        aval[ab + i * 6 + j] = w * (dn[i][0] * dn[j][0] + dn[i][1] * dn[j][1]);
      }
    const long long bb = tq * 36;
    for (int k = 0; k < 3; ++k) {
      const int pr = sv ? 3 * t + k : tri[k];
      for (int j = 0; j < 6; ++j) {
        const long long e = bb + k * 12 + 2 * j;
        bkey[e] = key_of(pr, dofs[j]);
        bval[e] = -w * l[k] * dn[j][0];
        bkey[e + 1] = key_of(pr, n_s + dofs[j]);
        bval[e + 1] = -w * l[k] * dn[j][1];
      }
    }
    if (fq) {
      // p2_values (fem.cpp:84-89); fx[dofs[j]] += w * n[j] * f[0] (:382-387)
      double nn[6];
      for (int i = 0; i < 3; ++i) nn[i] = l[i] * (2 * l[i] - 1);
      for (int i = 0; i < 3; ++i) nn[3 + i] = 4 * l[(i + 1) % 3] * l[(i + 2) % 3];
      const double f0 = fq[2 * tq], f1 = fq[2 * tq + 1];
      for (int j = 0; j < 6; ++j) {
        fdof[tq * 6 + j] = dofs[j];
        fxv[tq * 6 + j] = w * nn[j] * f0;
        fyv[tq * 6 + j] = w * nn[j] * f1;
      }
    }
  }
}

// Per-element P1 pieces: stiffness (fem.cpp:310-323) / ISO A (:583-590) and
// mass (:325-335) / SV Mp, M_mix (:490-496), areas; ISO B (:593-598).
__global__ void p1_element_kernel(int nt, int nvf, const double* __restrict__ vx,
                                  const int* __restrict__ tris, int want,
                                  unsigned long long* skey, double* sval, unsigned long long* mkey,
                                  double* mval, unsigned long long* xkey, double* xval,
                                  double* areas, unsigned long long* bkey, double* bval) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int* tri = tris + 3 * t;
    const Geo g = tri_geo(vx, tri);
    if (want & 1)  // stiffness
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          skey[9LL * t + 3 * i + j] = key_of(tri[i], tri[j]);
          sval[9LL * t + 3 * i + j] =
              g.area * (g.gl[i][0] * g.gl[j][0] + g.gl[i][1] * g.gl[j][1]);
        }
    if (want & 2)  // P1 mass: signed_area (mesh.cpp:35-41) / 12 * (2 or 1)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          mkey[9LL * t + 3 * i + j] = key_of(tri[i], tri[j]);
          mval[9LL * t + 3 * i + j] = g.area / 12.0 * (i == j ? 2.0 : 1.0);
        }
    if (want & 4)  // SV: element mass (3t+i, 3t+j), mixed mass (tri[i], 3t+j), areas
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double v = g.area / 12.0 * (i == j ? 2.0 : 1.0);
          mkey[9LL * t + 3 * i + j] = key_of(3 * t + i, 3 * t + j);
          mval[9LL * t + 3 * i + j] = v;
          xkey[9LL * t + 3 * i + j] = key_of(tri[i], 3 * t + j);
          xval[9LL * t + 3 * i + j] = v;
        }
    if (want & 4) areas[t] = g.area;
    if (want & 8)  // ISO divergence against the fine P1 pressure (one-third rule)
      for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) {
          const long long e = (3LL * t + k) * 6 + 2 * j;
          bkey[e] = key_of(tri[k], tri[j]);
          bval[e] = -g.area / 3.0 * g.gl[j][0];
          bkey[e + 1] = key_of(tri[k], nvf + tri[j]);
          bval[e + 1] = -g.area / 3.0 * g.gl[j][1];
        }
  }
}

// ISO load (fem.cpp:599-608): fx[tri[j]] += w * lambda_j * f[0]
__global__ void iso_load_kernel(int nt, const double* __restrict__ vx, const int* __restrict__ tris,
                                const double* __restrict__ fq, int* fdof, double* fxv,
                                double* fyv) {
  const long long total = (long long)nt * 6;
  for (long long tq = blockIdx.x * (long long)blockDim.x + threadIdx.x; tq < total;
       tq += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(tq / 6), qi = (int)(tq % 6);
    const int* tri = tris + 3 * t;
    const Geo g = tri_geo(vx, tri);
    const Quad6 Q = tri_quad();
    const double w = Q.w[qi] * g.area;
    const double f0 = fq[2 * tq], f1 = fq[2 * tq + 1];
    for (int j = 0; j < 3; ++j) {
      fdof[tq * 3 + j] = tri[j];
      fxv[tq * 3 + j] = w * Q.l[qi][j] * f0;
      fyv[tq * 3 + j] = w * Q.l[qi][j] * f1;
    }
  }
}

// a load vector: per dof, its contributions summed from 0.0 in generation
// order (a stable sort by dof keeps that order within a dof)
__global__ void load_sum_kernel(long long m, const int* __restrict__ dof_sorted,
                                const int* __restrict__ idx_sorted, const double* __restrict__ fx,
                                const double* __restrict__ fy, double* ox, double* oy) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = dof_sorted[i];
    if (i > 0 && dof_sorted[i - 1] == d) continue;  // not the run's first
    double sx = 0.0, sy = 0.0;
    for (long long j = i; j < m && dof_sorted[j] == d; ++j) {
      sx += fx[idx_sorted[j]];
      sy += fy[idx_sorted[j]];
    }
    ox[d] = sx;
    oy[d] = sy;
  }
}

void load_vector(Ctx& c, long long m, const int* dof, const double* fxv, const double* fyv, int n,
                 double* ox, double* oy) {
  SAG_CUDA(cudaMemsetAsync(ox, 0, sizeof(double) * n, c.stream));
  SAG_CUDA(cudaMemsetAsync(oy, 0, sizeof(double) * n, c.stream));
  if (m == 0) return;
  DevBuf<int> idx(m), idx2(m), dof2(m);
  iota_kernel<<<grid_n(c, m), 256, 0, c.stream>>>(m, idx.p);
  SAG_LAUNCHED(c);
  size_t t = 0;
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t, dof, dof2.p, idx.p, idx2.p, (int)m, 0, 32,
                                           c.stream));
  DevBuf<unsigned char> ws(std::max<size_t>(t, 1));
  SAG_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, t, dof, dof2.p, idx.p, idx2.p, (int)m, 0, 32,
                                           c.stream));
  load_sum_kernel<<<grid_n(c, m), 256, 0, c.stream>>>(m, dof2.p, idx2.p, fxv, fyv, ox, oy);
  SAG_LAUNCHED(c);
}

template <class T>
DevBuf<T> upload(Ctx& c, const T* h, size_t n) {
  DevBuf<T> d(std::max<size_t>(n, 1));
  if (n) SAG_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * n, cudaMemcpyDefault, c.stream));
  return d;
}

// reduce_scalar (fem.cpp:207-229): kept rows / columns renumbered, the
// eliminated columns' A g summed into the lifts in column order
__global__ void reduce_scalar_count_kernel(int n, const int* __restrict__ rp,
                                           const int* __restrict__ ci, const int* __restrict__ o2n,
                                           int* cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int rn = o2n[r];
    if (rn < 0) continue;
    int k = 0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) k += o2n[ci[q]] >= 0;
    cnt[rn] = k;
  }
}
__global__ void reduce_scalar_fill_kernel(int n, const int* __restrict__ rp,
                                          const int* __restrict__ ci, const double* __restrict__ v,
                                          const int* __restrict__ o2n, const double* __restrict__ gx,
                                          const double* __restrict__ gy, const int* __restrict__ orp,
                                          int* oci, double* ov, double* lx, double* ly) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int rn = o2n[r];
    if (rn < 0) continue;
    int o = orp[rn];
    double sx = 0.0, sy = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      const int cn = o2n[ci[q]];
      if (cn >= 0) {
        oci[o] = cn;
        ov[o] = v[q];
        ++o;
      } else {
        sx += v[q] * gx[ci[q]];
        sy += v[q] * gy[ci[q]];
      }
    }
    lx[rn] = sx;
    ly[rn] = sy;
  }
}

// reduce_divergence (fem.cpp:233-252): columns [x | y] of scalar width n_s
__global__ void reduce_div_count_kernel(int nr, int n_s, const int* __restrict__ rp,
                                        const int* __restrict__ ci, const int* __restrict__ o2n,
                                        int* cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    int k = 0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) k += o2n[ci[q] % n_s] >= 0;
    cnt[r] = k;
  }
}
__global__ void reduce_div_fill_kernel(int nr, int n_s, int ns_red, const int* __restrict__ rp,
                                       const int* __restrict__ ci, const double* __restrict__ v,
                                       const int* __restrict__ o2n, const double* __restrict__ gx,
                                       const double* __restrict__ gy, const int* __restrict__ orp,
                                       int* oci, double* ov, double* rhs_p) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    int o = orp[r];
    double s = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      const int c = ci[q], comp = c / n_s, sc = c % n_s, cn = o2n[sc];
      if (cn >= 0) {
        oci[o] = comp * ns_red + cn;
        ov[o] = v[q];
        ++o;
      } else {
        s -= v[q] * (comp == 0 ? gx[sc] : gy[sc]);
      }
    }
    rhs_p[r] = s;
  }
}

template <class Count, class Fill>
std::unique_ptr<Matrix> csr_build(Ctx& c, int nrows, int ncols, Count count, Fill fill) {
  DevBuf<int> cnt(nrows + 1), rp(nrows + 1);
  SAG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (nrows + 1), c.stream));
  count(cnt.p);
  size_t t = 0;
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t, cnt.p, rp.p, nrows + 1, c.stream));
  DevBuf<unsigned char> ws(std::max<size_t>(t, 1));
  SAG_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, t, cnt.p, rp.p, nrows + 1, c.stream));
  int nnz = 0;
  SAG_CUDA(cudaMemcpyAsync(&nnz, rp.p + nrows, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SAG_CUDA(cudaStreamSynchronize(c.stream));
  DevBuf<int> ci(std::max(nnz, 1));
  DevBuf<double> v(std::max(nnz, 1));
  fill(rp.p, ci.p, v.p);
  return matrix_upload(c, nrows, ncols, nnz, rp.p, ci.p, v.p);
}

}  // namespace

}  // namespace sag

// =================================================================== C-ABI
using namespace sag;

namespace {
sag_matrix* wrap_m(std::unique_ptr<Matrix> m) {
  auto* h = new sag_matrix;
  h->m = std::move(*m);
  return h;
}
void check_mesh(const sag_mesh2d* m) {
  SAG_NOTNULL(m);
  SAG_REQUIRE(m->num_vertices >= 0 && m->num_triangles >= 0 && m->num_edges >= 0,
              SAG_DIMENSION_MISMATCH, "mesh: negative size");
  SAG_REQUIRE(m->num_triangles == 0 || (m->vertices && m->triangles), SAG_INVALID_ARGUMENT,
              "mesh: null array");
}
}  // namespace

extern "C" {

int sag_from_triplets(sag_ctx* ctx, int nrows, int ncols, long long n, const int* rows,
                      const int* cols, const double* values, sag_matrix** out) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(out);
    SAG_REQUIRE(nrows >= 0 && ncols >= 0 && n >= 0, SAG_DIMENSION_MISMATCH,
                "from_triplets: negative size");
    Ctx& c = ctx->c;
    std::vector<unsigned long long> hk(n);
    std::vector<int> hr(n), hc(n);
    if (n) {
      SAG_NOTNULL(rows);
      SAG_NOTNULL(cols);
      SAG_NOTNULL(values);
      SAG_CUDA(cudaMemcpy(hr.data(), rows, 4 * n, cudaMemcpyDefault));
      SAG_CUDA(cudaMemcpy(hc.data(), cols, 4 * n, cudaMemcpyDefault));
    }
    for (long long i = 0; i < n; ++i) {
      SAG_REQUIRE(hr[i] >= 0 && hr[i] < nrows && hc[i] >= 0 && hc[i] < ncols,
                  SAG_DIMENSION_MISMATCH, "from_triplets: index out of range");
      hk[i] = ((unsigned long long)(unsigned)hr[i] << 32) | (unsigned)hc[i];
    }
    DevBuf<unsigned long long> k = upload(c, hk.data(), n);
    DevBuf<double> v = upload(c, values, n);
    *out = wrap_m(from_triplets_dev(c, nrows, ncols, n, k.p, v.p));
  });
}

int sag_sort_permutation(sag_ctx* ctx, long long n, const unsigned long long* keys, int* perm,
                         int* heap_ranges) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    Ctx& c = ctx->c;
    if (heap_ranges) *heap_ranges = 0;
    if (n <= 0) return;
    SAG_NOTNULL(keys);
    SAG_NOTNULL(perm);
    DevBuf<unsigned long long> K = upload(c, keys, n);
    DevBuf<int> I(n);
    iota_kernel<<<grid_n(c, n), 256, 0, c.stream>>>(n, I.p);
    SAG_LAUNCHED(c);
    const int nh = sort_like_std(c, n, K.p, I.p);
    if (heap_ranges) *heap_ranges = nh;
    SAG_CUDA(cudaMemcpy(perm, I.p, 4 * n, cudaMemcpyDefault));
  });
}

int sag_assemble_p2(sag_ctx* ctx, const sag_mesh2d* mesh, int sv, const double* force_qp,
                    sag_matrix** a_full, sag_matrix** b_full, double* fx, double* fy,
                    sag_matrix** mp, sag_matrix** m_mix, double* areas) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    check_mesh(mesh);
    SAG_NOTNULL(a_full);
    SAG_NOTNULL(b_full);
    SAG_REQUIRE(mesh->tri_edges || mesh->num_triangles == 0, SAG_INVALID_ARGUMENT,
                "assemble_p2: mesh has no edge table");
    Ctx& c = ctx->c;
    const int nv = mesh->num_vertices, nt = mesh->num_triangles;
    const int n_s = nv + mesh->num_edges;
    const int n_p = sv ? 3 * nt : nv;
    DevBuf<double> vx = upload(c, mesh->vertices, 2 * (size_t)nv);
    DevBuf<int> tr = upload(c, mesh->triangles, 3 * (size_t)nt);
    DevBuf<int> te = upload(c, mesh->tri_edges, 3 * (size_t)nt);
    const long long ntq = 6LL * nt;
    DevBuf<unsigned long long> ak(36 * ntq), bk(36 * ntq);
    DevBuf<double> av(36 * ntq), bv(36 * ntq);
    DevBuf<double> fq;
    DevBuf<int> fdof;
    DevBuf<double> fxv, fyv;
    if (force_qp) {
      fq = upload(c, force_qp, 2 * (size_t)ntq);
      fdof.alloc(6 * ntq);
      fxv.alloc(6 * ntq);
      fyv.alloc(6 * ntq);
    }
    p2_element_kernel<<<grid_n(c, ntq, 128), 128, 0, c.stream>>>(
        nt, nv, n_s, sv ? 1 : 0, vx.p, tr.p, te.p, force_qp ? fq.p : nullptr, ak.p, av.p, bk.p,
        bv.p, fdof.p, fxv.p, fyv.p);
    SAG_LAUNCHED(c);
    *a_full = wrap_m(from_triplets_dev(c, n_s, n_s, 36 * ntq, ak.p, av.p));
    ak.reset();
    av.reset();
    *b_full = wrap_m(from_triplets_dev(c, n_p, 2 * n_s, 36 * ntq, bk.p, bv.p));
    bk.reset();
    bv.reset();
    if (fx && fy) {
      DevBuf<double> ox(n_s), oy(n_s);
      if (force_qp) {
        load_vector(c, 6 * ntq, fdof.p, fxv.p, fyv.p, n_s, ox.p, oy.p);
      } else {
        SAG_CUDA(cudaMemsetAsync(ox.p, 0, sizeof(double) * n_s, c.stream));
        SAG_CUDA(cudaMemsetAsync(oy.p, 0, sizeof(double) * n_s, c.stream));
      }
      SAG_CUDA(cudaMemcpyAsync(fx, ox.p, sizeof(double) * n_s, cudaMemcpyDefault, c.stream));
      SAG_CUDA(cudaMemcpyAsync(fy, oy.p, sizeof(double) * n_s, cudaMemcpyDefault, c.stream));
    }
    if (sv && (mp || m_mix || areas)) {
      DevBuf<unsigned long long> mk(9LL * nt), xk(9LL * nt);
      DevBuf<double> mv(9LL * nt), xv(9LL * nt), ar(nt);
      p1_element_kernel<<<grid_n(c, nt, 128), 128, 0, c.stream>>>(
          nt, 0, vx.p, tr.p, 4, nullptr, nullptr, mk.p, mv.p, xk.p, xv.p, ar.p, nullptr, nullptr);
      SAG_LAUNCHED(c);
      if (mp) *mp = wrap_m(from_triplets_dev(c, n_p, n_p, 9LL * nt, mk.p, mv.p));
      if (m_mix) *m_mix = wrap_m(from_triplets_dev(c, nv, n_p, 9LL * nt, xk.p, xv.p));
      if (areas) SAG_CUDA(cudaMemcpyAsync(areas, ar.p, sizeof(double) * nt, cudaMemcpyDefault, c.stream));
    }
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_assemble_p1(sag_ctx* ctx, const sag_mesh2d* mesh, sag_matrix** stiffness,
                    sag_matrix** mass) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    check_mesh(mesh);
    Ctx& c = ctx->c;
    const int nv = mesh->num_vertices, nt = mesh->num_triangles;
    DevBuf<double> vx = upload(c, mesh->vertices, 2 * (size_t)nv);
    DevBuf<int> tr = upload(c, mesh->triangles, 3 * (size_t)nt);
    DevBuf<unsigned long long> sk(9LL * nt), mk(9LL * nt);
    DevBuf<double> sv(9LL * nt), mv(9LL * nt);
    p1_element_kernel<<<grid_n(c, nt, 128), 128, 0, c.stream>>>(
        nt, 0, vx.p, tr.p, (stiffness ? 1 : 0) | (mass ? 2 : 0), sk.p, sv.p, mk.p, mv.p, nullptr,
        nullptr, nullptr, nullptr, nullptr);
    SAG_LAUNCHED(c);
    if (stiffness) *stiffness = wrap_m(from_triplets_dev(c, nv, nv, 9LL * nt, sk.p, sv.p));
    if (mass) *mass = wrap_m(from_triplets_dev(c, nv, nv, 9LL * nt, mk.p, mv.p));
  });
}

int sag_assemble_iso(sag_ctx* ctx, const sag_mesh2d* fine, const double* force_qp,
                     sag_matrix** a_full, sag_matrix** b_fine, double* fx, double* fy) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    check_mesh(fine);
    SAG_NOTNULL(a_full);
    SAG_NOTNULL(b_fine);
    Ctx& c = ctx->c;
    const int nvf = fine->num_vertices, nt = fine->num_triangles;
    DevBuf<double> vx = upload(c, fine->vertices, 2 * (size_t)nvf);
    DevBuf<int> tr = upload(c, fine->triangles, 3 * (size_t)nt);
    DevBuf<unsigned long long> sk(9LL * nt), bk(18LL * nt);
    DevBuf<double> sv(9LL * nt), bv(18LL * nt);
    p1_element_kernel<<<grid_n(c, nt, 128), 128, 0, c.stream>>>(
        nt, nvf, vx.p, tr.p, 1 | 8, sk.p, sv.p, nullptr, nullptr, nullptr, nullptr, nullptr, bk.p,
        bv.p);
    SAG_LAUNCHED(c);
    *a_full = wrap_m(from_triplets_dev(c, nvf, nvf, 9LL * nt, sk.p, sv.p));
    *b_fine = wrap_m(from_triplets_dev(c, nvf, 2 * nvf, 18LL * nt, bk.p, bv.p));
    if (fx && fy) {
      DevBuf<double> ox(nvf), oy(nvf);
      if (force_qp) {
        const long long ntq = 6LL * nt;
        DevBuf<double> fq = upload(c, force_qp, 2 * (size_t)ntq);
        DevBuf<int> fdof(3 * ntq);
        DevBuf<double> fxv(3 * ntq), fyv(3 * ntq);
        iso_load_kernel<<<grid_n(c, ntq, 128), 128, 0, c.stream>>>(nt, vx.p, tr.p, fq.p, fdof.p,
                                                                   fxv.p, fyv.p);
        SAG_LAUNCHED(c);
        load_vector(c, 3 * ntq, fdof.p, fxv.p, fyv.p, nvf, ox.p, oy.p);
      } else {
        SAG_CUDA(cudaMemsetAsync(ox.p, 0, sizeof(double) * nvf, c.stream));
        SAG_CUDA(cudaMemsetAsync(oy.p, 0, sizeof(double) * nvf, c.stream));
      }
      SAG_CUDA(cudaMemcpyAsync(fx, ox.p, sizeof(double) * nvf, cudaMemcpyDefault, c.stream));
      SAG_CUDA(cudaMemcpyAsync(fy, oy.p, sizeof(double) * nvf, cudaMemcpyDefault, c.stream));
    }
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int sag_reduce_dirichlet(sag_ctx* ctx, const sag_matrix* a_full, const sag_matrix* b_full,
                         int n_s, const int* old_to_new, const double* gx, const double* gy,
                         sag_matrix** a_red, sag_matrix** b_red, double* lift_x, double* lift_y,
                         double* rhs_p) {
  return guard([&] {
    SAG_NOTNULL(ctx);
    SAG_NOTNULL(a_full);
    SAG_NOTNULL(b_full);
    SAG_NOTNULL(old_to_new);
    SAG_NOTNULL(gx);
    SAG_NOTNULL(gy);
    SAG_NOTNULL(a_red);
    SAG_NOTNULL(b_red);
    Ctx& c = ctx->c;
    const Matrix& A = a_full->m;
    const Matrix& B = b_full->m;
    SAG_REQUIRE(A.nrows == n_s && A.ncols == n_s && B.ncols == 2 * n_s, SAG_DIMENSION_MISMATCH,
                "reduce_dirichlet: shapes do not match the scalar width");
    std::vector<int> h(n_s);
    SAG_CUDA(cudaMemcpy(h.data(), old_to_new, 4 * (size_t)n_s, cudaMemcpyDefault));
    int ns_red = 0;
    for (int i = 0; i < n_s; ++i) ns_red += h[i] >= 0;
    DevBuf<int> o2n = upload(c, h.data(), n_s);
    DevBuf<double> dgx = upload(c, gx, n_s), dgy = upload(c, gy, n_s);
    DevBuf<double> lx(ns_red), ly(ns_red), rp_(B.nrows);
    const int g = grid_n(c, std::max(n_s, B.nrows));
    *a_red = wrap_m(csr_build(
        c, ns_red, ns_red,
        [&](int* cnt) {
          reduce_scalar_count_kernel<<<g, 256, 0, c.stream>>>(n_s, A.rp.p, A.ci.p, o2n.p, cnt);
          SAG_LAUNCHED(c);
        },
        [&](int* rp, int* ci, double* v) {
          reduce_scalar_fill_kernel<<<g, 256, 0, c.stream>>>(n_s, A.rp.p, A.ci.p, A.v.p, o2n.p,
                                                             dgx.p, dgy.p, rp, ci, v, lx.p, ly.p);
          SAG_LAUNCHED(c);
        }));
    *b_red = wrap_m(csr_build(
        c, B.nrows, 2 * ns_red,
        [&](int* cnt) {
          reduce_div_count_kernel<<<g, 256, 0, c.stream>>>(B.nrows, n_s, B.rp.p, B.ci.p, o2n.p,
                                                           cnt);
          SAG_LAUNCHED(c);
        },
        [&](int* rp, int* ci, double* v) {
          reduce_div_fill_kernel<<<g, 256, 0, c.stream>>>(B.nrows, n_s, ns_red, B.rp.p, B.ci.p,
                                                          B.v.p, o2n.p, dgx.p, dgy.p, rp, ci, v,
                                                          rp_.p);
          SAG_LAUNCHED(c);
        }));
    if (lift_x)
      SAG_CUDA(cudaMemcpyAsync(lift_x, lx.p, sizeof(double) * ns_red, cudaMemcpyDefault, c.stream));
    if (lift_y)
      SAG_CUDA(cudaMemcpyAsync(lift_y, ly.p, sizeof(double) * ns_red, cudaMemcpyDefault, c.stream));
    if (rhs_p)
      SAG_CUDA(cudaMemcpyAsync(rhs_p, rp_.p, sizeof(double) * B.nrows, cudaMemcpyDefault,
                               c.stream));
    SAG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
