// libsag partition planner (host C++, no device): the row/patch partition of
// the distributed solve for one rank, computed identically on
// every rank from the global CSR arrays (no communication).
//
// Ownership: rank r owns the contiguous range of K0 Vanka patches
// [npatch r / N, npatch (r+1) / N) (pressure seeds are numbered by mesh vertex,
// so ranges are strips of the domain) and every dof whose lowest-numbered K0
// patch it owns. K0 and level 0 of the low-order hierarchy (the P1isoP2/P1
// operator on the same dofs, transfer.cpp:97-110) are distributed by that map;
// the coarser levels are agglomerated (every rank holds them).
//
// Rank-local numbering: owned dofs plus the ghosts its owned rows and its
// patches read, in ascending GLOBAL order. The map is monotone, so local CSR
// rows keep the reference's column order (sparse.cpp:84-87), local patch lists
// stay sorted with x before y (patch factors bitwise the global ones,
// vanka.cpp:88-140) and the [x | y | p] split is one threshold.
//
// paper_2306_06795_b200/partition.py is the numpy statement of the same plan
// (the CPU tests compare the two).
#include "dist_plan.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace sag {

namespace {

struct Pat {
  std::vector<int> pptr, pidx, vptr, vidx, nx;
  int count() const { return (int)pptr.size() - 1; }
};

// build_patches (vanka.cpp:11-42) for one pressure seed per patch
Pat th_patches(const HostCsr& m, int n_x, int n_y, int n_p) {
  const int n_u = n_x + n_y;
  Pat p;
  p.pptr.resize(n_p + 1);
  p.pidx.resize(n_p);
  p.vptr.assign(n_p + 1, 0);
  p.nx.assign(n_p, 0);
  for (int i = 0; i < n_p; ++i) {
    p.pptr[i] = i;
    p.pidx[i] = n_u + i;
    const int row = n_u + i;
    int cnt = 0;
    for (long long q = m.rp[row]; q < m.rp[row + 1]; ++q) {
      const int c = m.ci[q];
      if (c < n_u) {
        p.vidx.push_back(c);
        ++cnt;
        if (c < n_x) ++p.nx[i];
      }
    }
    if (cnt == 0)
      throw std::runtime_error("build_patches: pressure row " + std::to_string(i) +
                               " couples to no velocity DoFs");
    p.vptr[i + 1] = p.vptr[i] + cnt;
  }
  p.pptr[n_p] = n_p;
  return p;
}

// partition-of-unity weights w_d = 1 / multiplicity (vanka.cpp:67-73)
std::vector<double> pou_weights(int n, const Pat& p) {
  std::vector<long long> mult(n, 0);
  for (int v : p.vidx) ++mult[v];
  for (int v : p.pidx) ++mult[v];
  std::vector<double> w(n, 0.0);
  for (int i = 0; i < n; ++i)
    if (mult[i] > 0) w[i] = 1.0 / (double)mult[i];
  return w;
}

void local_csr(const HostCsr& m, const std::vector<long long>& l2g, const std::vector<int>& g2l,
               const std::vector<unsigned char>& rows_mask, LocalCsr& out) {
  const int nl = (int)l2g.size();
  out.n = nl;
  out.rp.assign(nl + 1, 0);
  out.ci.clear();
  out.v.clear();
  for (int i = 0; i < nl; ++i) {
    if (rows_mask[i]) {
      const long long g = l2g[i];
      for (long long q = m.rp[g]; q < m.rp[g + 1]; ++q) {
        const int c = g2l[m.ci[q]];
        if (c >= 0) {
          out.ci.push_back(c);
          out.v.push_back(m.v[q]);
        }
      }
    }
    out.rp[i + 1] = (int)out.ci.size();
  }
}

void split_rows(const LocalCsr& a, const std::vector<unsigned char>& owned, LocalCsr& in,
                LocalCsr& bnd) {
  const int nl = a.n;
  in.n = bnd.n = nl;
  in.rp.assign(nl + 1, 0);
  bnd.rp.assign(nl + 1, 0);
  in.ci.clear();
  in.v.clear();
  bnd.ci.clear();
  bnd.v.clear();
  for (int r = 0; r < nl; ++r) {
    bool interior = true;
    for (int q = a.rp[r]; q < a.rp[r + 1]; ++q)
      if (!owned[a.ci[q]]) interior = false;
    LocalCsr& d = interior ? in : bnd;
    for (int q = a.rp[r]; q < a.rp[r + 1]; ++q) {
      d.ci.push_back(a.ci[q]);
      d.v.push_back(a.v[q]);
    }
    in.rp[r + 1] = (int)in.ci.size();
    bnd.rp[r + 1] = (int)bnd.ci.size();
  }
}

void select_patches(const LocalPatches& p, const std::vector<char>& keep, LocalPatches& out) {
  out = LocalPatches{};
  out.pptr.push_back(0);
  out.vptr.push_back(0);
  for (int i = 0; i + 1 < (int)p.pptr.size(); ++i) {
    if (!keep[i]) continue;
    for (int q = p.pptr[i]; q < p.pptr[i + 1]; ++q) out.pidx.push_back(p.pidx[q]);
    for (int q = p.vptr[i]; q < p.vptr[i + 1]; ++q) out.vidx.push_back(p.vidx[q]);
    out.pptr.push_back((int)out.pidx.size());
    out.vptr.push_back((int)out.vidx.size());
    out.nx.push_back(p.nx[i]);
  }
}

}  // namespace

RankPlan plan_rank(int nranks, int rank, const HostCsr& k0, const HostCsr& l0, const HostCsr* p0,
                   int n_x, int n_y, int n_p) {
  if (nranks < 1 || rank < 0 || rank >= nranks)
    throw std::runtime_error("partition: rank out of range");
  const int n = n_x + n_y + n_p;
  if (k0.nrows != n || l0.nrows != n)
    throw std::runtime_error(
        "partition: the low-order level 0 must live on the K0 dofs (Taylor-Hood transfer)");
  const int n_u = n_x + n_y;
  const Pat pk = th_patches(k0, n_x, n_y, n_p), pl = th_patches(l0, n_x, n_y, n_p);
  const int npatch = pk.count();
  std::vector<long long> bounds(nranks + 1);
  for (int r = 0; r <= nranks; ++r) bounds[r] = (long long)npatch * r / nranks;
  // owner: rank of the lowest-numbered K0 patch containing the dof
  std::vector<int> first(n, -1);
  for (int i = 0; i < npatch; ++i) {
    for (int q = pk.vptr[i]; q < pk.vptr[i + 1]; ++q)
      if (first[pk.vidx[q]] < 0) first[pk.vidx[q]] = i;
    for (int q = pk.pptr[i]; q < pk.pptr[i + 1]; ++q)
      if (first[pk.pidx[q]] < 0) first[pk.pidx[q]] = i;
  }
  std::vector<int> owner(n);
  for (int d = 0; d < n; ++d) {
    if (first[d] >= 0)
      owner[d] = (int)(std::upper_bound(bounds.begin() + 1, bounds.end(), (long long)first[d]) -
                       (bounds.begin() + 1));
    else
      owner[d] = std::min((int)((long long)d * nranks / std::max(n, 1)), nranks - 1);
  }
  const std::vector<double> wk = pou_weights(n, pk), wl = pou_weights(n, pl);
  // every rank's ghosts (the peers' send lists need them): columns of owned
  // rows of K0 and L0, dofs of own patches of both levels
  std::vector<std::vector<int>> need(nranks), touch(nranks);
  std::vector<int> mark(n, -1), tmark(n, -1);
  for (int r = 0; r < nranks; ++r) {
    auto add = [&](int d) {
      if (owner[d] != r && mark[d] != r) {
        mark[d] = r;
        need[r].push_back(d);
      }
    };
    auto addt = [&](int d) {
      if (owner[d] != r && tmark[d] != r) {
        tmark[d] = r;
        touch[r].push_back(d);
      }
    };
    for (int d = 0; d < n; ++d) {
      if (owner[d] != r) continue;
      for (const HostCsr* m : {&k0, &l0})
        for (long long q = m->rp[d]; q < m->rp[d + 1]; ++q) add(m->ci[q]);
    }
    for (const Pat* pt : {&pk, &pl})
      for (long long i = bounds[r]; i < bounds[r + 1]; ++i) {
        for (int q = pt->vptr[i]; q < pt->vptr[i + 1]; ++q) {
          add(pt->vidx[q]);
          addt(pt->vidx[q]);
        }
        for (int q = pt->pptr[i]; q < pt->pptr[i + 1]; ++q) {
          add(pt->pidx[q]);
          addt(pt->pidx[q]);
        }
      }
    std::sort(need[r].begin(), need[r].end());
    std::sort(touch[r].begin(), touch[r].end());
  }
  RankPlan rs;
  rs.rank = rank;
  rs.nranks = nranks;
  rs.n = n;
  rs.n_u = n_u;
  rs.n_p = n_p;
  rs.patch_lo = bounds[rank];
  rs.patch_hi = bounds[rank + 1];
  {
    std::vector<long long> own;
    for (int d = 0; d < n; ++d)
      if (owner[d] == rank) own.push_back(d);
    rs.l2g.resize(own.size() + need[rank].size());
    std::merge(own.begin(), own.end(), need[rank].begin(), need[rank].end(), rs.l2g.begin());
  }
  const int nl = (int)rs.l2g.size();
  std::vector<int> g2l(n, -1);
  for (int i = 0; i < nl; ++i) g2l[rs.l2g[i]] = i;
  rs.owned.resize(nl);
  for (int i = 0; i < nl; ++i) rs.owned[i] = owner[rs.l2g[i]] == rank;
  rs.n_u_loc = (int)(std::lower_bound(rs.l2g.begin(), rs.l2g.end(), (long long)n_u) -
                     rs.l2g.begin());
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    auto pick = [&](const std::vector<int>& src, int who, std::map<int, std::vector<int>>& dst,
                    int key) {
      std::vector<int> loc;
      for (int d : src)
        if (owner[d] == who) loc.push_back(g2l[d]);
      if (!loc.empty()) dst[key] = std::move(loc);
    };
    pick(need[rank], q, rs.fwd_recv, q);   // my ghosts owned by q
    pick(need[q], rank, rs.fwd_send, q);   // my owned dofs q reads
    pick(touch[rank], q, rs.rev_send, q);  // my patches' dofs owned by q
    pick(touch[q], rank, rs.rev_recv, q);  // q's patches' dofs I own
  }
  std::vector<unsigned char> all(nl, 1);
  const Pat* pts[2] = {&pk, &pl};
  const HostCsr* ms[2] = {&k0, &l0};
  const std::vector<double>* ws[2] = {&wk, &wl};
  for (int li = 0; li < 2; ++li) {
    LocalLevel& L = li == 0 ? rs.k0 : rs.l0;
    LocalCsr rows;
    local_csr(*ms[li], rs.l2g, g2l, rs.owned, rows);
    local_csr(*ms[li], rs.l2g, g2l, all, L.ext);
    split_rows(rows, rs.owned, L.rows_int, L.rows_bnd);
    L.rows_nnz = (long long)rows.ci.size();
    const Pat& pt = *pts[li];
    LocalPatches lp;
    lp.pptr.push_back(0);
    lp.vptr.push_back(0);
    for (long long i = bounds[rank]; i < bounds[rank + 1]; ++i) {
      for (int q = pt.pptr[i]; q < pt.pptr[i + 1]; ++q) lp.pidx.push_back(g2l[pt.pidx[q]]);
      for (int q = pt.vptr[i]; q < pt.vptr[i + 1]; ++q) lp.vidx.push_back(g2l[pt.vidx[q]]);
      lp.pptr.push_back((int)lp.pidx.size());
      lp.vptr.push_back((int)lp.vidx.size());
      lp.nx.push_back(pt.nx[i]);
    }
    // interior patches touch owned dofs only
    const int np_loc = (int)lp.nx.size();
    std::vector<char> interior(np_loc, 1);
    for (int i = 0; i < np_loc; ++i) {
      for (int q = lp.vptr[i]; q < lp.vptr[i + 1]; ++q)
        if (!rs.owned[lp.vidx[q]]) interior[i] = 0;
      for (int q = lp.pptr[i]; q < lp.pptr[i + 1]; ++q)
        if (!rs.owned[lp.pidx[q]]) interior[i] = 0;
    }
    std::vector<char> boundary(np_loc);
    for (int i = 0; i < np_loc; ++i) boundary[i] = !interior[i];
    select_patches(lp, interior, L.p_int);
    select_patches(lp, boundary, L.p_bnd);
    L.w.resize(nl);
    for (int i = 0; i < nl; ++i) L.w[i] = (*ws[li])[rs.l2g[i]];
  }
  if (p0) {
    // P0's owned rows (ghost rows empty), columns global (agglomerated level 1)
    rs.n1 = p0->ncols;
    rs.p_own.n = nl;
    rs.p_own.ncols = p0->ncols;
    rs.p_own.rp.assign(nl + 1, 0);
    for (int i = 0; i < nl; ++i) {
      if (rs.owned[i]) {
        const long long g = rs.l2g[i];
        for (long long q = p0->rp[g]; q < p0->rp[g + 1]; ++q) {
          rs.p_own.ci.push_back(p0->ci[q]);
          rs.p_own.v.push_back(p0->v[q]);
        }
      }
      rs.p_own.rp[i + 1] = (int)rs.p_own.ci.size();
    }
  }
  return rs;
}

}  // namespace sag
