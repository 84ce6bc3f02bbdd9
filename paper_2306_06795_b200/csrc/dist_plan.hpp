// Partition plan of the distributed solve (host-side, sag_dist_plan.cpp).
#pragma once

#include <map>
#include <vector>

namespace sag {

// a caller's CSR in host memory (sag_csr in sag.h)
struct HostCsr {
  int nrows = 0, ncols = 0;
  const int* rp = nullptr;
  const int* ci = nullptr;
  const double* v = nullptr;
};

// n x ncols CSR in rank-local numbering
struct LocalCsr {
  int n = 0, ncols = 0;
  std::vector<int> rp, ci;
  std::vector<double> v;
};

// patch lists (pptr, pidx, vptr, vidx, nx) in local ids
struct LocalPatches {
  std::vector<int> pptr, pidx, vptr, vidx, nx;
  int count() const { return (int)nx.size(); }
};

// one distributed level (K0 or L0) on a rank
struct LocalLevel {
  LocalCsr ext;                 // every local row restricted to local columns (factoring)
  LocalCsr rows_int, rows_bnd;  // owned rows reading owned columns only / the others
  long long rows_nnz = 0;
  LocalPatches p_int, p_bnd;    // own patches touching owned dofs only / the others
  std::vector<double> w;        // global partition-of-unity weights at the local dofs
};

struct RankPlan {
  int rank = 0, nranks = 1, n = 0, n_u = 0, n_p = 0;
  std::vector<long long> l2g;         // local -> global, ascending
  std::vector<unsigned char> owned;   // per local dof
  int n_u_loc = 0;                    // local velocity dofs ([x | y | p] split)
  long long patch_lo = 0, patch_hi = 0;
  // neighbour q -> local ids: owned values q reads (fwd_send), ghosts owned
  // by q (fwd_recv), ghosts owned by q that own patches touch (rev_send),
  // owned dofs q's patches touch (rev_recv); ascending global order
  std::map<int, std::vector<int>> fwd_send, fwd_recv, rev_send, rev_recv;
  LocalLevel k0, l0;
  LocalCsr p_own;                     // P0's owned rows (nl x n1), ghost rows empty
  int n1 = 0;
  int nl() const { return (int)l2g.size(); }
};

RankPlan plan_rank(int nranks, int rank, const HostCsr& k0, const HostCsr& l0, const HostCsr* p0,
                   int n_x, int n_y, int n_p);

}  // namespace sag
