// Multi-GPU partition of one KIFMM matvec: contiguous Morton ranges
// of leaves per rank, chosen by a prefix sum of a per-leaf work estimate, and the
// ghost plans that make every rank's share of the matvec complete.
//
// Every rank holds the same (replicated) tree and lists, so every rank derives the
// same partition and the same send AND receive lists without any negotiation.
//
// Ownership.  Rank r owns the sorted points [bnd[r], bnd[r+1]) (leaf boundaries).
//   D_r        boxes whose point range intersects the owned range: the boxes rank r
//              computes (partial) multipoles for and local expansions of.
//   straddle   boxes whose point range meets two or more ranks (at most P-1 per
//              level): their multipoles are sums of per-rank partials (allreduce).
// Work of rank r (by linearity of every translation):
//   S2M for owned leaves; M2M for children in D_r (partial multipoles);
//   M2L / X into targets in D_r; L2L into children in D_r;
//   L2T, W, P2P (U, direct W/X) for owned leaves.
// Ghosts of rank r (received from their unique owner s):
//   q^' rows: sources of V pairs (target in D_r) and of non-direct W pairs (owned
//             target leaf) that are neither complete on r nor straddling;
//   densities: points of U / direct-W / direct-X sources of owned leaves and of
//             non-direct X sources of targets in D_r, outside the owned range.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fmm_internal.h"

namespace kifmm {

namespace {

struct Interval {
  int b, e;
};

void merge_intervals(std::vector<Interval>& v) {
  std::sort(v.begin(), v.end(), [](const Interval& x, const Interval& y) { return x.b < y.b || (x.b == y.b && x.e < y.e); });
  size_t w = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i].e <= v[i].b) continue;
    if (w > 0 && v[i].b <= v[w - 1].e) v[w - 1].e = std::max(v[w - 1].e, v[i].e);
    else v[w++] = v[i];
  }
  v.resize(w);
}

}  // namespace

int build_partition(const PartitionInput& in, int nranks, int rank, DistPlan* out) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !out) {
    set_error("build_partition: bad nranks / rank");
    return -1;
  }
  const int nb = in.nboxes;
  DistPlan& D = *out;
  D = DistPlan();
  D.nranks = nranks;
  D.rank = rank;
  auto npts = [&](int b) { return (double)(in.pend[b] - in.pbeg[b]); };
  const int64_t N = nb > 0 ? in.pend[0] : 0;  // root holds every point
  auto U3 = [&](int64_t i, int f) { return in.U[i * in.ustride + f]; };
  auto V3 = [&](int64_t i, int f) { return in.V[i * in.vstride + f]; };
  auto W3 = [&](int64_t i, int f) { return in.W[i * in.wstride + f]; };
  auto X3 = [&](int64_t i, int f) { return in.X[i * in.xstride + f]; };

  // ---- per-leaf work estimate (pair-evaluation units; one V pair = 2k^2 DMMA flops
  //      ~ k^2/10 pair evaluations at the measured rates of the two FP64 paths)
  const double n = in.n, vcost = (double)in.k * in.k / 10.0;
  std::vector<double> leafw(nb, 0.0), boxw(nb, 0.0);
  for (int b = 0; b < nb; ++b) {
    if (in.leaf[b]) leafw[b] += 2.0 * n * npts(b);  // S2M + L2T evaluations
    boxw[b] += 2.0 * vcost;                            // M2M + L2L
  }
  for (int64_t i = 0; i < in.nU; ++i) leafw[U3(i, 0)] += npts(U3(i, 0)) * npts(U3(i, 1));
  for (int64_t i = 0; i < in.nV; ++i) boxw[V3(i, 0)] += vcost;
  for (int64_t i = 0; i < in.nW; ++i) leafw[W3(i, 0)] += npts(W3(i, 0)) * (W3(i, 2) ? npts(W3(i, 1)) : n);
  for (int64_t i = 0; i < in.nX; ++i) {
    if (X3(i, 2)) leafw[X3(i, 0)] += npts(X3(i, 0)) * npts(X3(i, 1));
    else boxw[X3(i, 0)] += n * npts(X3(i, 1));
  }
  // box costs spread over the box's points, pushed down to the leaves (boxes are
  // level-major, so a parent precedes its children)
  std::vector<double> perpt(nb, 0.0);
  for (int b = 0; b < nb; ++b) {
    const double m = std::max(1.0, npts(b));
    perpt[b] = (in.parent[b] >= 0 ? perpt[in.parent[b]] : 0.0) + boxw[b] / m;
    if (in.leaf[b]) leafw[b] += perpt[b] * npts(b);
  }
  std::vector<int> leaves;
  for (int b = 0; b < nb; ++b)
    if (in.leaf[b] && in.pend[b] > in.pbeg[b]) leaves.push_back(b);
  std::sort(leaves.begin(), leaves.end(), [&](int a, int b) { return in.pbeg[a] < in.pbeg[b]; });
  double total = 0;
  for (int b : leaves) total += leafw[b];
  // rank of a leaf: the share its weight midpoint falls in
  D.bnd.assign(nranks + 1, (int)N);
  D.bnd[0] = 0;
  {
    double run = 0;
    int r = 0;
    for (int b : leaves) {
      const double mid = run + 0.5 * leafw[b];
      int rr = total > 0 ? (int)std::floor(mid / total * nranks) : 0;
      rr = std::min(nranks - 1, std::max(rr, r));
      while (r < rr) D.bnd[++r] = in.pbeg[b];
      run += leafw[b];
    }
    while (r < nranks) D.bnd[++r] = (int)N;
  }
  D.own_lo = D.bnd[rank];
  D.own_hi = D.bnd[rank + 1];
  D.work.assign(nranks, 0.0);
  for (int b : leaves) {
    int r = (int)(std::upper_bound(D.bnd.begin(), D.bnd.end(), in.pbeg[b]) - D.bnd.begin()) - 1;
    D.work[std::min(r, nranks - 1)] += leafw[b];
  }
  // owner of a sorted point: the rank whose (non-empty) range contains it
  auto owner = [&](int i) {
    int r = (int)(std::upper_bound(D.bnd.begin(), D.bnd.end(), i) - D.bnd.begin()) - 1;
    return std::min(r, nranks - 1);
  };
  std::vector<int> rlo(nb), rhi(nb);  // ranks a box's points span (inclusive)
  for (int b = 0; b < nb; ++b) {
    if (in.pend[b] > in.pbeg[b]) { rlo[b] = owner(in.pbeg[b]); rhi[b] = owner(in.pend[b] - 1); }
    else { rlo[b] = 1; rhi[b] = 0; }
  }
  D.inD.assign(nb, 0);
  D.full.assign(nb, 0);
  for (int b = 0; b < nb; ++b) {
    D.inD[b] = rlo[b] <= rank && rank <= rhi[b];
    D.full[b] = rlo[b] == rank && rhi[b] == rank;
    if (rlo[b] < rhi[b]) D.straddle.push_back(b);
  }
  if (nranks == 1) return 0;

  // ---- ghost multipoles: need[r][s] = boxes r receives from s
  std::vector<std::vector<int>> qneed((size_t)nranks * nranks);
  auto need_q = [&](int tgt, int src) {
    if (rlo[src] != rhi[src]) return;  // straddling: allreduced
    const int s = rlo[src];
    for (int r = rlo[tgt]; r <= rhi[tgt]; ++r)
      if (r != s) qneed[(size_t)r * nranks + s].push_back(src);
  };
  for (int64_t i = 0; i < in.nV; ++i) need_q(V3(i, 0), V3(i, 1));
  for (int64_t i = 0; i < in.nW; ++i)
    if (!W3(i, 2)) need_q(W3(i, 0), W3(i, 1));
  // ---- ghost densities: point intervals r receives from s
  std::vector<std::vector<Interval>> dneed((size_t)nranks * nranks);
  auto need_d = [&](int tgt, int src) {
    const int b0 = in.pbeg[src], b1 = in.pend[src];
    if (b1 <= b0) return;
    for (int r = rlo[tgt]; r <= rhi[tgt]; ++r)
      for (int s = rlo[src]; s <= rhi[src]; ++s) {
        if (s == r) continue;
        const int lo = std::max(b0, D.bnd[s]), hi = std::min(b1, D.bnd[s + 1]);
        if (lo < hi) dneed[(size_t)r * nranks + s].push_back(Interval{lo, hi});
      }
  };
  for (int64_t i = 0; i < in.nU; ++i) need_d(U3(i, 0), U3(i, 1));
  for (int64_t i = 0; i < in.nW; ++i)
    if (W3(i, 2)) need_d(W3(i, 0), W3(i, 1));
  for (int64_t i = 0; i < in.nX; ++i) need_d(X3(i, 0), X3(i, 1));
  // ---- this rank's CSR lists (peer-major); send to s = what s needs from this rank
  auto flatten_q = [&](bool recv, std::vector<int>& list, std::vector<int>& off) {
    off.assign(nranks + 1, 0);
    list.clear();
    for (int s = 0; s < nranks; ++s) {
      std::vector<int>& v = recv ? qneed[(size_t)rank * nranks + s] : qneed[(size_t)s * nranks + rank];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      list.insert(list.end(), v.begin(), v.end());
      off[s + 1] = (int)list.size();
    }
  };
  flatten_q(true, D.q_recv, D.q_recv_off);
  flatten_q(false, D.q_send, D.q_send_off);
  auto flatten_d = [&](bool recv, std::vector<int>& list, std::vector<int>& off) {
    off.assign(nranks + 1, 0);
    list.clear();
    for (int s = 0; s < nranks; ++s) {
      std::vector<Interval>& v = recv ? dneed[(size_t)rank * nranks + s] : dneed[(size_t)s * nranks + rank];
      merge_intervals(v);
      for (const Interval& iv : v)
        for (int i = iv.b; i < iv.e; ++i) list.push_back(i);
      off[s + 1] = (int)list.size();
    }
  };
  flatten_d(true, D.d_recv, D.d_recv_off);
  flatten_d(false, D.d_send, D.d_send_off);
  return 0;
}

}  // namespace kifmm
