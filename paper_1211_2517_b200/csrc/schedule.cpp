// Launch schedules of the matvec, derived once at setup from the device tree and
// lists: pair lists + tiles for the grouped GEMM kernel, and segment CSRs for the
// evaluation kernel.  Applies the W/X "direct" shortcut of reading O5.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>

#include "fmm_internal.h"

namespace kifmm {

// device memory the automatic leaf / X operators leave free: max(16 GB, 10% of the device)
// (measured headroom need: the plan's own work buffers are allocated before this check)
static double leaf_op_reserve(size_t total) { return std::max(16.0 * (1 << 30), 0.10 * (double)total); }


namespace {

template <typename T>
int upload(Plan& P, T** dst, const std::vector<T>& v, cudaStream_t st) {
  KIFMM_CUDA(cudaMalloc((void**)dst, sizeof(T) * std::max<size_t>(v.size(), 1)));
  P.allocations.push_back(*dst);
  if (!v.empty()) KIFMM_CUDA(cudaMemcpyAsync(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  return 0;
}

struct PairGroup {
  int op;
  double scale;
  std::vector<int2> pairs;
};

// tiles of <= width pairs that never straddle a group
int make_launch(Plan& P, GemmLaunch& L, const std::vector<PairGroup>& groups, int width, cudaStream_t st) {
  std::vector<int2> pairs;
  std::vector<GemmTile> tiles;
  for (const auto& g : groups) {
    int base = (int)pairs.size();
    pairs.insert(pairs.end(), g.pairs.begin(), g.pairs.end());
    for (int b = 0; b < (int)g.pairs.size(); b += width)
      tiles.push_back(GemmTile{g.op, base + b, std::min(width, (int)g.pairs.size() - b), 0, g.scale});
  }
  L.npairs = (int)pairs.size();
  L.ntiles = (int)tiles.size();
  if (upload(P, &L.d_pairs, pairs, st) || upload(P, &L.d_tiles, tiles, st)) return -3;
  return 0;
}

}  // namespace

int build_schedules(Plan& P, cudaStream_t st) {
  // KIFMM_DEBUG_SETUP=1: host time per section (device work synchronised) on stderr
  static const bool dbg = std::getenv("KIFMM_DEBUG_SETUP") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "schedule %-14s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  Tree& T = P.tree;
  Lists& Ls = P.lists;
  const int nb = T.nboxes, n = P.n, np = P.np, kp = P.kp;
  // lists back to the host (setup only)
  std::vector<int2> U(Ls.nU);
  std::vector<int4> V(Ls.nV), W(Ls.nW), X(Ls.nX);
  if (Ls.nU) KIFMM_CUDA(cudaMemcpyAsync(U.data(), Ls.d_U, sizeof(int2) * Ls.nU, cudaMemcpyDeviceToHost, st));
  if (Ls.nV) KIFMM_CUDA(cudaMemcpyAsync(V.data(), Ls.d_V, sizeof(int4) * Ls.nV, cudaMemcpyDeviceToHost, st));
  if (Ls.nW) KIFMM_CUDA(cudaMemcpyAsync(W.data(), Ls.d_W, sizeof(int4) * Ls.nW, cudaMemcpyDeviceToHost, st));
  if (Ls.nX) KIFMM_CUDA(cudaMemcpyAsync(X.data(), Ls.d_X, sizeof(int4) * Ls.nX, cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  // validate the device lists before indexing host arrays with them
  auto bad = [&](int b) { return b < 0 || b >= nb; };
  for (auto& u : U)
    if (bad(u.x) || bad(u.y) || !T.leaf[u.x] || !T.leaf[u.y]) { set_error("build_schedules: corrupt U list"); return -3; }
  for (auto& v : V)
    if (bad(v.x) || bad(v.y) || v.z < 0 || v.z >= kNumOffsets) { set_error("build_schedules: corrupt V list"); return -3; }
  for (auto& w : W)
    if (bad(w.x) || bad(w.y) || !T.leaf[w.x]) { set_error("build_schedules: corrupt W list"); return -3; }
  for (auto& x : X)
    if (bad(x.x) || bad(x.y) || !T.leaf[x.y] || (x.z && !T.leaf[x.x])) { set_error("build_schedules: corrupt X list"); return -3; }
  auto npts = [&](int b) { return T.pend[b] - T.pbeg[b]; };
  auto rl = [&](int b) { return std::ldexp(T.r0, -T.level[b]); };
  mark("lists+validate");

  // ---- partition; one rank owns everything
  {
    PartitionInput in;
    in.nboxes = nb;
    in.level = T.level.data(); in.parent = T.parent.data(); in.pbeg = T.pbeg.data(); in.pend = T.pend.data();
    in.leaf = T.leaf.data();
    in.nU = U.size(); in.U = reinterpret_cast<const int*>(U.data()); in.ustride = 2;
    in.nV = V.size(); in.V = reinterpret_cast<const int*>(V.data()); in.vstride = 4;
    in.nW = W.size(); in.W = reinterpret_cast<const int*>(W.data()); in.wstride = 4;
    in.nX = X.size(); in.X = reinterpret_cast<const int*>(X.data()); in.xstride = 4;
    in.n = n; in.k = P.k;
    const int nr = P.dist.nranks, rk = P.dist.rank;
    if (build_partition(in, nr, rk, &P.dist)) return -1;
  }
  mark("partition");
  const DistPlan& Dp = P.dist;
  auto inD = [&](int b) { return Dp.inD[b] != 0; };
  // per-leaf S2M / L2T operators (owned points x kp doubles each): on request, or
  // automatically while they leave kLeafOpReserve free (S2M first)
  {
    const double one = (double)(Dp.own_hi - Dp.own_lo) * kp * sizeof(double);
    size_t fr = 0, tot = 0;
    KIFMM_CUDA(cudaMemGetInfo(&fr, &tot));
    const double budget = (double)fr - leaf_op_reserve(tot);
    const bool on = P.leaf_ops_opt > 0, au = P.leaf_ops_opt < 0;
    P.leaf_s2m = on || P.bem || (au && one <= budget);  // BEM: S2M by element integration, always an operator
    P.leaf_l2t = on || (au && one * (P.leaf_s2m ? 2 : 1) <= budget);
  }

  // ---- target leaves (owned), near (P2P) and far (L2T + W) segment CSRs
  std::vector<int> leaf_row(nb, -1);
  std::vector<int4> titems;
  for (int b = 0; b < nb; ++b)
    if (T.leaf[b] && inD(b)) { leaf_row[b] = (int)titems.size(); titems.push_back(make_int4(b, (int)titems.size(), 0, 0)); }
  const int nt = (int)titems.size();
  std::vector<std::vector<int4>> near(nt), far(nt);
  // the target leaf's own points first: only they can coincide with a target (equal
  // coordinates give equal Morton keys, hence the same leaf), so k_eval tests r = 0
  // on the first m_B sources only
  for (int i = 0; i < nt; ++i) {
    const int b = titems[i].x;
    near[i].push_back(make_int4(0, T.pbeg[b], 0, npts(b)));
  }
  // Symmetric near field: U pairs and direct W pairs with a leaf source (whose mirror is
  // the direct X pair), both leaves owned, evaluated once for both sides.
  //  * mutual mode (default): the pair becomes a mutual source segment of ONE of its
  //    leaves, evaluated by k_near (near.cu: ~13 FP64 ops per unordered pair against
  //    2 x 12 one-sided); the target side is the leaf whose k_near pass pads least
  //    (TB x MQ slots), ties split by index parity;
  //  * warp-pair mode (KIFMM_SYM=2): k_p2p_sym, one warp per pair, chosen per pair when
  //    its padding (targets in passes of 32 TB lanes, sources in batches of 16) is small.
  bool mutual = P.sym_opt == -1 || P.sym_opt == 1;
  const bool sym = P.sym_opt == 2;
  if (mutual) {  // k_near's source-slot table (4 B per near-field source) must fit the budget
    int64_t slots = 0;
    for (auto& u : U)
      if (inD(u.x)) slots += npts(u.y);
    for (auto& w : W)
      if (inD(w.x) && w.z) slots += npts(w.y);
    for (auto& x : X)
      if (inD(x.x) && x.z) slots += npts(x.y);
    size_t fr = 0, tot = 0;
    KIFMM_CUDA(cudaMemGetInfo(&fr, &tot));
    const double budget = (double)fr - leaf_op_reserve(tot);
    // (slot offsets are int32: past ~2e9 slots the one-sided k_eval path takes over)
    if (4.0 * (double)slots > budget || slots > 2000000000LL) mutual = false;
  }
  constexpr double sym_r = 1.4;  // padding-factor threshold of the warp-pair mode (measured scan 1.1-2.0)
  auto pass_slots = [](int m) { int full = m / 96, rem = m - 96 * full; return 96 * full + 32 * ((rem + 31) / 32); };
  auto pad_ratio = [&](int mt, int ms) {
    return (double)pass_slots(mt) / mt * (double)((ms + 15) / 16 * 16) / ms;
  };
  // returns 0: one-sided, 1: symmetric with (a, b), 2: symmetric with (b, a)
  auto sym_choice = [&](int a, int b) {
    if (!sym || !inD(a) || !inD(b)) return 0;
    const double r1 = pad_ratio(npts(a), npts(b)), r2 = pad_ratio(npts(b), npts(a));
    if (std::min(r1, r2) > sym_r) return 0;
    return r1 <= r2 ? 1 : 2;
  };
  // k_near pass shape of an m-point leaf (the least padding; passes of the largest beyond it)
  const bool dl = P.d_nrm != nullptr;
  const int nr_tab = dl ? 3 : 0;  // double layer: shapes up to 160 targets
  P.nr_table = nr_tab;
  const int kNearShapes = near_shape_count(nr_tab);
  auto nr_shape = [&](int m) {
    for (int c = 0; c < kNearShapes; ++c)
      if (m <= near_shape_cap(nr_tab, c)) return c;
    return kNearShapes - 1;
  };
  auto nr_slots = [&](int m) {
    const int cap = near_shape_cap(nr_tab, nr_shape(m));
    return (m + cap - 1) / cap * cap;
  };
  // target side of a mutual pair {a, b}, or -1 (not both owned)
  std::vector<int> leaf_slots(nb, 0);  // nr_slots of every owned leaf, once
  if (mutual)
    for (int i = 0; i < nt; ++i) leaf_slots[titems[i].x] = nr_slots(npts(titems[i].x));
  auto mut_target = [&](int a, int b) {
    if (!mutual || !inD(a) || !inD(b)) return -1;
    const int64_t ca = (int64_t)leaf_slots[a] * npts(b), cb = (int64_t)leaf_slots[b] * npts(a);
    if (ca != cb) return ca < cb ? a : b;
    return ((a ^ b) & 1) ? std::min(a, b) : std::max(a, b);
  };
  mark("segments setup");
  std::vector<std::vector<int4>> mnear(nt);
  std::vector<int2> sympairs;
  auto add_sym = [&](int a, int b, int c) { sympairs.push_back(c == 1 ? make_int2(a, b) : make_int2(b, a)); };
  for (auto& u : U) {
    if (!inD(u.x) || u.y == u.x) continue;
    if (int t = mut_target(u.x, u.y); t >= 0) {
      if (t == u.x) mnear[leaf_row[u.x]].push_back(make_int4(3, T.pbeg[u.y], 0, npts(u.y)));
      continue;
    }
    if (int c = sym_choice(u.x, u.y)) {
      if (u.x < u.y) add_sym(u.x, u.y, c);
      continue;
    }
    near[leaf_row[u.x]].push_back(make_int4(0, T.pbeg[u.y], 0, npts(u.y)));
  }
  mark("segments U");
  // W pairs: direct -> P2P over the source subtree; else M2T through the source's equivalent density
  std::vector<PairGroup> wgroups;  // grouped by source level (scale r_A)
  std::map<int, int> wlevel;
  int n_wnd = 0;
  for (auto& w : W) {
    if (!inD(w.x)) continue;
    if (w.z && T.leaf[w.y]) {
      if (int t = mut_target(w.x, w.y); t >= 0) {
        const int o = t == w.x ? w.y : w.x;
        mnear[leaf_row[t]].push_back(make_int4(3, T.pbeg[o], 0, npts(o)));
        continue;
      }
      if (int c = sym_choice(w.x, w.y)) {
        add_sym(w.x, w.y, c);
        continue;
      }
    }
    if (w.z) {
      near[leaf_row[w.x]].push_back(make_int4(0, T.pbeg[w.y], 0, npts(w.y)));
    } else {
      int lv = T.level[w.y];
      if (!wlevel.count(lv)) { wlevel[lv] = (int)wgroups.size(); wgroups.push_back(PairGroup{0, rl(w.y), {}}); }
      wgroups[wlevel[lv]].pairs.push_back(make_int2(w.y, n_wnd));
      far[leaf_row[w.x]].push_back(make_int4(2, n_wnd, w.y, n));
      ++n_wnd;
    }
  }
  // X pairs: direct (target leaf small) -> P2P; else S2L through the target's check potential
  std::vector<int4> xitems, xsegs;
  std::vector<int> xoff{0};
  std::vector<PairGroup> xgroup{PairGroup{0, 1.0, {}}};
  for (auto& x : X) {
    if (!inD(x.x)) continue;
    if (x.z && (mut_target(x.x, x.y) >= 0 || sym_choice(x.x, x.y))) continue;  // mirror of a symmetric W pair
    if (x.z) {
      near[leaf_row[x.x]].push_back(make_int4(0, T.pbeg[x.y], 0, npts(x.y)));
    } else {
      int row = (int)xitems.size();
      xitems.push_back(make_int4(x.x, row, 0, 0));
      xsegs.push_back(make_int4(0, T.pbeg[x.y], 0, npts(x.y)));
      xoff.push_back((int)xsegs.size());
      xgroup[0].pairs.push_back(make_int2(row, x.x));
    }
  }
  // L2T for leaves at level >= 2 (grouped by level for the r_l factor)
  std::vector<PairGroup> lgroups;
  std::map<int, int> llevel;
  int n_l2t = 0;
  for (int i = 0; i < nt; ++i) {
    int b = titems[i].x;
    if (T.level[b] < 2 || P.leaf_l2t) continue;  // L2T as a GEMV with the leaf's operator
    int lv = T.level[b];
    if (!llevel.count(lv)) { llevel[lv] = (int)lgroups.size(); lgroups.push_back(PairGroup{0, rl(b), {}}); }
    lgroups[llevel[lv]].pairs.push_back(make_int2(b, n_l2t));
    far[i].insert(far[i].begin(), make_int4(1, n_l2t, b, n));
    ++n_l2t;
  }
  mark("segments");
  // k_near tables (mutual mode): per target leaf its source list — own points (checked),
  // mutual segments, one-sided point segments — cut into chunks of near_ch(cap) source slots;
  // work units = (pass of <= TB x MQ targets, <= kUnitChunks chunks), grouped by pass
  // shape (see below), longest first
  P.nr_on = mutual;
  P.n_tleaf_mut = 0;
  P.n_mut_pairs = 0;
  P.n_near_pairs = 0;
  P.nr_groups.clear();
  if (mutual && nt > 0) {
    constexpr int kMinGroup = 2048;  // leaves per pass-shape launch (smaller groups fold into a neighbour)
    constexpr int kUnitChunks = 4;   // chunks per work unit (C3 6.2 -> 5.3 ms against whole leaves)
    // pass shape per leaf: the least-padding shape, unless its group would have fewer than
    // kMinGroup leaves — then the next larger kept shape (more padding), or for the
    // largest leaves the largest kept smaller shape (more passes)
    // (a leaf above the largest capacity runs in equal passes: ceil(m / cap_max) of them)
    const int cap_max = near_shape_cap(nr_tab, kNearShapes - 1);
    auto pass_size = [&](int m) { const int np = (m + cap_max - 1) / cap_max; return (m + np - 1) / np; };
    std::vector<int> shp(nt), cnt(kNearShapes, 0);
    for (int i = 0; i < nt; ++i) ++cnt[shp[i] = nr_shape(pass_size(npts(titems[i].x)))];
    {
      std::vector<int> kept;
      for (int c = 0; c < kNearShapes; ++c)
        if (cnt[c] >= kMinGroup) kept.push_back(c);
      if (kept.empty()) kept.push_back(*std::max_element(shp.begin(), shp.end()));
      std::vector<int> remap(kNearShapes);
      for (int c = 0; c < kNearShapes; ++c) {
        auto it = std::lower_bound(kept.begin(), kept.end(), c);
        remap[c] = it != kept.end() ? *it : kept.back();
      }
      for (int i = 0; i < nt; ++i) shp[i] = remap[shp[i]];
      std::fill(cnt.begin(), cnt.end(), 0);
    }
    // sizes per leaf (slots, chunks = ceil(slots / CH), units = passes x ceil(chunks / kUnitChunks)),
    // prefix offsets, then every leaf's slots / chunks / units filled in parallel at its offsets
    std::vector<int64_t> slot_off(nt + 1, 0), chunk_off(nt + 1, 0), unit_off(nt + 1, 0);
    for (int i = 0; i < nt; ++i) {
      const int b = titems[i].x, m = npts(b);
      if (!mnear[i].empty()) ++P.n_tleaf_mut;
      int64_t slots = m;
      P.n_near_pairs += (int64_t)m * m;
      for (auto& sg : mnear[i]) {
        slots += sg.w;
        P.n_mut_pairs += (int64_t)m * sg.w;
        P.n_near_pairs += 2 * (int64_t)m * sg.w;
      }
      for (size_t k = 1; k < near[i].size(); ++k) {
        slots += near[i][k].w;
        P.n_near_pairs += (int64_t)m * near[i][k].w;
      }
      const int CH = near_ch(near_shape_cap(nr_tab, shp[i]), dl);
      const int cap = std::min(near_shape_cap(nr_tab, shp[i]), pass_size(m));
      const int64_t nch = (slots + CH - 1) / CH;
      slot_off[i + 1] = slot_off[i] + slots;
      chunk_off[i + 1] = chunk_off[i] + nch;
      unit_off[i + 1] = unit_off[i] + (int64_t)((m + cap - 1) / cap) * ((nch + kUnitChunks - 1) / kUnitChunks);
    }
    if (slot_off[nt] > INT32_MAX || chunk_off[nt] > INT32_MAX) {
      set_error("build_schedules: near-field slot table exceeds 2^31 entries");
      return -3;
    }
    std::vector<int4> nchunks(chunk_off[nt]);
    std::vector<int> nsrc(slot_off[nt]);
    std::vector<std::pair<int64_t, int4>> uall(unit_off[nt]);  // (cost, unit), leaf order
#pragma omp parallel for schedule(dynamic, 256)
    for (int i = 0; i < nt; ++i) {
      const int b = titems[i].x;
      const int CH = near_ch(near_shape_cap(nr_tab, shp[i]), dl);
      int64_t spos = slot_off[i];
      int cpos = (int)chunk_off[i];
      int n = 0, nchk = 0, ml = -1, mh = -1;
      auto flush = [&]() {
        if (n == 0) return;
        if (ml < 0) ml = mh = n;
        nchunks[cpos++] = make_int4((int)(spos - n), n | (nchk << 10) | (ml << 20), mh, 0);
        n = nchk = 0;
        ml = mh = -1;
      };
      auto add = [&](int kind, int a, int len) {  // kind 0 one-sided, 1 own points, 3 mutual
        for (int off = 0; off < len;) {
          const int take = std::min(len - off, CH - n);
          if (kind == 1) nchk = n + take;
          if (kind == 3) { if (ml < 0) ml = n; mh = n + take; }
          for (int t = 0; t < take; ++t) nsrc[spos++] = a + off + t;
          n += take;
          off += take;
          if (n == CH) flush();
        }
      };
      add(1, T.pbeg[b], npts(b));
      for (auto& sg : mnear[i]) add(3, sg.y, sg.w);
      for (size_t k = 1; k < near[i].size(); ++k) add(0, near[i][k].y, near[i][k].w);
      flush();
      const int cb = (int)chunk_off[i], ce = (int)chunk_off[i + 1];
      const int cap = std::min(near_shape_cap(nr_tab, shp[i]), pass_size(npts(b)));
      int64_t upos = unit_off[i];
      for (int t0 = 0; t0 < npts(b); t0 += cap)
        for (int c0 = cb; c0 < ce; c0 += kUnitChunks) {
          const int c1 = std::min(ce, c0 + kUnitChunks);
          int64_t srcs = 0;
          for (int c = c0; c < c1; ++c) srcs += nchunks[c].y & 1023;
          uall[upos++] = {srcs * cap, make_int4(T.pbeg[b] + t0, std::min(cap, npts(b) - t0), c0, c1)};
        }
    }
    std::vector<std::vector<std::pair<int64_t, int4>>> units(kNearShapes);  // (cost, unit) per shape
    for (int i = 0; i < nt; ++i) {
      cnt[shp[i]] += (int)(unit_off[i + 1] - unit_off[i]);
      units[shp[i]].insert(units[shp[i]].end(), uall.begin() + unit_off[i], uall.begin() + unit_off[i + 1]);
    }
    std::vector<int4> nitems;
    for (int c = 0; c < kNearShapes; ++c) {
      std::vector<std::pair<int64_t, int4>>& g = units[c];
      if (g.empty()) continue;
      std::stable_sort(g.begin(), g.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
      const int first = (int)nitems.size();
      for (auto& u : g) nitems.push_back(u.second);
      P.nr_groups.push_back(make_int3(c, first, (int)nitems.size() - first));
    }
    P.nr_src_bytes = (int64_t)nsrc.size() * sizeof(int);
    std::vector<int> counters(2 * P.nr_groups.size(), 0);
    if (upload(P, &P.d_nr_items, nitems, st) || upload(P, &P.d_nr_chunks, nchunks, st) ||
        upload(P, &P.d_nr_src, nsrc, st) || upload(P, &P.d_nr_counters, counters, st))
      return -3;
  }
  mark("k_near tables");
  std::vector<int> near_off{0}, far_off{0}, all_off{0};
  std::vector<int4> near_seg, far_seg, all_seg;
  for (int i = 0; i < nt; ++i) {
    near_seg.insert(near_seg.end(), near[i].begin(), near[i].end());
    near_off.push_back((int)near_seg.size());
    far_seg.insert(far_seg.end(), far[i].begin(), far[i].end());
    far_off.push_back((int)far_seg.size());
    all_seg.insert(all_seg.end(), near[i].begin(), near[i].end());
    all_seg.insert(all_seg.end(), far[i].begin(), far[i].end());
    all_off.push_back((int)all_seg.size());
  }
  P.n_tleaf = nt;
  // costliest pairs first (one warp each)
  std::stable_sort(sympairs.begin(), sympairs.end(), [&](const int2& a, const int2& b) {
    return (int64_t)npts(a.x) * npts(a.y) > (int64_t)npts(b.x) * npts(b.y);
  });
  P.n_sym = (int)sympairs.size();
  if (upload(P, &P.d_sym, sympairs, st)) return -3;

  P.n_near_seg = (int)near_seg.size();
  if (P.bem) {  // near-field block matrix (S2T by element integration)
    std::vector<int4> blocks;
    blocks.reserve(near_seg.size());
    for (int i = 0; i < nt; ++i) {
      const int b = titems[i].x;
      for (int s = near_off[i]; s < near_off[i + 1]; ++s)
        blocks.push_back(make_int4(T.pbeg[b], npts(b), near_seg[s].y, near_seg[s].w));
    }
    if (upload(P, &P.d_near_seg, near_seg, st) || upload(P, &P.d_near_off, near_off, st)) return -3;
    if (int rc = bem_build_near(P, blocks, st)) return rc;
  }
  P.n_far_seg = (int)far_seg.size();
  {  // the far pass over only the leaves with far segments (when it adds to stored results)
    std::vector<int4> fi, fs;
    std::vector<int> fo{0};
    for (int i = 0; i < nt; ++i) {
      if (far[i].empty()) continue;
      fi.push_back(titems[i]);
      fs.insert(fs.end(), far[i].begin(), far[i].end());
      fo.push_back((int)fs.size());
    }
    P.n_fitems = (int)fi.size();
    if (P.n_fitems > 0 &&
        (upload(P, &P.d_fitems, fi, st) || upload(P, &P.d_fitem_off, fo, st) || upload(P, &P.d_fitem_seg, fs, st)))
      return -3;
  }
  if (upload(P, &P.d_tleaf_items, titems, st) ||
      (!P.bem && (upload(P, &P.d_near_off, near_off, st) || upload(P, &P.d_near_seg, near_seg, st))) ||
      upload(P, &P.d_far_off, far_off, st) ||
      upload(P, &P.d_far_seg, far_seg, st) || upload(P, &P.d_all_off, all_off, st) ||
      upload(P, &P.d_all_seg, all_seg, st))
    return -3;
  mark("csr uploads");
  // ---- S2M: leaves at level >= 2
  std::vector<int4> sitems, ssegs;
  std::vector<int> soff{0};
  std::vector<PairGroup> sgroup{PairGroup{0, 1.0, {}}};
  for (int b = 0; b < nb; ++b) {
    if (!T.leaf[b] || T.level[b] < 2 || !inD(b)) continue;
    int row = (int)sitems.size();
    sitems.push_back(make_int4(b, row, 0, 0));
    ssegs.push_back(make_int4(0, T.pbeg[b], 0, npts(b)));
    soff.push_back((int)ssegs.size());
    sgroup[0].pairs.push_back(make_int2(row, b));
  }
  P.n_s2m = (int)sitems.size();
  P.n_xnd = (int)xitems.size();
  P.n_l2t = n_l2t;
  P.n_wnd = n_wnd;
  if (upload(P, &P.d_s2m_items, sitems, st) || upload(P, &P.d_s2m_off, soff, st) || upload(P, &P.d_s2m_seg, ssegs, st) ||
      upload(P, &P.d_x_items, xitems, st) || upload(P, &P.d_x_off, xoff, st) || upload(P, &P.d_x_seg, xsegs, st))
    return -3;
  mark("s2m items");
  // ---- dense-algebra launches
  const int w_sq = ggs_tile_width(kp, kp), w_kn = ggs_tile_width(kp, np), w_nk = ggs_tile_width(np, kp);
  if (make_launch(P, P.g_s2m, sgroup, w_kn, st) || make_launch(P, P.g_x, xgroup, w_kn, st) ||
      make_launch(P, P.g_l2t, lgroups, w_nk, st) || make_launch(P, P.g_w, wgroups, w_nk, st))
    return -3;
  // M2L.  Every V pair runs in the sibling-class kernel: as a step of its sibling group's
  // column (full or masked class), or as a one-operator pseudo-class column.
  {
    auto anchor = [&](int b, int out[3]) {
      uint64_t k = T.key[b];
      out[0] = out[1] = out[2] = 0;
      for (int bit = 0; bit < 21; ++bit) {
        out[0] |= (int)((k >> (3 * bit + 2)) & 1) << bit;
        out[1] |= (int)((k >> (3 * bit + 1)) & 1) << bit;
        out[2] |= (int)((k >> (3 * bit)) & 1) << bit;
      }
    };
    // class table: class = didx * 8 + a; record = nvalid, b[8], offset id[8].  Classes
    // 208 + o are one-operator pseudo-classes (C_o) carrying the pairs of sparse sibling
    // groups through the same kernel (column: target, src, -1 x 7)
    constexpr int kSib = 26 * 8, kCls = kSib + kNumOffsets;
    std::vector<int> classes(kCls * 17, -1);
    std::vector<int> nvalid(kCls, 0);
    for (int o = 0; o < kNumOffsets; ++o) {
      int* rec = &classes[(kSib + o) * 17];
      rec[0] = 1; rec[1] = 0; rec[9] = o;
      nvalid[kSib + o] = 1;
    }
    for (int lin = 0; lin < 27; ++lin) {
      if (lin == 13) continue;
      const int didx = lin < 13 ? lin : lin - 1;
      const int dl[3] = {lin / 9 - 1, (lin / 3) % 3 - 1, lin % 3 - 1};
      for (int a = 0; a < 8; ++a) {
        const int av[3] = {(a >> 2) & 1, (a >> 1) & 1, a & 1};
        int* rec = &classes[(didx * 8 + a) * 17];
        int nv = 0;
        for (int b = 0; b < 8; ++b) {
          const int bv[3] = {(b >> 2) & 1, (b >> 1) & 1, b & 1};
          int D[3], m = 0;
          for (int d = 0; d < 3; ++d) { D[d] = 2 * dl[d] + bv[d] - av[d]; m = std::max(m, std::abs(D[d])); }
          if (m <= 1) continue;
          int id = 0;  // lexicographic index in [-3,3]^3 \ [-1,1]^3
          for (int i = -3; i <= 3; ++i)
            for (int j = -3; j <= 3; ++j)
              for (int l = -3; l <= 3; ++l) {
                if (std::max(std::abs(i), std::max(std::abs(j), std::abs(l))) <= 1) continue;
                if (i == D[0] && j == D[1] && l == D[2]) { rec[1 + nv] = b; rec[9 + nv] = id; }
                ++id;
              }
          ++nv;
        }
        rec[0] = nv;
        nvalid[didx * 8 + a] = nv;
      }
    }
    // V pairs -> CSR by target, then sibling groups per (target, Q)
    std::vector<int> vcnt(nb + 1, 0);
    for (auto& v : V) ++vcnt[v.x + 1];
    for (int b = 0; b < nb; ++b) vcnt[b + 1] += vcnt[b];
    std::vector<int4> vby(V.size());
    {
      std::vector<int> fill(vcnt.begin(), vcnt.end() - 1);
      for (auto& v : V) vby[fill[v.x]++] = v;
    }
    // Sibling groups (target B, source parent Q) with only some of Q's V-children present
    // (surface trees) become columns of a *masked* class — the class's steps restricted to
    // the present children (same kernel, no absent-child GEMM steps, one RED row per
    // column) — when that (class, mask) gathers at least mask_min columns; the rest go in
    // runs by the cost model below (the masked class of the run's union of masks, or
    // one-operator pseudo-classes per pair).
    const int NTs = sib_tile_width(kp, P.lr.on && P.lr.rp <= 32);  // (k_m2l_lr2 takes rp 16 / 32)
    // 256 measured best of 16-2048 (round 1, a since-retired environment switch): C4 M2L 6.50 -> 5.61 ms, C5 29.0 ->
    // 28.0 ms; C3 neutral (below ~512 its sparse masks split into partly filled tiles)
    constexpr int mask_min = 256;
    struct SibGroup { int b, cls, mask, cnt; int src[8]; };
    std::vector<SibGroup> sgs;
    sgs.reserve(V.size() / 4 + 16);
    std::vector<int> mcount(kSib * 256, 0);
    // integer anchors of every box (its coordinates at its own level), once
    std::vector<int> anc(3 * (size_t)nb);
#pragma omp parallel for schedule(static)
    for (int b = 0; b < nb; ++b) anchor(b, &anc[3 * (size_t)b]);
    for (int b = 0; b < nb; ++b) {
      const int e0 = vcnt[b], e1 = vcnt[b + 1];
      if (e0 == e1 || !inD(b)) continue;
      P.nV_local += e1 - e0;
      for (int e = e0; e < e1; ++e)  // algorithmic flops: 2 k^2 (dense core) or 4 k r_o (stage 2)
        P.m2l_flops += P.lr.on ? 4.0 * P.k * P.tables.ranks[vby[e].z] : 2.0 * P.k * P.k;
      const int* ap = &anc[3 * (size_t)T.parent[b]];
      const int a = (int)(T.key[b] & 7);
      // one group per distinct source parent Q (<= 26; Q's offset from parent(b) identifies
      // it), in order of first appearance
      SibGroup gq[27];
      int order[27], nq = 0;
      bool used[27] = {};
      for (int e = e0; e < e1; ++e) {
        const int src = vby[e].y;
        const int* aq = &anc[3 * (size_t)T.parent[src]];
        const int lin = (aq[0] - ap[0] + 1) * 9 + (aq[1] - ap[1] + 1) * 3 + (aq[2] - ap[2] + 1);
        if (!used[lin]) {
          used[lin] = true;
          order[nq++] = lin;
          gq[lin] = SibGroup{b, (lin < 13 ? lin : lin - 1) * 8 + a, 0, 0, {-1, -1, -1, -1, -1, -1, -1, -1}};
        }
        SibGroup& g = gq[lin];
        const int cb = (int)(T.key[src] & 7);
        g.src[cb] = src;
        g.mask |= 1 << cb;
        ++g.cnt;
      }
      for (int i = 0; i < nq; ++i) {
        ++mcount[gq[order[i]].cls * 256 + gq[order[i]].mask];
        sgs.push_back(gq[order[i]]);
      }
    }
    mark("m2l groups");
    std::vector<int> full_mask(kSib, 0);
    for (int c = 0; c < kSib; ++c)
      for (int j = 0; j < classes[c * 17]; ++j) full_mask[c] |= 1 << classes[c * 17 + 1 + j];
    std::vector<int> vclass(kSib * 256, -1);  // (class, mask) -> masked class id
    std::vector<std::vector<int>> cls_cols(kCls);  // column records (9 ints) per class
    auto add_col = [&](int c, const SibGroup& g) {
      auto& cc = cls_cols[c];
      cc.push_back(g.b);
      for (int j = 0; j < 8; ++j) cc.push_back(g.src[j]);
    };
    auto masked_class = [&](int cls, int mask) -> int {  // the full class's steps whose child is present
      int& id = vclass[cls * 256 + mask];
      if (id < 0) {
        id = (int)cls_cols.size();
        cls_cols.emplace_back();
        std::vector<int> rec(17, -1);
        const int* fr = &classes[cls * 17];
        int nv = 0;
        for (int j = 0; j < fr[0]; ++j)
          if (mask >> fr[1 + j] & 1) { rec[1 + nv] = fr[1 + j]; rec[9 + nv] = fr[9 + j]; ++nv; }
        rec[0] = nv;
        classes.insert(classes.end(), rec.begin(), rec.end());
        nvalid.push_back(nv);
      }
      return id;
    };
    std::vector<std::vector<int>> sparse(kSib);  // per class: its remaining sparse groups
    for (int i = 0; i < (int)sgs.size(); ++i) {
      const SibGroup& g = sgs[i];
      if (g.mask == full_mask[g.cls]) add_col(g.cls, g);
      else if (mcount[g.cls * 256 + g.mask] >= mask_min) add_col(masked_class(g.cls, g.mask), g);
      else sparse[g.cls].push_back(i);
    }
    // The sparse groups of a class, ordered by mask, in runs of one tile: a run becomes
    // columns of the masked class of its masks' union (absent children inside the union
    // are zero GEMM columns; one RED row per column) or one-operator pseudo-class columns
    // (one RED row per pair), whichever the cost model prices lower.  Cost per column
    // (FP64 peak 37 TF/s, fp64 L2 RED 5.2e11/s; the RED weight 0.5 is the measured best of
    // 0.25 / 0.5 / 1 / 2 over C3-C5 in round 1).
    // (round 2, with the runs: 0.25 / 0.5 / 1 / 2 / 4 / all-union: C3 M2L 1.966 / 1.976 /
    // 2.009 / 2.049 / 2.093 / 2.152 ms, C4 5.42-5.48 — the union's zero columns cost more
    // than the REDs they save)
    constexpr double red_scale = 0.5;
    const double Gc = 2.0 * kp * kp / 37e12, Rr = red_scale * kp / 5.2e11;
    for (int c = 0; c < kSib; ++c) {
      std::vector<int>& sp = sparse[c];
      std::stable_sort(sp.begin(), sp.end(), [&](int x, int y) { return sgs[x].mask < sgs[y].mask; });
      for (size_t r0 = 0; r0 < sp.size(); r0 += NTs) {
        const size_t r1 = std::min(sp.size(), r0 + NTs);
        int u = 0, pairs = 0;
        for (size_t r = r0; r < r1; ++r) { u |= sgs[sp[r]].mask; pairs += sgs[sp[r]].cnt; }
        const double cu = (double)(r1 - r0) * (__builtin_popcount(u) * Gc + Rr), cp = pairs * (Gc + Rr);
        if (cu <= cp) {
          const int id = u == full_mask[c] ? c : masked_class(c, u);
          for (size_t r = r0; r < r1; ++r) add_col(id, sgs[sp[r]]);
          continue;
        }
        for (size_t r = r0; r < r1; ++r) {
          const SibGroup& g = sgs[sp[r]];
          for (int j = 0; j < 8; ++j) {
            if (g.src[j] < 0) continue;
            int o = -1;  // the pair's offset id: the class step of child j
            for (int t = 0; t < classes[g.cls * 17]; ++t)
              if (classes[g.cls * 17 + 1 + t] == j) o = classes[g.cls * 17 + 9 + t];
            auto& cc = cls_cols[kSib + o];  // a one-operator pseudo-class column
            cc.push_back(g.b);
            cc.push_back(g.src[j]);
            for (int t = 1; t < 8; ++t) cc.push_back(-1);
          }
        }
      }
    }
    mark("m2l classes");
    if (std::getenv("KIFMM_DEBUG_M2L")) {  // diagnostics: columns per class kind
      int64_t full = 0, masked = 0, pseudo = 0;
      for (size_t c = 0; c < cls_cols.size(); ++c) {
        const int64_t n = cls_cols[c].size() / 9;
        if ((int)c < kSib) full += n; else if ((int)c < kCls) pseudo += n; else masked += n;
      }
      std::fprintf(stderr, "m2l columns: full-class %lld masked %lld (classes %zu) pseudo %lld; groups %zu\n",
                   (long long)full, (long long)masked, cls_cols.size() - kCls, (long long)pseudo, sgs.size());
    }
    P.m2l_exec_flops = 0;
    const int ncls = (int)cls_cols.size();
    for (int cls = 0; cls < ncls; ++cls) P.m2l_exec_flops += (double)nvalid[cls] * (cls_cols[cls].size() / 9) * 2.0 * P.k * P.k;
    // sibling tiles: per class, columns in target order, NT columns per tile.  Two launches:
    // columns whose sources are all complete on this rank after its own M2M ("local": every
    // present source box lies in the owned range) and the rest (ghost or straddling sources,
    // complete only after the allreduce and the ghost exchange).  NCCL plans run the local
    // tiles while the exchanges are in flight (matvec_device); one rank: all local.
    auto build_tiles = [&](bool ghost, SibLaunch& L) -> int {
      std::vector<int> cols;
      std::vector<int4> tiles;
      for (int cls = 0; cls < ncls; ++cls) {
        const auto& cc = cls_cols[cls];
        const int ncol = (int)cc.size() / 9;
        const int base = (int)cols.size() / 9;
        for (int c = 0; c < ncol; ++c) {
          bool local = true;
          for (int j = 1; j < 9; ++j) {
            const int src = cc[(size_t)c * 9 + j];
            if (src >= 0 && !Dp.full[src]) local = false;
          }
          if (local != ghost) cols.insert(cols.end(), cc.begin() + (size_t)c * 9, cc.begin() + (size_t)(c + 1) * 9);
        }
        const int nc = (int)cols.size() / 9 - base;
        for (int c = 0; c < nc; c += NTs) tiles.push_back(make_int4(cls, base + c, std::min(NTs, nc - c), 0));
      }
      // longest tiles first (the kernel hands tiles out dynamically: LPT order balances the
      // SMs; a Morton-window order for L2 locality measured no better on C2 / C3 / C5;
      // class-major order for stage 2 neither)
      std::stable_sort(tiles.begin(), tiles.end(), [&](const int4& a, const int4& b) {
        return nvalid[a.x] * a.z > nvalid[b.x] * b.z;
      });
      L.ntiles = (int)tiles.size();
      L.ncols = (int)cols.size() / 9;
      if (upload(P, &L.d_tiles, tiles, st) || upload(P, &L.d_cols, cols, st) ||
          upload(P, &L.d_counter, std::vector<int>(1, 0), st))
        return -3;
      return 0;
    };
    if (build_tiles(false, P.g_m2l_sib) || build_tiles(true, P.g_m2l_sib_ghost) ||
        upload(P, &P.g_m2l_sib.d_classes, classes, st))
      return -3;
    P.g_m2l_sib_ghost.d_classes = P.g_m2l_sib.d_classes;
    mark("m2l tiles");
  }
  mark("m2l schedule");
  // M2M per child level (finest first) and L2L per parent level (coarsest first), by octant
  P.g_m2m.clear();
  P.g_l2l.clear();
  for (int l = T.nlevels - 1; l >= 3; --l) {
    std::vector<PairGroup> groups(8);
    for (int o = 0; o < 8; ++o) groups[o] = PairGroup{o, 0.5, {}};
    for (int b = T.level_begin[l]; b < T.level_begin[l + 1]; ++b)
      if (inD(b)) groups[T.key[b] & 7].pairs.push_back(make_int2(b, T.parent[b]));
    P.g_m2m.emplace_back();
    if (make_launch(P, P.g_m2m.back(), groups, w_sq, st)) return -3;
  }
  for (int l = 2; l + 1 < T.nlevels; ++l) {
    std::vector<PairGroup> groups(8);
    for (int o = 0; o < 8; ++o) groups[o] = PairGroup{o, 1.0, {}};
    for (int b = T.level_begin[l + 1]; b < T.level_begin[l + 2]; ++b)
      if (inD(b)) groups[T.key[b] & 7].pairs.push_back(make_int2(T.parent[b], b));
    P.g_l2l.emplace_back();
    if (make_launch(P, P.g_l2l.back(), groups, w_sq, st)) return -3;
  }
  // ---- work buffers (padding columns stay zero)
  auto zalloc = [&](double** p, size_t cnt) -> int {
    KIFMM_CUDA(cudaMalloc((void**)p, sizeof(double) * std::max<size_t>(cnt, 1)));
    P.allocations.push_back(*p);
    KIFMM_CUDA(cudaMemsetAsync(*p, 0, sizeof(double) * std::max<size_t>(cnt, 1), st));
    return 0;
  };
  // q^' has one extra row, never written: the zero row absent sibling sources point at (the
  // M2L gathers every column row with one bulk copy)
  if (zalloc(&P.d_qhat, (size_t)(nb + 1) * kp) || zalloc(&P.d_lhat, (size_t)nb * kp) ||
      zalloc(&P.d_chk_s2m, P.leaf_s2m ? 1 : (size_t)P.n_s2m * np) || zalloc(&P.d_chk_x, P.leaf_x ? 1 : (size_t)P.n_xnd * np) ||
      zalloc(&P.d_eqd_l2t, (size_t)n_l2t * np) || zalloc(&P.d_eqd_w, (size_t)n_wnd * np) ||
      zalloc(&P.d_pot_near, T.N) || zalloc(&P.d_pot_far, T.N) || zalloc(&P.d_io, 2 * T.N))
    return -3;
  // ---- exchange buffers (empty on one rank)
  auto make_exchange = [&](Exchange& E, int row, const std::vector<int>& sl, const std::vector<int>& so,
                           const std::vector<int>& rlst, const std::vector<int>& ro) -> int {
    E.row = row;
    E.send_off = so.empty() ? std::vector<int>(Dp.nranks + 1, 0) : so;
    E.recv_off = ro.empty() ? std::vector<int>(Dp.nranks + 1, 0) : ro;
    E.nsend = (int)sl.size();
    E.nrecv = (int)rlst.size();
    if (upload(P, &E.d_send_idx, sl, st) || upload(P, &E.d_recv_idx, rlst, st)) return -3;
    if (zalloc(&E.d_send, (size_t)E.nsend * row) || zalloc(&E.d_recv, (size_t)E.nrecv * row)) return -3;
    return 0;
  };
  if (make_exchange(P.xq, kp, Dp.q_send, Dp.q_send_off, Dp.q_recv, Dp.q_recv_off) ||
      make_exchange(P.xd, 1, Dp.d_send, Dp.d_send_off, Dp.d_recv, Dp.d_recv_off))
    return -3;
  P.n_straddle = Dp.nranks > 1 ? (int)Dp.straddle.size() : 0;
  {
    std::vector<int> sl = Dp.nranks > 1 ? Dp.straddle : std::vector<int>();
    if (upload(P, &P.d_straddle, sl, st) || zalloc(&P.d_straddle_buf, (size_t)P.n_straddle * kp)) return -3;
  }
  mark("m2m/l2l+buffers");
  // X-list operators (after S2M / L2T, same reserve; BEM: always, its runtime integrals are slow)
  {
    int64_t xcnt = 0;
    std::vector<int64_t> xo(xitems.size() + 1, 0);
    for (size_t r = 0; r < xitems.size(); ++r) xo[r + 1] = xo[r] + (int64_t)xsegs[r].w * kp;
    xcnt = xo.back();
    size_t fr = 0, tot = 0;
    KIFMM_CUDA(cudaMemGetInfo(&fr, &tot));
    const double used = (P.leaf_s2m ? 1.0 : 0.0) + (P.leaf_l2t ? 1.0 : 0.0);
    const double budget = (double)fr - leaf_op_reserve(tot) - used * (double)(Dp.own_hi - Dp.own_lo) * kp * sizeof(double);
    P.leaf_x = !xitems.empty() && (P.leaf_ops_opt > 0 || P.bem ||
                                   (P.leaf_ops_opt < 0 && (double)xcnt * sizeof(double) <= budget));
    if (P.leaf_x) {
      if (zalloc(&P.d_x_mat, (size_t)xcnt) || upload(P, &P.d_x_moff, xo, st)) return -3;
      P.leaf_op_bytes += xcnt * (int64_t)sizeof(double);
      std::vector<int4> xt;  // rows are grouped by target (X list order (tgt, src))
      for (size_t r = 0; r < xitems.size();) {
        size_t e = r;
        while (e < xitems.size() && xitems[e].x == xitems[r].x) ++e;
        xt.push_back(make_int4(xitems[r].x, (int)r, (int)e, 0));
        r = e;
      }
      P.n_xt = (int)xt.size();
      if (upload(P, &P.d_xt_items, xt, st)) return -3;
    }
  }
  if (P.leaf_x && build_x_ops(P, st)) return -3;
  mark("x operators");
  if (P.leaf_s2m || P.leaf_l2t) {
    const size_t cnt = (size_t)(Dp.own_hi - Dp.own_lo) * kp;
    if (P.leaf_s2m && zalloc(&P.d_s2m_mat, cnt)) return -3;
    if (P.leaf_l2t && zalloc(&P.d_l2t_mat, cnt)) return -3;
    P.leaf_op_bytes += (int64_t)((P.leaf_s2m ? 1 : 0) + (P.leaf_l2t ? 1 : 0)) * cnt * sizeof(double);
    if (build_leaf_ops(P, st)) return -3;
  }
  mark("leaf operators");
  // ---- work lists of the bulk-copy streamed GEMVs (stream.cu): one rank (the streamed
  // weights are a sorted copy of the owned densities: no ghosts), S2M / X operators built
  P.stream_ok = false;
  if (Dp.nranks == 1 && !P.bem && P.leaf_s2m && (xitems.empty() || P.leaf_x)) {
    std::vector<int4> s2m, xw;
    s2m.reserve(sitems.size());
    for (const int4& it : sitems) {
      const int b = it.x;
      s2m.push_back(make_int4(T.pbeg[b] - Dp.own_lo, npts(b), T.pbeg[b], b));
    }
    std::sort(s2m.begin(), s2m.end(), [](const int4& a, const int4& b) { return a.x < b.x; });
    int64_t xrow = 0;  // X operator rows: items in X-list order, grouped by target
    for (size_t r = 0; r < xitems.size(); ++r) {
      xw.push_back(make_int4((int)xrow, xsegs[r].w, xsegs[r].y, xitems[r].x));
      xrow += xsegs[r].w;
    }
    if (xrow > INT32_MAX || stream_plan(P, P.sw_s2m, s2m, st) || stream_plan(P, P.sw_x, xw, st) ||
        zalloc(&P.d_q_sorted, (size_t)T.N + 2))
      return -3;
    P.stream_ok = true;
  }
  mark("stream lists");
  KIFMM_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int upload_tables(Plan& P) {
  const HostTables& H = P.tables;
  const int k = H.k, n = H.n, kp = P.kp, np = P.np;
  std::vector<double> C((size_t)316 * kp * kp, 0.0), M((size_t)8 * kp * kp, 0.0), L((size_t)8 * kp * kp, 0.0);
  std::vector<double> S((size_t)kp * np, 0.0), Ut((size_t)kp * np, 0.0), Tt((size_t)np * kp, 0.0), Ue((size_t)np * kp, 0.0);
  for (int o = 0; o < 316; ++o)
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) C[((size_t)o * kp + a) * kp + b] = H.C[((size_t)o * k + a) * k + b];
  for (int o = 0; o < 8; ++o)
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        M[((size_t)o * kp + a) * kp + b] = H.M[((size_t)o * k + a) * k + b];
        L[((size_t)o * kp + a) * kp + b] = H.L[((size_t)o * k + a) * k + b];
      }
  for (int a = 0; a < k; ++a)
    for (int i = 0; i < n; ++i) {
      S[(size_t)a * np + i] = H.S[(size_t)a * n + i];
      Ut[(size_t)a * np + i] = H.U[(size_t)i * k + a];
      Tt[(size_t)i * kp + a] = H.T[(size_t)i * k + a];
      Ue[(size_t)i * kp + a] = H.U[(size_t)i * k + a];
    }
  cudaStream_t st = P.stream;
  if (upload(P, &P.d_C, C, st) || upload(P, &P.d_M, M, st) || upload(P, &P.d_L, L, st) || upload(P, &P.d_S, S, st) ||
      upload(P, &P.d_Ut, Ut, st) || upload(P, &P.d_T, Tt, st) || upload(P, &P.d_Ue, Ue, st))
    return -3;
  if (upload(P, &P.d_surf, H.surf, st)) return -3;
  // stage-2 factors, zero padded to kp x rp / rp x kp (rp = max rank rounded up to 16)
  P.lr = LowRank();
  if (!H.ranks.empty()) {
    const int rp = std::max(16, (H.rmax + 15) / 16 * 16);
    std::vector<double> Uh((size_t)316 * kp * rp, 0.0), Vh((size_t)316 * rp * kp, 0.0);
    for (int o = 0; o < 316; ++o) {
      const int r = H.ranks[o];
      for (int a = 0; a < k; ++a)
        for (int c = 0; c < r; ++c) Uh[((size_t)o * kp + a) * rp + c] = H.Uh[o][(size_t)a * r + c];
      for (int c = 0; c < r; ++c)
        for (int b = 0; b < k; ++b) Vh[((size_t)o * rp + c) * kp + b] = H.Vh[o][(size_t)c * k + b];
    }
    P.lr.on = true;
    P.lr.rp = rp;
    if (upload(P, &P.lr.d_Uh, Uh, st) || upload(P, &P.lr.d_Vh, Vh, st) || upload(P, &P.lr.d_rank, H.ranks, st))
      return -3;
  }
  KIFMM_CUDA(cudaStreamSynchronize(st));
  return 0;
}

}  // namespace kifmm
