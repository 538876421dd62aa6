// =============================================================================
// KIFMM ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the point-source
// SVD-compressed KIFMM matvec of arXiv 1211.2517, in FP64.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// this library.  It shares no code with paper_1211_2517_b200/ (the product).
//
// Paper anchors ("P:n" = /root/reference/PAPER.md line n):
//   eq_eval           P:65-77   p_i = sum_j G(x_i, y_j) q_j
//   kernel            P:374     G(x, y) = 1 / (4 pi |x - y|)
//   double layer      P:458-464 dG/dn(y) in S2T and the first S2M step (eq-doubles2m)
//   octree            P:79-84   subdivide into 8 until <= s points per leaf
//   near / far field  P:86-88   N^C: same-level cubes sharing a vertex; I^C = F^C \ F^B
//   surfaces          P:109-113 UE, DC at (1+d) r; UC, DE at (3-2d) r
//   translations      P:117-159 S2M, M2M, M2L, L2L, L2T; p = T L K M S q
//   compression       P:205-235 K ~ U (U^T K R) R^T; homogeneous scaling
//   pass operators    P:315-355 M~ = R^T M R, S~ = R^T S, L~ = U^T L U, T~ = T U
//   algorithm         P:466-522 setup, upward (postorder), downward (preorder), near
// Readings where the paper is silent:
//   O1 root cube + 21-bit quantisation, O3 adaptive tree (subdivide iff count > s),
//   O5 adaptive U/V/W/X lists + the W/X "direct" shortcut rule, Q1 pairs with r == 0
//   contribute 0, Q15 level normalisation q^' = q^/r_l (M2L scale-free).
//
// Operator tables (U, C_delta, S', T', M~_o, L~_o) are computed by
// oracle/precompute.py (numpy) and passed in; the passes here follow O7-O10.
// Built with -O2 -ffp-contract=off -fopenmp.  Parallel loops run over target
// boxes/points only; every per-target reduction is in a fixed (canonical) order.
// =============================================================================
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

namespace {

const int MAXLEV = 21;  // O1: 21 bits per coordinate

inline double G(double x0, double x1, double x2, double y0, double y1, double y2) {
  // P:374 G(x,y) = 1/(4 pi |x-y|); pairs with r == 0 contribute 0 (reading Q1).
  double dx = x0 - y0, dy = x1 - y1, dz = x2 - y2;
  double r = std::sqrt(dx * dx + dy * dy + dz * dz);
  if (r == 0.0) return 0.0;
  return 1.0 / (4.0 * M_PI * r);
}

inline double Gdl(double x0, double x1, double x2, double y0, double y1, double y2, double n0, double n1, double n2) {
  // double-layer kernel dG/dn(y) = (x - y) . n(y) / (4 pi |x - y|^3) (eq-doubles2m);
  // pairs with r == 0 contribute 0 (reading Q1)
  double dx = x0 - y0, dy = x1 - y1, dz = x2 - y2;
  double r = std::sqrt(dx * dx + dy * dy + dz * dz);
  if (r == 0.0) return 0.0;
  return (dx * n0 + dy * n1 + dz * n2) / (4.0 * M_PI * r * r * r);
}

// ---- BEM elements: flat triangles, piecewise-constant density, collocation at
// centroids.  Element integral of the single-layer kernel, reading R-BEM (the
// paper specifies no quadrature):
//   self (x = the element's own collocation point): the analytic flat-triangle value
//        int_T 1/|x - y| dA = sum over edges of  h_e ln((s2 + r2) / (s1 + r1))
//        (x in the plane: h_e = distance from x to the edge line, s1, s2 the endpoints'
//        coordinates along the edge measured from the foot of the perpendicular, r1, r2
//        their distances to x), divided by 4 pi;
//   else if |x - centroid| > 2 diam (diam = longest edge): Dunavant's 6-point degree-4 rule;
//   else: split into 4 (edge midpoints) and recurse, at depth 8 the 6-point rule.
struct Tri {
  double v[3][3];
};

inline double tri_area(const Tri& T) {
  double a[3], b[3];
  for (int d = 0; d < 3; ++d) { a[d] = T.v[1][d] - T.v[0][d]; b[d] = T.v[2][d] - T.v[0][d]; }
  double c0 = a[1] * b[2] - a[2] * b[1], c1 = a[2] * b[0] - a[0] * b[2], c2 = a[0] * b[1] - a[1] * b[0];
  return 0.5 * std::sqrt(c0 * c0 + c1 * c1 + c2 * c2);
}

inline double tri_diam(const Tri& T) {
  double m = 0;
  for (int e = 0; e < 3; ++e) {
    const double* p = T.v[e];
    const double* q = T.v[(e + 1) % 3];
    double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
    m = std::max(m, std::sqrt(dx * dx + dy * dy + dz * dz));
  }
  return m;
}

// Dunavant (1985) degree-4 rule: barycentric (a, a, 1 - 2a) and permutations
double tri_rule6(const Tri& T, const double x[3]) {
  static const double A[2] = {0.445948490915965, 0.091576213509771};
  static const double W[2] = {0.223381589678011, 0.109951743655322};
  double acc = 0;
  for (int g = 0; g < 2; ++g)
    for (int perm = 0; perm < 3; ++perm) {
      double l[3] = {A[g], A[g], A[g]};
      l[perm] = 1.0 - 2.0 * A[g];
      double y[3];
      for (int d = 0; d < 3; ++d) y[d] = l[0] * T.v[0][d] + l[1] * T.v[1][d] + l[2] * T.v[2][d];
      acc += W[g] * G(x[0], x[1], x[2], y[0], y[1], y[2]);
    }
  return acc * tri_area(T);
}

double tri_self(const Tri& T, const double x[3]) {
  double acc = 0;
  for (int e = 0; e < 3; ++e) {
    const double* p1 = T.v[e];
    const double* p2 = T.v[(e + 1) % 3];
    double t[3], L = 0;
    for (int d = 0; d < 3; ++d) { t[d] = p2[d] - p1[d]; L += t[d] * t[d]; }
    L = std::sqrt(L);
    for (int d = 0; d < 3; ++d) t[d] /= L;
    double s1 = 0, s2 = 0, r1 = 0, r2 = 0;
    for (int d = 0; d < 3; ++d) {
      s1 += (p1[d] - x[d]) * t[d];
      s2 += (p2[d] - x[d]) * t[d];
      r1 += (p1[d] - x[d]) * (p1[d] - x[d]);
      r2 += (p2[d] - x[d]) * (p2[d] - x[d]);
    }
    r1 = std::sqrt(r1);
    r2 = std::sqrt(r2);
    const double h = std::sqrt(std::max(0.0, r1 * r1 - s1 * s1));
    acc += h * std::log((s2 + r2) / (s1 + r1));
  }
  return acc / (4.0 * M_PI);
}

double tri_integral(const Tri& T, const double x[3], int depth) {
  double c[3];
  for (int d = 0; d < 3; ++d) c[d] = (T.v[0][d] + T.v[1][d] + T.v[2][d]) / 3.0;
  double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
  const double dist = std::sqrt(dx * dx + dy * dy + dz * dz);
  if (depth >= 8 || dist > 2.0 * tri_diam(T)) return tri_rule6(T, x);
  double m[3][3];
  for (int e = 0; e < 3; ++e)
    for (int d = 0; d < 3; ++d) m[e][d] = 0.5 * (T.v[e][d] + T.v[(e + 1) % 3][d]);
  // children: corner 0 (v0, m01, m20), corner 1 (m01, v1, m12), corner 2 (m20, m12, v2), centre (m01, m12, m20)
  Tri ch[4];
  for (int d = 0; d < 3; ++d) {
    ch[0].v[0][d] = T.v[0][d]; ch[0].v[1][d] = m[0][d]; ch[0].v[2][d] = m[2][d];
    ch[1].v[0][d] = m[0][d]; ch[1].v[1][d] = T.v[1][d]; ch[1].v[2][d] = m[1][d];
    ch[2].v[0][d] = m[2][d]; ch[2].v[1][d] = m[1][d]; ch[2].v[2][d] = T.v[2][d];
    ch[3].v[0][d] = m[0][d]; ch[3].v[1][d] = m[1][d]; ch[3].v[2][d] = m[2][d];
  }
  double acc = 0;
  for (int i = 0; i < 4; ++i) acc += tri_integral(ch[i], x, depth + 1);
  return acc;
}

struct Box {
  int level;
  uint64_t key;     // Morton prefix at `level` (3*level bits)
  int anchor[3];    // integer cube index at `level`
  int parent;
  int child[8];     // by octant (x_bit<<2 | y_bit<<1 | z_bit), -1 if empty
  int pbeg, pend;   // sorted point range
  bool leaf;
  double c[3];      // centre
  double r;         // halfwidth r_l = r0 / 2^l
};

uint64_t interleave(uint32_t ux, uint32_t uy, uint32_t uz) {
  uint64_t k = 0;
  for (int b = 0; b < MAXLEV; ++b) {
    k |= (uint64_t)((ux >> b) & 1) << (3 * b + 2);
    k |= (uint64_t)((uy >> b) & 1) << (3 * b + 1);
    k |= (uint64_t)((uz >> b) & 1) << (3 * b);
  }
  return k;
}

struct Plan {
  int64_t N = 0;
  int s = 0;
  int wx_direct_max = 0;
  double lo_root[3], r0, scale;
  std::vector<double> xs;        // sorted points, 3 per point
  std::vector<int32_t> perm;     // sorted index -> caller index
  std::vector<Box> boxes;        // level-major, key order within a level
  std::vector<int> level_begin;  // box index where each level starts (+ end sentinel)
  std::vector<std::unordered_map<uint64_t, int>> lookup;  // per level: key -> box
  // lists (all in canonical order)
  std::vector<std::vector<int>> U;                    // per box (leaves only)
  std::vector<std::vector<std::pair<int, int>>> V;    // per box: (src, offset id)
  std::vector<std::vector<int>> W;                    // per box (leaves): src boxes
  std::vector<std::vector<int>> X;                    // per box: src leaves
  int nlevels() const { return (int)level_begin.size() - 1; }
};

int find_box(const Plan& P, int level, int ax, int ay, int az) {
  int lim = 1 << level;
  if (ax < 0 || ay < 0 || az < 0 || ax >= lim || ay >= lim || az >= lim) return -1;
  if (level >= (int)P.lookup.size()) return -1;
  auto it = P.lookup[level].find(interleave(ax, ay, az));
  return it == P.lookup[level].end() ? -1 : it->second;
}

// closed boxes intersect, compared in level-21 integer coordinates (O5)
bool adjacent(const Box& a, const Box& b) {
  for (int d = 0; d < 3; ++d) {
    int64_t alo = (int64_t)a.anchor[d] << (MAXLEV - a.level), ahi = (int64_t)(a.anchor[d] + 1) << (MAXLEV - a.level);
    int64_t blo = (int64_t)b.anchor[d] << (MAXLEV - b.level), bhi = (int64_t)(b.anchor[d] + 1) << (MAXLEV - b.level);
    if (alo > bhi || blo > ahi) return false;
  }
  return true;
}

// offset id of delta in the lexicographic table of [-3,3]^3 \ [-1,1]^3 (316 entries)
int offset_id(int dx, int dy, int dz) {
  int id = 0;
  for (int i = -3; i <= 3; ++i)
    for (int j = -3; j <= 3; ++j)
      for (int k = -3; k <= 3; ++k) {
        if (std::max(std::abs(i), std::max(std::abs(j), std::abs(k))) <= 1) continue;
        if (i == dx && j == dy && k == dz) return id;
        ++id;
      }
  return -1;
}

void build_tree(Plan& P, const double* pts) {
  const int64_t N = P.N;
  // O1: root cube and quantisation
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) { lo[d] = pts[d]; hi[d] = pts[d]; }
  for (int64_t i = 0; i < N; ++i)
    for (int d = 0; d < 3; ++d) { lo[d] = std::min(lo[d], pts[3 * i + d]); hi[d] = std::max(hi[d], pts[3 * i + d]); }
  double ext = 0;
  for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
  double r0 = ext / 2.0 * (1.0 + 1e-6);
  if (r0 == 0.0) r0 = 1.0;
  P.r0 = r0;
  P.scale = (double)(1u << MAXLEV) / (2.0 * r0);
  for (int d = 0; d < 3; ++d) P.lo_root[d] = (lo[d] + hi[d]) / 2.0 - r0;
  std::vector<uint64_t> key(N);
  for (int64_t i = 0; i < N; ++i) {
    uint32_t u[3];
    for (int d = 0; d < 3; ++d) {
      double t = std::floor((pts[3 * i + d] - P.lo_root[d]) * P.scale);
      if (t < 0) t = 0;
      if (t > (double)((1u << MAXLEV) - 1)) t = (double)((1u << MAXLEV) - 1);
      u[d] = (uint32_t)t;
    }
    key[i] = interleave(u[0], u[1], u[2]);
  }
  // O2: stable order by key, ties by input index
  P.perm.resize(N);
  for (int64_t i = 0; i < N; ++i) P.perm[i] = (int32_t)i;
  std::stable_sort(P.perm.begin(), P.perm.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
  P.xs.resize(3 * N);
  std::vector<uint64_t> skey(N);
  for (int64_t i = 0; i < N; ++i) {
    for (int d = 0; d < 3; ++d) P.xs[3 * i + d] = pts[3 * (int64_t)P.perm[i] + d];
    skey[i] = key[P.perm[i]];
  }
  // O3: level by level; subdivide iff count > s and level < 21; only non-empty children
  P.boxes.clear();
  P.level_begin.clear();
  Box root{};
  root.level = 0; root.key = 0; root.anchor[0] = root.anchor[1] = root.anchor[2] = 0;
  root.parent = -1; root.pbeg = 0; root.pend = (int)N;
  P.boxes.push_back(root);
  P.level_begin.push_back(0);
  int lb = 0;
  for (int l = 0;; ++l) {
    int le = (int)P.boxes.size();
    bool any = false;
    for (int b = lb; b < le; ++b) {
      for (int o = 0; o < 8; ++o) P.boxes[b].child[o] = -1;
      const int pbeg = P.boxes[b].pbeg, pend = P.boxes[b].pend;
      P.boxes[b].leaf = !((pend - pbeg) > P.s && l < MAXLEV);
      if (P.boxes[b].leaf) continue;
      any = true;
      int sh = 3 * (MAXLEV - (l + 1));
      int i = pbeg;
      while (i < pend) {
        uint64_t ck = skey[i] >> sh;
        int j = i;
        while (j < pend && (skey[j] >> sh) == ck) ++j;
        Box C{};
        C.level = l + 1; C.key = ck; C.parent = b; C.pbeg = i; C.pend = j;
        for (int d = 0; d < 3; ++d) C.anchor[d] = 0;
        for (int bit = 0; bit <= l; ++bit) {
          C.anchor[0] |= (int)((ck >> (3 * bit + 2)) & 1) << bit;
          C.anchor[1] |= (int)((ck >> (3 * bit + 1)) & 1) << bit;
          C.anchor[2] |= (int)((ck >> (3 * bit)) & 1) << bit;
        }
        P.boxes[b].child[ck & 7] = (int)P.boxes.size();
        P.boxes.push_back(C);
        i = j;
      }
    }
    P.level_begin.push_back(le);
    lb = le;
    if (!any) break;
  }
  // box geometry: centre = lo_root + (2a+1) r_l (O3), r_l = r0 / 2^l
  for (Box& B : P.boxes) {
    B.r = std::ldexp(P.r0, -B.level);
    for (int d = 0; d < 3; ++d) B.c[d] = P.lo_root[d] + (double)(2 * (int64_t)B.anchor[d] + 1) * B.r;
  }
  P.lookup.assign(P.nlevels(), {});
  for (int b = 0; b < (int)P.boxes.size(); ++b) P.lookup[P.boxes[b].level][P.boxes[b].key] = b;
}

void build_lists(Plan& P) {
  const int nb = (int)P.boxes.size();
  P.U.assign(nb, {}); P.V.assign(nb, {}); P.W.assign(nb, {}); P.X.assign(nb, {});
  for (int b = 0; b < nb; ++b) {
    const Box& B = P.boxes[b];
    // V(B), level >= 2: children of colleagues of parent(B) not adjacent to B
    if (B.level >= 2) {
      const Box& Pa = P.boxes[B.parent];
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            int c = find_box(P, Pa.level, Pa.anchor[0] + dx, Pa.anchor[1] + dy, Pa.anchor[2] + dz);
            if (c < 0) continue;
            for (int o = 0; o < 8; ++o) {
              int a = P.boxes[c].child[o];
              if (a < 0 || adjacent(P.boxes[a], B)) continue;
              const Box& A = P.boxes[a];
              P.V[b].push_back({a, offset_id(A.anchor[0] - B.anchor[0], A.anchor[1] - B.anchor[1], A.anchor[2] - B.anchor[2])});
            }
          }
      std::sort(P.V[b].begin(), P.V[b].end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.second < y.second; });
    }
    if (!B.leaf) continue;
    // U(B): all leaves adjacent to B (any level), incl. B
    std::vector<int> u;
    std::vector<int> stack;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          int ax = B.anchor[0] + dx, ay = B.anchor[1] + dy, az = B.anchor[2] + dz;
          int lim = 1 << B.level;
          if (ax < 0 || ay < 0 || az < 0 || ax >= lim || ay >= lim || az >= lim) continue;
          int c = find_box(P, B.level, ax, ay, az);
          if (c >= 0) {
            stack.assign(1, c);
            while (!stack.empty()) {
              int x = stack.back(); stack.pop_back();
              const Box& Xb = P.boxes[x];
              if (Xb.leaf) { u.push_back(x); continue; }
              for (int o = 0; o < 8; ++o) {
                int ch = Xb.child[o];
                if (ch < 0) continue;
                if (adjacent(P.boxes[ch], B)) stack.push_back(ch);
                else if (x != b) P.W[b].push_back(ch);  // W(B): parent adjacent, child not (O5)
              }
            }
          } else {
            // coarser neighbour: first existing ancestor of the same-level cell
            for (int l = B.level - 1; l >= 0; --l) {
              int sh = B.level - l;
              int y = find_box(P, l, ax >> sh, ay >> sh, az >> sh);
              if (y >= 0) { if (P.boxes[y].leaf) u.push_back(y); break; }
            }
          }
        }
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    P.U[b] = u;
    std::sort(P.W[b].begin(), P.W[b].end());
  }
  // X(B) = {A : B in W(A)}
  for (int a = 0; a < nb; ++a)
    for (int w : P.W[a]) P.X[w].push_back(a);
  for (auto& x : P.X) std::sort(x.begin(), x.end());
}

// unit surface grid (O4): boundary nodes of the p^3 grid on [-1,1]^3, lexicographic
std::vector<double> surface(int p) {
  std::vector<double> g;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        int mn = std::min(i, std::min(j, k)), mx = std::max(i, std::max(j, k));
        if (mn != 0 && mx != p - 1) continue;
        g.push_back(-1.0 + 2.0 * i / (p - 1));
        g.push_back(-1.0 + 2.0 * j / (p - 1));
        g.push_back(-1.0 + 2.0 * k / (p - 1));
      }
  return g;
}

}  // namespace

extern "C" {

struct oracle_tables {
  int p, n, k;
  double d;
  const double* U;   // n x k, row-major
  const double* C;   // 316 x k x k
  const double* S;   // k x n   (S' = U^T pinv(E_u))
  const double* T;   // n x k   (T' = pinv(E_d) U)
  const double* M;   // 8 x k x k (M~_o)
  const double* L;   // 8 x k x k (L~_o)
};

// direct sum: out[t] = sum_j G(x_{tgt[t]}, x_j) q_j, j ascending, r == 0 skipped
void oracle_direct(int64_t N, const double* pts, const double* q, int64_t ntgt, const int64_t* tgt, double* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < ntgt; ++t) {
    const double* x = pts + 3 * tgt[t];
    double acc = 0;
    for (int64_t j = 0; j < N; ++j) acc += G(x[0], x[1], x[2], pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]) * q[j];
    out[t] = acc;
  }
}

// double-layer direct sum: out[t] = sum_j dG(x_{tgt[t]}, x_j)/dn(x_j) q_j (nrm: N x 3 normals)
void oracle_direct_dl(int64_t N, const double* pts, const double* nrm, const double* q, int64_t ntgt, const int64_t* tgt,
                      double* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < ntgt; ++t) {
    const double* x = pts + 3 * tgt[t];
    double acc = 0;
    for (int64_t j = 0; j < N; ++j)
      acc += Gdl(x[0], x[1], x[2], pts[3 * j], pts[3 * j + 1], pts[3 * j + 2], nrm[3 * j], nrm[3 * j + 1], nrm[3 * j + 2]) * q[j];
    out[t] = acc;
  }
}

// element integral of G over triangle tri (9 doubles) at x; self = 1: analytic (x = centroid)
double oracle_tri_integral(const double* tri, const double* x, int self) {
  Tri T;
  for (int e = 0; e < 3; ++e)
    for (int d = 0; d < 3; ++d) T.v[e][d] = tri[3 * e + d];
  return self ? tri_self(T, x) : tri_integral(T, x, 0);
}

// dense BEM collocation product: out[t] = sum_j A_{tgt[t], j} q_j with
// A_ij = int_Tj G(x_i, y) dy (analytic self term for j = i); x_i = pts (centroids)
void oracle_direct_bem(int64_t N, const double* pts, const double* tri, const double* q, int64_t ntgt,
                       const int64_t* tgt, double* out) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < ntgt; ++t) {
    const int64_t i = tgt[t];
    double acc = 0;
    for (int64_t j = 0; j < N; ++j) acc += oracle_tri_integral(tri + 9 * j, pts + 3 * i, j == i) * q[j];
    out[t] = acc;
  }
}

// dense collocation matrix A (N x N, row-major): A_ij = int_Tj G(x_i, y) dy
void oracle_bem_matrix(int64_t N, const double* pts, const double* tri, double* A) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = 0; j < N; ++j) A[i * N + j] = oracle_tri_integral(tri + 9 * j, pts + 3 * i, j == i);
}

void* oracle_plan(int64_t N, const double* pts, int s, int wx_direct_max) {
  Plan* P = new Plan();
  P->N = N; P->s = s; P->wx_direct_max = wx_direct_max;
  build_tree(*P, pts);
  build_lists(*P);
  return P;
}

void oracle_free(void* h) { delete (Plan*)h; }

// counts: 0 nboxes, 1 nleaves, 2 nlevels, 3 |U|, 4 |V|, 5 |W|, 6 |X|
int64_t oracle_count(void* h, int what) {
  Plan* P = (Plan*)h;
  int64_t c = 0;
  switch (what) {
    case 0: return (int64_t)P->boxes.size();
    case 1: for (auto& b : P->boxes) c += b.leaf; return c;
    case 2: return P->nlevels();
    case 3: for (auto& x : P->U) c += x.size(); return c;
    case 4: for (auto& x : P->V) c += x.size(); return c;
    case 5: for (auto& x : P->W) c += x.size(); return c;
    case 6: for (auto& x : P->X) c += x.size(); return c;
  }
  return -1;
}

// geom: lo_root[3], r0, scale
void oracle_export_tree(void* h, int32_t* level, uint64_t* key, int32_t* parent, int32_t* pbeg, int32_t* pend,
                        uint8_t* leaf, int32_t* perm, double* geom) {
  Plan* P = (Plan*)h;
  for (size_t b = 0; b < P->boxes.size(); ++b) {
    const Box& B = P->boxes[b];
    level[b] = B.level; key[b] = B.key; parent[b] = B.parent; pbeg[b] = B.pbeg; pend[b] = B.pend; leaf[b] = B.leaf;
  }
  std::memcpy(perm, P->perm.data(), sizeof(int32_t) * P->N);
  for (int d = 0; d < 3; ++d) geom[d] = P->lo_root[d];
  geom[3] = P->r0; geom[4] = P->scale;
}

// canonical list dumps.
//   U: (tgt, src) by (tgt, src)
//   V: (tgt, src, offset id) by (offset id, tgt)        [tgt order = (level, key)]
//   W: (tgt, src, direct) by (tgt, src);  X: (tgt, src, direct) by (tgt, src)
void oracle_export_lists(void* h, int32_t* U, int32_t* V, int32_t* W, int32_t* X) {
  Plan* P = (Plan*)h;
  int64_t i = 0;
  for (size_t b = 0; b < P->U.size(); ++b)
    for (int s : P->U[b]) { U[2 * i] = (int32_t)b; U[2 * i + 1] = s; ++i; }
  i = 0;
  {
    std::vector<std::array<int32_t, 3>> v;
    for (size_t b = 0; b < P->V.size(); ++b)
      for (auto& e : P->V[b]) v.push_back({e.second, (int32_t)b, e.first});
    std::sort(v.begin(), v.end());
    for (auto& e : v) { V[3 * i] = e[1]; V[3 * i + 1] = e[2]; V[3 * i + 2] = e[0]; ++i; }
  }
  auto npts = [&](int a) { return P->boxes[a].pend - P->boxes[a].pbeg; };
  i = 0;
  for (size_t b = 0; b < P->W.size(); ++b)
    for (int s : P->W[b]) { W[3 * i] = (int32_t)b; W[3 * i + 1] = s; W[3 * i + 2] = npts(s) <= P->wx_direct_max; ++i; }
  i = 0;
  for (size_t b = 0; b < P->X.size(); ++b)
    for (int s : P->X[b]) {
      X[3 * i] = (int32_t)b; X[3 * i + 1] = s;
      X[3 * i + 2] = P->boxes[b].leaf && npts((int)b) <= P->wx_direct_max; ++i;
    }
}


// Full matvec, O7-O10 (P:466-522 restated for points, with the compressed
// operators of P:205-235 / P:315-355).  q and pot are in caller order.
// Optional phase outputs (may be NULL): qhat [nboxes x k] (level-normalised
// q^'), lhat [nboxes x k], pot_near / pot_far [N] in SORTED order.
// nrm (may be NULL): N x 3 source normals in caller order -> double-layer sources: the kernel
// of every evaluation whose source is an input point (S2M check potential, X check potential,
// near field) is dG/dn(y) ("only the integral kernel function in S2T translation
// and the first step in S2M translation should be replaced"); surfaces stay single layer.
// tri (may be NULL): N x 9 triangle vertices in caller order -> BEM elements:
// the points are the elements' centroids (collocation points) and every evaluation whose
// source is an element integrates G over it (reading R-BEM): S2T, the S2M check
// potential and the X check potential.
void oracle_matvec(void* h, const oracle_tables* tb, const double* q, const double* nrm, const double* tri, double* pot,
                   double* qhat_out, double* lhat_out, double* near_out, double* far_out) {
  Plan* P = (Plan*)h;
  const int64_t N = P->N;
  const int n = tb->n, k = tb->k;
  const double d = tb->d;
  const int nb = (int)P->boxes.size();
  const std::vector<double> g = surface(tb->p);  // n x 3 unit surface
  const double f_in = 1.0 + d, f_out = 3.0 - 2.0 * d;
  std::vector<double> qs(N);
  for (int64_t i = 0; i < N; ++i) qs[i] = q[P->perm[i]];
  const double* xs = P->xs.data();
  std::vector<double> ns;  // sorted normals (double layer)
  if (nrm) {
    ns.resize(3 * N);
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < 3; ++c) ns[3 * i + c] = nrm[3 * (int64_t)P->perm[i] + c];
  }
  std::vector<Tri> ts;  // sorted triangles (BEM)
  if (tri) {
    ts.resize(N);
    for (int64_t i = 0; i < N; ++i)
      for (int e = 0; e < 3; ++e)
        for (int c = 0; c < 3; ++c) ts[i].v[e][c] = tri[9 * (int64_t)P->perm[i] + 3 * e + c];
  }
  // source kernel: single layer G, double layer dG/dn(y), or (BEM) the element integral;
  // self = the target is source j's own collocation point
  auto Gsrc_t = [&](double x0, double x1, double x2, int j, bool self) {
    if (tri) {
      const double x[3] = {x0, x1, x2};
      return self ? tri_self(ts[j], x) : tri_integral(ts[j], x, 0);
    }
    return nrm ? Gdl(x0, x1, x2, xs[3 * j], xs[3 * j + 1], xs[3 * j + 2], ns[3 * j], ns[3 * j + 1], ns[3 * j + 2])
               : G(x0, x1, x2, xs[3 * j], xs[3 * j + 1], xs[3 * j + 2]);
  };
  auto Gsrc = [&](double x0, double x1, double x2, int j) { return Gsrc_t(x0, x1, x2, j, false); };
  std::vector<double> qhat((size_t)nb * k, 0.0), lhat((size_t)nb * k, 0.0);
  std::vector<double> pnear(N, 0.0), pfar(N, 0.0);
  auto npts = [&](int a) { return P->boxes[a].pend - P->boxes[a].pbeg; };
  const int wx = P->wx_direct_max;

  // O7a  S2M (S~ = R^T S): c_i = sum_j G(c_B + r f_out g_i, x_j) q_j ; q^'_B = S' c
#pragma omp parallel for schedule(dynamic, 4)
  for (int b = 0; b < nb; ++b) {
    const Box& B = P->boxes[b];
    if (!B.leaf || B.level < 2) continue;
    std::vector<double> c(n, 0.0);
    for (int i = 0; i < n; ++i) {
      double y0 = B.c[0] + B.r * f_out * g[3 * i], y1 = B.c[1] + B.r * f_out * g[3 * i + 1], y2 = B.c[2] + B.r * f_out * g[3 * i + 2];
      double acc = 0;
      for (int j = B.pbeg; j < B.pend; ++j) acc += Gsrc(y0, y1, y2, j) * qs[j];
      c[i] = acc;
    }
    for (int a = 0; a < k; ++a) {
      double acc = 0;
      for (int i = 0; i < n; ++i) acc += tb->S[(size_t)a * n + i] * c[i];
      qhat[(size_t)b * k + a] = acc;
    }
  }
  // O7b  M2M (M~ = R^T M R), levels L..3 into parents at level >= 2:
  //      q^'_P += 1/2 M~_o q^'_child   (1/2 = r_child / r_parent, reading Q15)
  for (int l = P->nlevels() - 1; l >= 3; --l) {
    // parallel over parents; children of one parent summed in octant order
#pragma omp parallel for schedule(dynamic, 16)
    for (int pb = P->level_begin[l - 1]; pb < P->level_begin[l]; ++pb) {
      const Box& Pa = P->boxes[pb];
      if (Pa.leaf) continue;
      for (int o = 0; o < 8; ++o) {
        int c = Pa.child[o];
        if (c < 0) continue;
        for (int a = 0; a < k; ++a) {
          double acc = 0;
          for (int e = 0; e < k; ++e) acc += tb->M[((size_t)o * k + a) * k + e] * qhat[(size_t)c * k + e];
          qhat[(size_t)pb * k + a] += 0.5 * acc;
        }
      }
    }
  }
  // O8a  M2L (P:136-144 compressed per P:216-235): l^_B += C_delta q^'_A over V(B), offset order
#pragma omp parallel for schedule(dynamic, 16)
  for (int b = 0; b < nb; ++b) {
    for (auto& e : P->V[b]) {
      const double* C = tb->C + (size_t)e.second * k * k;
      for (int a = 0; a < k; ++a) {
        double acc = 0;
        for (int f = 0; f < k; ++f) acc += C[(size_t)a * k + f] * qhat[(size_t)e.first * k + f];
        lhat[(size_t)b * k + a] += acc;
      }
    }
  }
  // O8b  X (S2L, reading O5/Q18): l^_B += U^T G(c_B + r f_in g, x_A) q_A for non-direct X pairs
#pragma omp parallel for schedule(dynamic, 4)
  for (int b = 0; b < nb; ++b) {
    const Box& B = P->boxes[b];
    for (int a : P->X[b]) {
      bool direct = B.leaf && npts(b) <= wx;
      if (direct) continue;
      const Box& A = P->boxes[a];
      std::vector<double> c(n, 0.0);
      for (int i = 0; i < n; ++i) {
        double y0 = B.c[0] + B.r * f_in * g[3 * i], y1 = B.c[1] + B.r * f_in * g[3 * i + 1], y2 = B.c[2] + B.r * f_in * g[3 * i + 2];
        double acc = 0;
        for (int j = A.pbeg; j < A.pend; ++j) acc += Gsrc(y0, y1, y2, j) * qs[j];
        c[i] = acc;
      }
      for (int r = 0; r < k; ++r) {
        double acc = 0;
        for (int i = 0; i < n; ++i) acc += tb->U[(size_t)i * k + r] * c[i];
        lhat[(size_t)b * k + r] += acc;
      }
    }
  }
  // O8c  L2L (L~ = U^T L U), levels 2..L-1, preorder: l^_child += L~_o l^_B
  for (int l = 2; l < P->nlevels() - 1; ++l) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int pb = P->level_begin[l]; pb < P->level_begin[l + 1]; ++pb) {
      const Box& Pa = P->boxes[pb];
      if (Pa.leaf) continue;
      for (int o = 0; o < 8; ++o) {
        int c = Pa.child[o];
        if (c < 0) continue;
        for (int a = 0; a < k; ++a) {
          double acc = 0;
          for (int e = 0; e < k; ++e) acc += tb->L[((size_t)o * k + a) * k + e] * lhat[(size_t)pb * k + e];
          lhat[(size_t)c * k + a] += acc;
        }
      }
    }
  }
  // O9   per target leaf: L2T (T~ = T U), W (M2T), near field (S2T)
#pragma omp parallel for schedule(dynamic, 4)
  for (int b = 0; b < nb; ++b) {
    const Box& B = P->boxes[b];
    if (!B.leaf) continue;
    std::vector<double> qd(n);
    // L2T: q_d = r_l T' l^_B ; pot_i += sum_m G(x_i, c_B + r f_out g_m) q_d,m
    if (B.level >= 2) {
      for (int m = 0; m < n; ++m) {
        double acc = 0;
        for (int a = 0; a < k; ++a) acc += tb->T[(size_t)m * k + a] * lhat[(size_t)b * k + a];
        qd[m] = B.r * acc;
      }
      for (int i = B.pbeg; i < B.pend; ++i) {
        double acc = 0;
        for (int m = 0; m < n; ++m)
          acc += G(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2], B.c[0] + B.r * f_out * g[3 * m], B.c[1] + B.r * f_out * g[3 * m + 1],
                   B.c[2] + B.r * f_out * g[3 * m + 2]) * qd[m];
        pfar[i] += acc;
      }
    }
    // W (M2T): pot_i += sum_m G(x_i, c_A + r_A f_in g_m) (r_A U q^'_A)_m for non-direct W pairs
    for (int a : P->W[b]) {
      const Box& A = P->boxes[a];
      if (npts(a) <= wx) continue;
      for (int m = 0; m < n; ++m) {
        double acc = 0;
        for (int e = 0; e < k; ++e) acc += tb->U[(size_t)m * k + e] * qhat[(size_t)a * k + e];
        qd[m] = A.r * acc;
      }
      for (int i = B.pbeg; i < B.pend; ++i) {
        double acc = 0;
        for (int m = 0; m < n; ++m)
          acc += G(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2], A.c[0] + A.r * f_in * g[3 * m], A.c[1] + A.r * f_in * g[3 * m + 1],
                   A.c[2] + A.r * f_in * g[3 * m + 2]) * qd[m];
        pfar[i] += acc;
      }
    }
    // near field: U(B), then direct W pairs (A's subtree), then direct X pairs (A leaf)
    std::vector<std::pair<int, int>> ranges;
    for (int a : P->U[b]) ranges.push_back({P->boxes[a].pbeg, P->boxes[a].pend});
    for (int a : P->W[b]) if (npts(a) <= wx) ranges.push_back({P->boxes[a].pbeg, P->boxes[a].pend});
    if (npts(b) <= wx) for (int a : P->X[b]) ranges.push_back({P->boxes[a].pbeg, P->boxes[a].pend});
    for (int i = B.pbeg; i < B.pend; ++i) {
      double acc = 0;
      for (auto& rg : ranges)
        for (int j = rg.first; j < rg.second; ++j) acc += Gsrc_t(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2], j, j == i) * qs[j];
      pnear[i] = acc;
    }
  }
  // O10 output in caller order
  for (int64_t i = 0; i < N; ++i) pot[P->perm[i]] = pnear[i] + pfar[i];
  if (qhat_out) std::memcpy(qhat_out, qhat.data(), sizeof(double) * qhat.size());
  if (lhat_out) std::memcpy(lhat_out, lhat.data(), sizeof(double) * lhat.size());
  if (near_out) std::memcpy(near_out, pnear.data(), sizeof(double) * N);
  if (far_out) std::memcpy(far_out, pfar.data(), sizeof(double) * N);
}

}  // extern "C"
