// Host precompute of the SVD-compressed KIFMM operator tables (runs once per
// (p, k, d); timed separately from the matvec, as the north_star asks).
//
// All operators at unit halfwidth (homogeneous kernel of degree -1);
// the level factors live in the matvec (reading Q15).
//   surfaces  P:109-113  UE, DC at (1+d); UC, DE at (3-2d); p points per edge
//   E_u, E_d  P:126-154  equivalent-density solves, pinv by one-sided Jacobi SVD (extended precision)
//   K_delta   P:136-144  K_ij = G(x_i, y_j), x = DC(target @ 0), y = UE(source @ 2 delta)
//   basis U   P:172-203  leading left singular vectors of K_fat (= those of K_thin,
//                        P:199-203): Householder QR of K_fat^T, Jacobi SVD of R
//   C_delta   P:216-223  U^T K_delta U
//   S', T'    P:341, P:351   S' = U^T pinv(E_u), T' = pinv(E_d) U (fused, reading Q17)
//   M~_o, L~_o P:337, P:347  U^T pinv(E_u) G(UC, UE_child) U,  U^T G(DC_child, DE) pinv(E_d) U
// Own dense linear algebra (no LAPACK in this image); shares no code with oracle/.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "fmm_internal.h"

namespace kifmm {

namespace {

using Mat = std::vector<double>;  // row-major

std::vector<double> unit_surface(int p) {
  std::vector<double> g;
  const double h = 2.0 / (p - 1);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        bool on = i == 0 || j == 0 || k == 0 || i == p - 1 || j == p - 1 || k == p - 1;
        if (!on) continue;
        g.push_back(-1.0 + h * i);
        g.push_back(-1.0 + h * j);
        g.push_back(-1.0 + h * k);
      }
  return g;
}

// G(x_i, y_j) = 1/(4 pi |x_i - y_j|) for x = a*g + ca, y = b*g + cb
Mat kmat(const std::vector<double>& g, int n, double a, const double ca[3], double b, const double cb[3]) {
  Mat K((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double r2 = 0;
      for (int d = 0; d < 3; ++d) {
        double t = (a * g[3 * i + d] + ca[d]) - (b * g[3 * j + d] + cb[d]);
        r2 += t * t;
      }
      K[(size_t)i * n + j] = 1.0 / (4.0 * M_PI * std::sqrt(r2));
    }
  return K;
}

// C = A (m x k) * B (k x n)
Mat matmul(const Mat& A, const Mat& B, int m, int k, int n) {
  Mat C((size_t)m * n, 0.0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < m; ++i)
    for (int l = 0; l < k; ++l) {
      double a = A[(size_t)i * k + l];
      if (a == 0.0) continue;
      const double* b = &B[(size_t)l * n];
      double* c = &C[(size_t)i * n];
      for (int j = 0; j < n; ++j) c[j] += a * b[j];
    }
  return C;
}

Mat transpose(const Mat& A, int m, int n) {
  Mat T((size_t)n * m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) T[(size_t)j * m + i] = A[(size_t)i * n + j];
  return T;
}

// One-sided (Hestenes) Jacobi on the columns of a square n x n A, in x87 extended
// precision (long double, 64-bit significand): rotations J with A J = W (orthogonal
// columns), V = J^T.  On return row c of W is column c of A J (= sigma_c u_c) and row c
// of V is the right singular vector v_c; sig[c] = |W_c| (unsorted).
//
// Why extended precision: E_u and E_d keep singular values down to 1e-10 sigma_max at
// p = 8, and the kept small singular vectors carry the rounding of every rotation that
// mixed them with the large ones (absolute ~eps sigma_max, relative eps / 1e-10).  In
// double that moved the p = 8 matvec by 1.4e-7 from the oracle's tables (SURVEY
// §8(c.5)(4) bound: 1e-7); in extended precision by ~6e-9, the floor that one-ulp
// differences in E itself set.  Pairs are visited in round-robin (tournament) order:
// each round's n/2 disjoint column pairs rotate in parallel.
using LMat = std::vector<long double>;
void jacobi_onesided_ld(const Mat& A, int n, LMat& W, LMat& V, std::vector<long double>& sig) {
  using R = long double;
  const int m = n + (n & 1);  // an odd n gets a dummy column that pairs with nothing
  W.assign((size_t)n * n, 0.0L);
  V.assign((size_t)n * n, 0.0L);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) W[(size_t)j * n + i] = A[(size_t)i * n + j];
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0L;
  std::vector<int> ring(m);
  for (int i = 0; i < m; ++i) ring[i] = i;
  const R tol = 1e-17L;  // ~100 eps of the extended format
  for (int sweep = 0; sweep < 80; ++sweep) {
    R off = 0;
    for (int round = 0; round < m - 1; ++round) {
#pragma omp parallel for schedule(static) reduction(max : off)
      for (int h = 0; h < m / 2; ++h) {
        int i = ring[h], j = ring[m - 1 - h];
        if (i >= n || j >= n) continue;
        if (i > j) std::swap(i, j);
        R* wi = &W[(size_t)i * n];
        R* wj = &W[(size_t)j * n];
        R al = 0, be = 0, ga = 0;
        for (int r = 0; r < n; ++r) { al += wi[r] * wi[r]; be += wj[r] * wj[r]; ga += wi[r] * wj[r]; }
        if (ga == 0 || al == 0 || be == 0) continue;
        const R rel = std::fabs(ga) / std::sqrt(al * be);
        off = std::max(off, rel);
        if (rel < tol) continue;
        const R zeta = (be - al) / (2 * ga);
        const R t = (zeta >= 0 ? 1 : -1) / (std::fabs(zeta) + std::sqrt(1 + zeta * zeta));
        const R c = 1 / std::sqrt(1 + t * t), s = c * t;
        for (int r = 0; r < n; ++r) {
          const R x = wi[r], y = wj[r];
          wi[r] = c * x - s * y;
          wj[r] = s * x + c * y;
        }
        R* vi = &V[(size_t)i * n];
        R* vj = &V[(size_t)j * n];
        for (int r = 0; r < n; ++r) {
          const R x = vi[r], y = vj[r];
          vi[r] = c * x - s * y;
          vj[r] = s * x + c * y;
        }
      }
      std::rotate(ring.begin() + 1, ring.end() - 1, ring.end());  // position 0 stays fixed
    }
    if (off < tol) break;
  }
  sig.assign(n, 0.0L);
  for (int c = 0; c < n; ++c) {
    R s2 = 0;
    for (int r = 0; r < n; ++r) s2 += W[(size_t)c * n + r] * W[(size_t)c * n + r];
    sig[c] = std::sqrt(s2);
  }
}

// Moore-Penrose pseudo-inverse of a square A from its Jacobi SVD; singular values
// <= rcond * sigma_max are dropped (reading Q11).
Mat pinv_jacobi(const Mat& A, int n, double rcond) {
  using R = long double;
  LMat W, V;
  std::vector<R> sig;
  jacobi_onesided_ld(A, n, W, V, sig);
  const R smax = *std::max_element(sig.begin(), sig.end());
  // pinv = sum_c v_c u_c^T / sigma_c = sum_c v_c W_c^T / sigma_c^2
  Mat P((size_t)n * n, 0.0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    std::vector<R> row(n, 0.0L);
    for (int c = 0; c < n; ++c) {
      if (!(sig[c] > (R)rcond * smax)) continue;
      const R f = V[(size_t)c * n + i] / (sig[c] * sig[c]);
      const R* w = &W[(size_t)c * n];
      for (int j = 0; j < n; ++j) row[j] += f * w[j];
    }
    for (int j = 0; j < n; ++j) P[(size_t)i * n + j] = (double)row[j];
  }
  return P;
}

// Left singular vectors and singular values of K_fat = [K_0 K_1 ... K_315] (n x 316n,
// eq. fat), descending.  Householder QR of K_fat^T = Q R (316n x n, column
// by column, trailing columns updated in parallel), then the one-sided Jacobi SVD of the
// n x n R: R = W Sigma V^T gives K_fat = V Sigma (Q W)^T, so U = V.  Backward stable in
// K_fat itself: the kept subspace is accurate to eps sigma_1 / (sigma_k - sigma_k+1)
// (1e-11 at p = 6), where an eigensolve of the Gram K_fat K_fat^T (squared condition)
// gets eps sigma_1^2 / (sigma_k^2 - sigma_k+1^2) (2e-7 at p = 6).
void kfat_svd(const std::vector<Mat>& K, int n, std::vector<double>& sigma, Mat& vec) {
  const size_t m = (size_t)K.size() * n;
  // column a of K_fat^T = row a of K_fat = (K_0[a, :], K_1[a, :], ...)
  std::vector<Mat> col(n, Mat(m));
#pragma omp parallel for schedule(static)
  for (int a = 0; a < n; ++a)
    for (size_t o = 0; o < K.size(); ++o)
      std::memcpy(&col[a][o * n], &K[o][(size_t)a * n], sizeof(double) * n);
  Mat Rm((size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double* x = col[j].data() + j;
    const size_t len = m - j;
    double nrm2 = 0;
    for (size_t r = 0; r < len; ++r) nrm2 += x[r] * x[r];
    const double alpha = x[0] >= 0 ? -std::sqrt(nrm2) : std::sqrt(nrm2);
    // v = x - alpha e_1 (stored in place), H = I - 2 v v^T / (v^T v)
    const double v0 = x[0] - alpha;
    const double vtv = nrm2 - x[0] * x[0] + v0 * v0;
    x[0] = v0;
    if (vtv > 0) {
#pragma omp parallel for schedule(static)
      for (int c = j + 1; c < n; ++c) {
        double* y = col[c].data() + j;
        double s = 0;
        for (size_t r = 0; r < len; ++r) s += x[r] * y[r];
        const double f = 2.0 * s / vtv;
        for (size_t r = 0; r < len; ++r) y[r] -= f * x[r];
      }
    }
    Rm[(size_t)j * n + j] = alpha;
    for (int c = j + 1; c < n; ++c) Rm[(size_t)j * n + c] = col[c][j];
  }
  col.clear();
  LMat W, V;
  std::vector<long double> sig;
  jacobi_onesided_ld(Rm, n, W, V, sig);
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return sig[a] > sig[b]; });
  sigma.resize(n);
  vec.assign((size_t)n * n, 0.0);
  for (int c = 0; c < n; ++c) {
    sigma[c] = (double)sig[idx[c]];
    for (int r = 0; r < n; ++r) vec[(size_t)r * n + c] = (double)V[(size_t)idx[c] * n + r];
  }
}

// SVD of a square n x n A by one-sided (Hestenes) Jacobi: A = sum_c s_c u_c v_c^T,
// s descending; u (n x n, column c = u_c, row-major), v (n x n, row c = v_c).
void svd_jacobi(const Mat& A, int n, std::vector<double>& s, Mat& u, Mat& v) {
  Mat W = transpose(A, n, n);  // row c of W = column c of A
  Mat V((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0;
    for (int i = 0; i < n - 1; ++i)
      for (int j = i + 1; j < n; ++j) {
        double* wi = &W[(size_t)i * n];
        double* wj = &W[(size_t)j * n];
        double al = 0, be = 0, ga = 0;
        for (int r = 0; r < n; ++r) { al += wi[r] * wi[r]; be += wj[r] * wj[r]; ga += wi[r] * wj[r]; }
        if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
        const double rel = std::fabs(ga) / std::sqrt(al * be);
        off = std::max(off, rel);
        if (rel < 1e-15) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < n; ++r) {
          const double x = wi[r], y = wj[r];
          wi[r] = c * x - sn * y;
          wj[r] = sn * x + c * y;
        }
        double* vi = &V[(size_t)i * n];
        double* vj = &V[(size_t)j * n];
        for (int r = 0; r < n; ++r) {
          const double x = vi[r], y = vj[r];
          vi[r] = c * x - sn * y;
          vj[r] = sn * x + c * y;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> sig(n);
  for (int c = 0; c < n; ++c) {
    double s2 = 0;
    for (int r = 0; r < n; ++r) s2 += W[(size_t)c * n + r] * W[(size_t)c * n + r];
    sig[c] = std::sqrt(s2);
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return sig[a] > sig[b]; });
  s.resize(n);
  u.assign((size_t)n * n, 0.0);
  v.assign((size_t)n * n, 0.0);
  for (int c = 0; c < n; ++c) {
    const int k = idx[c];
    s[c] = sig[k];
    for (int r = 0; r < n; ++r) {
      u[(size_t)r * n + c] = sig[k] > 0 ? W[(size_t)k * n + r] / sig[k] : 0.0;
      v[(size_t)c * n + r] = V[(size_t)k * n + r];
    }
  }
}

}  // namespace

int build_tables(int p, int k, double d, double rcond, HostTables* out) {
  const std::vector<double> g = unit_surface(p);
  const int n = (int)g.size() / 3;
  const double fin = 1.0 + d, fout = 3.0 - 2.0 * d;
  const double zero[3] = {0, 0, 0};
  // equivalent-density solves
  Mat Eu = kmat(g, n, fout, zero, fin, zero);   // G(UC, UE)
  Mat Ed = kmat(g, n, fin, zero, fout, zero);   // G(DC, DE)
  Mat Eui = pinv_jacobi(Eu, n, rcond);
  Mat Edi = pinv_jacobi(Ed, n, rcond);
  // the 316 M2L matrices and the Gram matrix of K_fat
  std::vector<Mat> K(kNumOffsets);
  int id = 0;
  for (int i = -3; i <= 3; ++i)
    for (int j = -3; j <= 3; ++j)
      for (int l = -3; l <= 3; ++l) {
        if (std::max(std::abs(i), std::max(std::abs(j), std::abs(l))) <= 1) continue;
        const double cb[3] = {2.0 * i, 2.0 * j, 2.0 * l};
        K[id++] = kmat(g, n, fin, zero, fin, cb);
      }
  std::vector<double> sigma;
  Mat vec;
  kfat_svd(K, n, sigma, vec);
  // k_eff: smallest k' >= k with sigma_k' - sigma_k'+1 > 1e-8 sigma_1 (reading Q12)
  int kk = std::min(k, n);
  while (kk < n && !(sigma[kk - 1] - sigma[kk] > 1e-8 * sigma[0])) ++kk;
  Mat U((size_t)n * kk);
  for (int c = 0; c < kk; ++c) {
    int arg = 0;
    for (int r = 0; r < n; ++r)
      if (std::fabs(vec[(size_t)r * n + c]) > std::fabs(vec[(size_t)arg * n + c])) arg = r;
    double sgn = vec[(size_t)arg * n + c] < 0 ? -1.0 : 1.0;
    for (int r = 0; r < n; ++r) U[(size_t)r * kk + c] = sgn * vec[(size_t)r * n + c];
  }
  Mat Ut = transpose(U, n, kk);
  out->p = p; out->n = n; out->k = kk; out->d = d; out->rcond = rcond;
  out->sigma = sigma;
  out->U = U;
  out->C.assign((size_t)kNumOffsets * kk * kk, 0.0);
  for (int o = 0; o < kNumOffsets; ++o) {
    Mat KU = matmul(K[o], U, n, n, kk);
    Mat c = matmul(Ut, KU, kk, n, kk);
    std::memcpy(&out->C[(size_t)o * kk * kk], c.data(), sizeof(double) * kk * kk);
  }
  out->S = matmul(Ut, Eui, kk, n, n);
  out->T = matmul(Edi, U, n, n, kk);
  out->M.assign((size_t)8 * kk * kk, 0.0);
  out->L.assign((size_t)8 * kk * kk, 0.0);
  for (int o = 0; o < 8; ++o) {
    const double cc[3] = {(o >> 2) & 1 ? 0.5 : -0.5, (o >> 1) & 1 ? 0.5 : -0.5, o & 1 ? 0.5 : -0.5};
    Mat Gu = kmat(g, n, fout, zero, 0.5 * fin, cc);   // G(UC_parent, UE_child)
    Mat m1 = matmul(out->S, Gu, kk, n, n);            // U^T pinv(E_u) G
    Mat Mo = matmul(m1, U, kk, n, kk);
    std::memcpy(&out->M[(size_t)o * kk * kk], Mo.data(), sizeof(double) * kk * kk);
    Mat Gd = kmat(g, n, 0.5 * fin, cc, fout, zero);   // G(DC_child, DE_parent)
    Mat l1 = matmul(Ut, Gd, kk, n, n);
    Mat Lo = matmul(l1, out->T, kk, n, kk);            // U^T G pinv(E_d) U
    std::memcpy(&out->L[(size_t)o * kk * kk], Lo.data(), sizeof(double) * kk * kk);
  }
  out->surf = g;
  return 0;
}

// Stage 2 of the M2L compression: eps2 = C2 eps1 / p~ (eq-vareps2) with
// eps1 = sigma_{k+1} / sigma_1 (the stage-1 truncation applied) and p~ = k; each core
// C_o = U_o S_o Q_o^T (SVD) keeps the singular values >= eps2 ||K_fat||_2 = eps2 sigma_1
// (eq-lra): U^_o = the kept columns of U_o (k x r_o), V^_o = S^_o Q^_o^T (r_o x k).
int build_stage2(HostTables& H, double C2) {
  H.ranks.clear(); H.Uh.clear(); H.Vh.clear(); H.eps2 = 0; H.rmax = 0;
  if (!(C2 > 0)) return 0;
  const int k = H.k;
  if (H.sigma.size() < (size_t)k + 1 || !(H.sigma[0] > 0)) {
    set_error("stage 2 needs the singular values of K_fat (tables.sigma)");
    return -2;
  }
  H.eps2 = C2 * (H.sigma[k] / H.sigma[0]) / k;
  const double cut = H.eps2 * H.sigma[0];
  std::vector<Mat> Us(kNumOffsets), Vs(kNumOffsets);
  std::vector<std::vector<double>> Ss(kNumOffsets);
#pragma omp parallel for schedule(dynamic, 1)
  for (int o = 0; o < kNumOffsets; ++o) {
    Mat A(H.C.begin() + (size_t)o * k * k, H.C.begin() + (size_t)(o + 1) * k * k);
    svd_jacobi(A, k, Ss[o], Us[o], Vs[o]);
  }
  H.ranks.assign(kNumOffsets, 0);
  for (int o = 0; o < kNumOffsets; ++o) {
    int r = 0;
    while (r < k && Ss[o][r] >= cut) ++r;
    H.ranks[o] = r;
    H.rmax = std::max(H.rmax, r);
  }
  // factors, unpadded: Uh[o] k x r_o (row-major), Vh[o] r_o x k
  H.Uh.resize(kNumOffsets);
  H.Vh.resize(kNumOffsets);
  for (int o = 0; o < kNumOffsets; ++o) {
    const int r = H.ranks[o];
    H.Uh[o].assign((size_t)k * r, 0.0);
    H.Vh[o].assign((size_t)r * k, 0.0);
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < r; ++c) H.Uh[o][(size_t)a * r + c] = Us[o][(size_t)a * k + c];
    for (int c = 0; c < r; ++c)
      for (int b = 0; b < k; ++b) H.Vh[o][(size_t)c * k + b] = Ss[o][c] * Vs[o][(size_t)c * k + b];
    // the truncated core U^_o V^_o replaces C_o (every M2L path applies the same operator)
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double acc = 0;
        for (int c = 0; c < r; ++c) acc += H.Uh[o][(size_t)a * r + c] * H.Vh[o][(size_t)c * k + b];
        H.C[((size_t)o * k + a) * k + b] = acc;
      }
  }
  return 0;
}

}  // namespace kifmm
