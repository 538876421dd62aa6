// Restarted GMRES on the device around the FMM matvec (the
// paper solves its BEM systems with GMRES, tolerance 1e-6 at P:539, and reports
// the time per iteration T_it, Tables 2-4).
//
// GMRES(m) (Saad & Schultz): Arnoldi with classical Gram-Schmidt applied twice (CGS2) —
// h = V^T w and w -= V h as two multi-vector kernels per pass, the norm fused into the
// second — so an iteration costs one FMM matvec and four multi-vector sweeps, all queued
// without host round trips; the (m + 1) x m Hessenberg least-squares problem is reduced
// by Givens rotations on the host (one small device-to-host copy per iteration).  All
// vectors are in caller order; the matvec is the plan's.
#include <cmath>
#include <vector>

#include "fmm_internal.h"

namespace kifmm {

namespace {

constexpr int GM_NT = 256;

// out[c] = sum_i V[c][i] w[i] for c < ncols (block partial sums, atomic into out).
// Columns in groups of MD_CB: each thread reads w[i] once per group and keeps MD_CB
// partial sums in registers (one pass over the group's V columns).
constexpr int MD_CB = 8;
__global__ void __launch_bounds__(GM_NT) k_multidot(const double* __restrict__ V, int64_t ld, int ncols,
                                                    const double* __restrict__ w, int64_t N, double* __restrict__ out) {
  __shared__ double red[GM_NT / 32][MD_CB];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < ncols; c0 += MD_CB) {
    double acc[MD_CB];
#pragma unroll
    for (int c = 0; c < MD_CB; ++c) acc[c] = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)GM_NT + threadIdx.x; i < N; i += (int64_t)gridDim.x * GM_NT) {
      const double wi = w[i];
#pragma unroll
      for (int c = 0; c < MD_CB; ++c)
        if (c0 + c < ncols) acc[c] = fma(__ldcs(V + (size_t)(c0 + c) * ld + i), wi, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < MD_CB; ++c) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < MD_CB; ++c) red[wp][c] = acc[c];
    }
    __syncthreads();
    if (threadIdx.x < MD_CB && c0 + (int)threadIdx.x < ncols) {
      double sum = 0.0;
      for (int k = 0; k < GM_NT / 32; ++k) sum += red[k][threadIdx.x];
      atomicAdd(out + c0 + threadIdx.x, sum);
    }
    __syncthreads();
  }
}

// w[i] -= sum_c V[c][i] h[c] (h on the device); NORM: also *nrm2 += sum_i w[i]^2 of the
// result (block partial sums, one atomic per block).  Eight independent partial sums:
// the column loads are not serialised behind one FMA chain.
template <bool NORM>
__global__ void __launch_bounds__(GM_NT) k_multiaxpy(const double* __restrict__ V, int64_t ld, int ncols,
                                                     const double* __restrict__ h, double* __restrict__ w, int64_t N,
                                                     double* __restrict__ nrm2) {
  double ss = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)GM_NT + threadIdx.x; i < N; i += (int64_t)gridDim.x * GM_NT) {
    double a[8] = {w[i], 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int c = 0;
    for (; c + 8 <= ncols; c += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = fma(-__ldcs(V + (size_t)(c + u) * ld + i), h[c + u], a[u]);
    }
    for (; c < ncols; ++c) a[0] = fma(-__ldcs(V + (size_t)c * ld + i), h[c], a[0]);
    const double r = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    w[i] = r;
    if (NORM) ss = fma(r, r, ss);
  }
  if (NORM) {
    __shared__ double red[GM_NT / 32];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < GM_NT / 32; ++k) t += red[k];
      atomicAdd(nrm2, t);
    }
  }
}


// y = x / sqrt(*nrm2) (zeros if the norm vanishes: Arnoldi breakdown, the loop stops there)
__global__ void k_scale_by_norm(const double* __restrict__ x, const double* __restrict__ nrm2, double* __restrict__ y,
                                int64_t N) {
  const double s = *nrm2 > 0.0 ? 1.0 / sqrt(*nrm2) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = s * x[i];
}

__global__ void k_scale_copy(const double* __restrict__ x, double a, double* __restrict__ y, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) y[i] = a * x[i];
}

// r = b - r  (r holds A x on entry)
__global__ void k_residual(const double* __restrict__ b, double* __restrict__ r, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) r[i] = b[i] - r[i];
}

// x += sum_c V[c] y[c]
__global__ void k_update(const double* __restrict__ V, int64_t ld, int ncols, const double* __restrict__ y,
                         double* __restrict__ x, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double a0 = x[i], a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = 0;
    for (; c + 4 <= ncols; c += 4) {
      a0 = fma(__ldcs(V + (size_t)c * ld + i), y[c], a0);
      a1 = fma(__ldcs(V + (size_t)(c + 1) * ld + i), y[c + 1], a1);
      a2 = fma(__ldcs(V + (size_t)(c + 2) * ld + i), y[c + 2], a2);
      a3 = fma(__ldcs(V + (size_t)(c + 3) * ld + i), y[c + 3], a3);
    }
    for (; c < ncols; ++c) a0 = fma(__ldcs(V + (size_t)c * ld + i), y[c], a0);
    x[i] = (a0 + a1) + (a2 + a3);
  }
}

}  // namespace

int gmres_solve(Plan& P, const double* b, double* x, int m, int maxit, double tol, cudaStream_t st, int* iters,
                double* relres, double* t_matvec_ms) {
  const int64_t N = P.tree.N;
  const int grid = std::max(1, std::min((int)((N + GM_NT - 1) / GM_NT), 4 * 148));
  double *V = nullptr, *h = nullptr, *w = nullptr;
  KIFMM_CUDA(cudaMalloc(&V, sizeof(double) * (size_t)(m + 1) * N));
  KIFMM_CUDA(cudaMalloc(&h, sizeof(double) * (2 * (m + 1) + 1)));  // CGS2 passes 1 / 2, ||w||^2
  KIFMM_CUDA(cudaMalloc(&w, sizeof(double) * N));
  struct Free {
    double *a, *b, *c;
    ~Free() { cudaFree(a); cudaFree(b); cudaFree(c); }
  } fr{V, h, w};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float mv_ms = 0;
  int nmv = 0;
  bool mv_pending = false;
  // matvec with its time taken from events read at the next host synchronisation (the
  // stream is never stalled for the timing)
  auto matvec = [&](const double* in, double* out) -> int {
    cudaEventRecord(e0, st);
    if (matvec_device(P, in, out, false, st)) return -3;
    cudaEventRecord(e1, st);
    mv_pending = true;
    return 0;
  };
  auto mv_account = [&]() {
    if (!mv_pending) return;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    mv_ms += ms;
    ++nmv;
    mv_pending = false;
  };
  auto dot_into = [&](const double* Vc, int ncols, const double* vec, std::vector<double>& hv) -> int {
    KIFMM_CUDA(cudaMemsetAsync(h, 0, sizeof(double) * ncols, st));
    k_multidot<<<grid, GM_NT, 0, st>>>(Vc, N, ncols, vec, N, h);
    KIFMM_CUDA(cudaGetLastError());
    hv.resize(ncols);
    KIFMM_CUDA(cudaMemcpyAsync(hv.data(), h, sizeof(double) * ncols, cudaMemcpyDeviceToHost, st));
    KIFMM_CUDA(cudaStreamSynchronize(st));
    mv_account();
    return 0;
  };
  std::vector<double> tmp;
  // ||b||
  if (dot_into(b, 1, b, tmp)) return -3;
  const double bnorm = std::sqrt(tmp[0]);
  *iters = 0;
  *relres = 0.0;
  if (bnorm == 0.0) {
    KIFMM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, st));
    KIFMM_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), hv;
  int it = 0;
  double res = 0;
  while (true) {
    // r = b - A x ; v0 = r / ||r||
    if (matvec(x, V)) return -3;
    k_residual<<<grid, GM_NT, 0, st>>>(b, V, N);
    if (dot_into(V, 1, V, tmp)) return -3;
    double beta = std::sqrt(tmp[0]);
    res = beta / bnorm;
    if (res <= tol || it >= maxit) break;
    k_scale_copy<<<grid, GM_NT, 0, st>>>(V, 1.0 / beta, V, N);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && it < maxit; ++j, ++it) {
      if (matvec(V + (size_t)j * N, w)) return -3;
      // CGS2 on the device (h = V^T w, w -= V h, twice; the second sweep also sums ||w||^2),
      // v_{j+1} = w / ||w||; one host synchronisation per iteration, for the Hessenberg
      // column.  (DGKS selective reorthogonalisation was measured: the BEM Krylov vectors
      // need the second pass in 118 of 124 steps, so it is always run.)
      double* const h1 = h;
      double* const h2 = h + (m + 1);
      double* const nrm = h + 2 * (m + 1);
      KIFMM_CUDA(cudaMemsetAsync(h, 0, sizeof(double) * (2 * (m + 1) + 1), st));
      k_multidot<<<grid, GM_NT, 0, st>>>(V, N, j + 1, w, N, h1);
      k_multiaxpy<false><<<grid, GM_NT, 0, st>>>(V, N, j + 1, h1, w, N, nullptr);
      k_multidot<<<grid, GM_NT, 0, st>>>(V, N, j + 1, w, N, h2);
      k_multiaxpy<true><<<grid, GM_NT, 0, st>>>(V, N, j + 1, h2, w, N, nrm);
      k_scale_by_norm<<<grid, GM_NT, 0, st>>>(w, nrm, V + (size_t)(j + 1) * N, N);
      KIFMM_CUDA(cudaGetLastError());
      hv.resize(2 * (m + 1) + 1);
      KIFMM_CUDA(cudaMemcpyAsync(hv.data(), h, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost, st));
      KIFMM_CUDA(cudaStreamSynchronize(st));
      mv_account();
      std::vector<double> hcol(j + 2, 0.0);
      for (int i = 0; i <= j; ++i) hcol[i] = hv[i] + hv[(m + 1) + i];
      hcol[j + 1] = std::sqrt(hv[2 * (m + 1)]);
      // apply the previous rotations, then a new one to annihilate h[j+1]
      for (int i = 0; i < j; ++i) {
        const double a = hcol[i], c = hcol[i + 1];
        hcol[i] = cs[i] * a + sn[i] * c;
        hcol[i + 1] = -sn[i] * a + cs[i] * c;
      }
      const double den = std::hypot(hcol[j], hcol[j + 1]);
      cs[j] = den > 0 ? hcol[j] / den : 1.0;
      sn[j] = den > 0 ? hcol[j + 1] / den : 0.0;
      hcol[j] = den;
      hcol[j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hcol[i];
      res = std::fabs(g[j + 1]) / bnorm;
      if (res <= tol || hcol[j] == 0.0) { ++j; ++it; break; }
    }
    // y = R^-1 g (back substitution), x += V y
    std::vector<double> y(j, 0.0);
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int c = i + 1; c < j; ++c) s -= H[(size_t)i * m + c] * y[c];
      y[i] = H[(size_t)i * m + i] != 0 ? s / H[(size_t)i * m + i] : 0.0;
    }
    if (j > 0) {
      KIFMM_CUDA(cudaMemcpyAsync(h, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, st));
      k_update<<<grid, GM_NT, 0, st>>>(V, N, j, h, x, N);
      KIFMM_CUDA(cudaGetLastError());
    }
    if (res <= tol || it >= maxit) {
      // true residual of the final iterate
      if (matvec(x, V)) return -3;
      k_residual<<<grid, GM_NT, 0, st>>>(b, V, N);
      if (dot_into(V, 1, V, tmp)) return -3;
      res = std::sqrt(tmp[0]) / bnorm;
      break;
    }
  }
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *iters = it;
  *relres = res;
  if (t_matvec_ms) *t_matvec_ms = nmv ? mv_ms / nmv : 0.0;
  return 0;
}

}  // namespace kifmm
