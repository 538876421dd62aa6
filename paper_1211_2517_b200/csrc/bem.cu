// BEM collocation operator on the device.
//   * triangles sorted like their centroids (the collocation points / tree points);
//   * enclosure check of the BEM surface condition: every element of a leaf
//     lies inside the leaf's upward equivalent surface, halfwidth (1 + d) r;
//   * near field (S2T): the block-sparse matrix A_ij = int_Tj G(x_i, y) dy over
//     every near segment of every owned target leaf is built once at setup and streamed
//     from HBM by each matvec (k_bem_near);
//   * S2M uses element-integrated leaf operators (kernels.cu, k_leafop_build)
//     and the X-list check potentials element integrals (k_chk).
#include <algorithm>
#include <vector>

#include "bem.cuh"
#include "fmm_internal.h"

namespace kifmm {

namespace {

__global__ void k_sort_tris(const double* __restrict__ tri, const int32_t* __restrict__ perm, int64_t N,
                            double4* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    const double* t = tri + 9 * (int64_t)perm[i];
    out[3 * i] = make_double4(t[0], t[1], t[2], 0.0);
    out[3 * i + 1] = make_double4(t[3], t[4], t[5], 0.0);
    out[3 * i + 2] = make_double4(t[6], t[7], t[8], 0.0);
  }
}

// per leaf: max over its elements' vertices of |v - c_B|_inf / r_B
__global__ void k_enclosure(const int* __restrict__ leaves, int nleaves, const double4* __restrict__ geom,
                            const int* __restrict__ pbeg, const int* __restrict__ pend,
                            const double4* __restrict__ tri, double* __restrict__ ratio) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int b = leaves[w];
  const double4 g = geom[b];
  double m = 0;
  for (int j = pbeg[b] + lane; j < pend[b]; j += 32)
    for (int e = 0; e < 3; ++e) {
      const double4 v = tri[3 * (int64_t)j + e];
      m = fmax(m, fmax(fabs(v.x - g.x), fmax(fabs(v.y - g.y), fabs(v.z - g.z))));
    }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) ratio[w] = m / g.w;
}

// one CTA per near block (target leaf t, source range [a, a + len)): column-major entries
// A[off + j * mp + i] = int_{T_{a+j}} G(x_{tb+i}, y) dy, analytic when tb + i == a + j;
// columns padded to mp = 4 ceil(m / 4) rows (zeros) so that the SpMV reads 32-byte quads
__global__ void __launch_bounds__(128) k_bem_near_build(const int4* __restrict__ blocks, const int64_t* __restrict__ off,
                                                        int nblocks, const double4* __restrict__ pts,
                                                        const double4* __restrict__ tri, double* __restrict__ A) {
  const int bi = blockIdx.x;
  if (bi >= nblocks) return;
  const int4 bk = blocks[bi];  // (tb, m, a, len)
  const int mp = (bk.y + 3) & ~3;
  const int64_t o = off[bi];
  const int64_t cnt = (int64_t)mp * bk.w;
  for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
    const int j = (int)(e / mp), i = (int)(e - (int64_t)j * mp);
    double v = 0.0;
    if (i < bk.y) {
      const double4 p = pts[bk.x + i];
      const double x[3] = {p.x, p.y, p.z};
      v = bem_integral(load_tri(tri + 3 * (int64_t)(bk.z + j)), x, bk.x + i == bk.z + j);
    }
    A[o + e] = v;
  }
}

// near field: pot[tb + i] = sum over the leaf's blocks of A[:, i] . q[a : a + len]; one CTA
// per target leaf; thread (c4, gi) owns targets 4 c4 .. 4 c4 + 3 and the source slice j = gi
// (mod G): each load is one 32-byte quad of a column (2 x 16-byte streaming loads), two
// sources in flight per thread; slices summed in shared memory (HBM-bound: every matrix
// entry is read once per matvec)
constexpr int BN_NT = 128;
__global__ void __launch_bounds__(BN_NT) k_bem_near(const int4* __restrict__ items, const int* __restrict__ pbeg,
                                                    const int* __restrict__ pend, const int* __restrict__ seg_off,
                                                    const int4* __restrict__ segs, const int64_t* __restrict__ moff,
                                                    const double4* __restrict__ pts, const double* __restrict__ A,
                                                    double* __restrict__ pot) {
  __shared__ double red[4 * BN_NT];
  const int item = blockIdx.x;
  const int b = items[item].x;
  const int tb = pbeg[b], m = pend[b] - tb, mp = (m + 3) & ~3;
  const int s0 = seg_off[item], s1 = seg_off[item + 1];
  for (int t0 = 0; t0 < mp; t0 += 4 * BN_NT) {
    const int nq = min(BN_NT, (mp - t0) >> 2);  // target quads in this pass
    const int G = BN_NT / nq;
    const int c4 = threadIdx.x % nq, gi = threadIdx.x / nq;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (gi < G) {
      for (int s = s0; s < s1; ++s) {
        const int4 sg = segs[s];
        const double* col = A + moff[s] + t0 + 4 * c4;
        int j = gi;
        for (; j + G < sg.w; j += 2 * G) {
          const double qa = pts[sg.y + j].w, qb = pts[sg.y + j + G].w;
          const double2* pa = reinterpret_cast<const double2*>(col + (int64_t)j * mp);
          const double2* pb = reinterpret_cast<const double2*>(col + (int64_t)(j + G) * mp);
          const double2 a0 = __ldcs(pa), a1 = __ldcs(pa + 1), b0 = __ldcs(pb), b1 = __ldcs(pb + 1);
          acc[0] = fma(b0.x, qb, fma(a0.x, qa, acc[0]));
          acc[1] = fma(b0.y, qb, fma(a0.y, qa, acc[1]));
          acc[2] = fma(b1.x, qb, fma(a1.x, qa, acc[2]));
          acc[3] = fma(b1.y, qb, fma(a1.y, qa, acc[3]));
        }
        if (j < sg.w) {
          const double qa = pts[sg.y + j].w;
          const double2* pa = reinterpret_cast<const double2*>(col + (int64_t)j * mp);
          const double2 a0 = __ldcs(pa), a1 = __ldcs(pa + 1);
          acc[0] = fma(a0.x, qa, acc[0]);
          acc[1] = fma(a0.y, qa, acc[1]);
          acc[2] = fma(a1.x, qa, acc[2]);
          acc[3] = fma(a1.y, qa, acc[3]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) red[e * BN_NT + threadIdx.x] = gi < G ? acc[e] : 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * nq; i += BN_NT) {  // target t0 + i = quad i / 4, entry i % 4
      const int q4 = i >> 2, e = i & 3;
      double sum = 0.0;
      for (int g = 0; g < G; ++g) sum += red[e * BN_NT + g * nq + q4];
      if (t0 + i < m) pot[tb + t0 + i] = sum;
    }
  }
}

}  // namespace

int bem_sort_triangles(Plan& P, const double* d_tri_caller, cudaStream_t st) {
  const int64_t N = P.tree.N;
  KIFMM_CUDA(cudaMalloc(&P.d_tri, sizeof(double4) * 3 * N));
  P.allocations.push_back(P.d_tri);
  k_sort_tris<<<(int)((N + 255) / 256), 256, 0, st>>>(d_tri_caller, P.tree.d_perm, N, P.d_tri);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

int bem_check_enclosure(Plan& P, cudaStream_t st) {
  const Tree& T = P.tree;
  std::vector<int> leaves;
  for (int b = 0; b < T.nboxes; ++b)
    if (T.leaf[b] && T.level[b] >= 2) leaves.push_back(b);
  if (leaves.empty()) return 0;
  int* d_leaves = nullptr;
  double* d_ratio = nullptr;
  KIFMM_CUDA(cudaMalloc(&d_leaves, sizeof(int) * leaves.size()));
  KIFMM_CUDA(cudaMalloc(&d_ratio, sizeof(double) * leaves.size()));
  KIFMM_CUDA(cudaMemcpyAsync(d_leaves, leaves.data(), sizeof(int) * leaves.size(), cudaMemcpyHostToDevice, st));
  const int nl = (int)leaves.size();
  k_enclosure<<<(nl * 32 + 255) / 256, 256, 0, st>>>(d_leaves, nl, T.d_geom, T.d_pbeg, T.d_pend, P.d_tri, d_ratio);
  std::vector<double> ratio(nl);
  KIFMM_CUDA(cudaMemcpyAsync(ratio.data(), d_ratio, sizeof(double) * nl, cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_leaves);
  cudaFree(d_ratio);
  // P:389-411 asks the upward equivalent surface ((1 + d) r) to enclose the leaf's elements;
  // d = C_d / sqrt(s) assumes leaves of size ~ sqrt(s) h, which an adaptive tree
  // does not guarantee (small leaves under large elements).  The overhang is reported
  // (fmm_info.bem_extrusion); setup refuses only elements reaching the upward CHECK surface
  // ((3 - 2d) r), where the S2M check evaluations would be near-singular.
  const double worst = *std::max_element(ratio.begin(), ratio.end());
  P.bem_extrusion = worst - 1.0;
  if (!(worst < 3.0 - 2.0 * P.d)) {
    set_error("fmm_setup: BEM surface condition violated (P:389-411): an element reaches its leaf's upward check "
              "surface (vertex at " + std::to_string(worst) + " r, check surface at " + std::to_string(3.0 - 2.0 * P.d) +
              " r); refine the mesh or raise the leaf size");
    return -1;
  }
  return 0;
}

// blocks: (target box first point, m, source first point, len) per near segment, aligned
// with the near segment CSR; offsets into the matrix (int64)
int bem_build_near(Plan& P, const std::vector<int4>& blocks, cudaStream_t st) {
  std::vector<int64_t> off(blocks.size() + 1, 0);  // columns of mp = 4 ceil(m / 4) rows: 32-byte aligned
  for (size_t i = 0; i < blocks.size(); ++i) off[i + 1] = off[i] + (int64_t)((blocks[i].y + 3) & ~3) * blocks[i].w;
  const int64_t entries = off.back();
  size_t fr = 0, tot = 0;
  KIFMM_CUDA(cudaMemGetInfo(&fr, &tot));
  const double bytes = (double)entries * sizeof(double);
  if (bytes > (double)fr - 4.0 * (1 << 30)) {
    set_error("fmm_setup: the BEM near-field matrix (" + std::to_string(bytes / 1e9) + " GB) does not fit");
    return -4;
  }
  KIFMM_CUDA(cudaMalloc(&P.d_bem_A, sizeof(double) * std::max<int64_t>(entries, 1)));
  P.allocations.push_back(P.d_bem_A);
  KIFMM_CUDA(cudaMalloc(&P.d_bem_moff, sizeof(int64_t) * off.size()));
  P.allocations.push_back(P.d_bem_moff);
  KIFMM_CUDA(cudaMemcpyAsync(P.d_bem_moff, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, st));
  int4* d_blocks = nullptr;
  KIFMM_CUDA(cudaMalloc(&d_blocks, sizeof(int4) * std::max<size_t>(blocks.size(), 1)));
  if (!blocks.empty()) {
    KIFMM_CUDA(cudaMemcpyAsync(d_blocks, blocks.data(), sizeof(int4) * blocks.size(), cudaMemcpyHostToDevice, st));
    k_bem_near_build<<<(int)blocks.size(), 128, 0, st>>>(d_blocks, P.d_bem_moff, (int)blocks.size(), P.tree.d_pts,
                                                         P.d_tri, P.d_bem_A);
    KIFMM_CUDA(cudaGetLastError());
  }
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_blocks);
  P.bem_near_bytes = (int64_t)bytes;
  return 0;
}

int bem_near_matvec(const Plan& P, cudaStream_t st) {
  if (P.n_tleaf == 0) return 0;
  k_bem_near<<<P.n_tleaf, BN_NT, 0, st>>>(P.d_tleaf_items, P.tree.d_pbeg, P.tree.d_pend, P.d_near_off,
                                                  P.d_near_seg, P.d_bem_moff, P.tree.d_pts, P.d_bem_A, P.d_pot_near);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace kifmm
