// Device octree build: quantise + Morton keys, CUB radix
// sort, level-by-level box construction.  Readings O1-O3:
//   root cube: c0 = (min+max)/2, r0 = max extent/2 * (1+1e-6)  ("root level cube")
//   u_d = floor((x_d - (c0_d - r0)) * 2^21/(2 r0)), clamped; key = interleave(x high)
//   a box is subdivided iff count > s and level < 21; only non-empty children.
// Box order: level-major, Morton key within a level.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "fmm_internal.h"

namespace kifmm {

namespace {

__global__ void k_bbox(const double* __restrict__ pts, int64_t N, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < 3; ++d) {
      double v = pts[3 * i + d];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
  __shared__ double s[6][256];
  for (int d = 0; d < 3; ++d) { s[d][threadIdx.x] = lo[d]; s[3 + d][threadIdx.x] = hi[d]; }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
        s[3 + d][threadIdx.x] = fmax(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int d = 0; d < 6; ++d) part[6 * blockIdx.x + d] = s[d][0];
}

__device__ __forceinline__ uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__global__ void k_quantize(const double* __restrict__ pts, int64_t N, double lx, double ly, double lz, double scale,
                           uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double lo[3] = {lx, ly, lz};
  uint32_t u[3];
  for (int d = 0; d < 3; ++d) {
    // no FMA contraction: keys must be bit-identical to the oracle's (reading Q27)
    double t = floor(__dmul_rn(__dsub_rn(pts[3 * i + d], lo[d]), scale));
    t = fmin(fmax(t, 0.0), (double)((1u << kMaxLevel) - 1));
    u[d] = (uint32_t)t;
  }
  key[i] = (spread3(u[0]) << 2) | (spread3(u[1]) << 1) | spread3(u[2]);
  idx[i] = (int32_t)i;
}

// caller -> sorted index (the output permutation gathers with it: coalesced stores)
__global__ void k_invert_perm(const int32_t* __restrict__ perm, int64_t N, int32_t* __restrict__ iperm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) iperm[perm[i]] = (int32_t)i;
}

__global__ void k_gather_points(const double* __restrict__ pts, const int32_t* __restrict__ perm, int64_t N,
                                double4* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int64_t j = perm[i];
  out[i] = make_double4(pts[3 * j], pts[3 * j + 1], pts[3 * j + 2], 0.0);
}

// head[i] = 1 iff point i is active and starts a new level-l cell
__global__ void k_heads(const uint64_t* __restrict__ key, const uint8_t* __restrict__ active, int64_t N, int shift,
                        uint8_t* __restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  uint8_t h = 0;
  if (active[i]) h = (i == 0) || ((key[i] >> shift) != (key[i - 1] >> shift));
  head[i] = h;
}

// parent (local index in the previous level) of each new box by binary search
__global__ void k_parent(const int* __restrict__ beg, int nb, const int* __restrict__ pbeg_prev, int nprev,
                         int* __restrict__ par) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  int b = beg[j];
  int lo = 0, hi = nprev;  // last index with pbeg_prev <= b
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pbeg_prev[mid] <= b) lo = mid; else hi = mid;
  }
  par[j] = lo;
}

__global__ void k_box_fill(const int* __restrict__ beg, const int* __restrict__ par, int nb,
                           const int* __restrict__ pend_prev, const uint64_t* __restrict__ skey, int level, int s,
                           int* __restrict__ end, uint64_t* __restrict__ bkey, uint8_t* __restrict__ leaf) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  int e = pend_prev[par[j]];
  if (j + 1 < nb && par[j + 1] == par[j]) e = beg[j + 1];
  end[j] = e;
  bkey[j] = skey[beg[j]] >> (3 * (kMaxLevel - level));
  leaf[j] = !((e - beg[j]) > s && level < kMaxLevel);
}

__global__ void k_deactivate(const int* __restrict__ beg, const int* __restrict__ end, const uint8_t* __restrict__ leaf,
                             int nb, uint8_t* __restrict__ active) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb || !leaf[j]) return;
  for (int i = beg[j]; i < end[j]; ++i) active[i] = 0;
}

__device__ __forceinline__ uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return (uint32_t)x;
}

__global__ void k_geom(const uint64_t* __restrict__ key, const int* __restrict__ level, int nb, double lx, double ly,
                       double lz, double r0, double4* __restrict__ geom) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  uint64_t k = key[b];
  double r = ldexp(r0, -level[b]);
  // centre = lo_root + (2a+1) r_l (reading O3), no contraction
  double cx = __dadd_rn(lx, __dmul_rn((double)(2 * (int64_t)compact3(k >> 2) + 1), r));
  double cy = __dadd_rn(ly, __dmul_rn((double)(2 * (int64_t)compact3(k >> 1) + 1), r));
  double cz = __dadd_rn(lz, __dmul_rn((double)(2 * (int64_t)compact3(k) + 1), r));
  geom[b] = make_double4(cx, cy, cz, r);
}

__global__ void k_children(const int* __restrict__ parent, const int* __restrict__ level_of, int nb,
                           int* __restrict__ child_begin, int* __restrict__ nchild) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int p = parent[b];
  if (p < 0) return;
  if (b == 0 || parent[b - 1] != p) child_begin[p] = b;
  atomicAdd(&nchild[p], 1);
}

template <typename T>
int dalloc(T** p, size_t n) {
  KIFMM_CUDA(cudaMalloc((void**)p, sizeof(T) * std::max<size_t>(n, 1)));
  return 0;
}

inline int nblk(int64_t n, int t = 256) { return std::max(1, (int)((n + t - 1) / t)); }

}  // namespace

int build_tree_device(Plan& P, const double* d_points, cudaStream_t st) {
  Tree& T = P.tree;
  const int64_t N = T.N;
  // O1: bounding box -> root cube (host arithmetic, same expression order as the reading)
  int nbb = std::min<int64_t>(1024, std::max<int64_t>(1, (N + 255) / 256));
  double* d_part;
  if (dalloc(&d_part, 6 * nbb)) return -3;
  k_bbox<<<nbb, 256, 0, st>>>(d_points, N, d_part);
  std::vector<double> part(6 * nbb);
  KIFMM_CUDA(cudaMemcpyAsync(part.data(), d_part, sizeof(double) * 6 * nbb, cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_part);
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) { lo[d] = part[d]; hi[d] = part[3 + d]; }
  for (int b = 1; b < nbb; ++b)
    for (int d = 0; d < 3; ++d) { lo[d] = std::min(lo[d], part[6 * b + d]); hi[d] = std::max(hi[d], part[6 * b + 3 + d]); }
  double ext = 0;
  for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
  double r0 = ext / 2.0 * (1.0 + 1e-6);
  if (r0 == 0.0) r0 = 1.0;
  T.r0 = r0;
  T.scale = (double)(1u << kMaxLevel) / (2.0 * r0);
  for (int d = 0; d < 3; ++d) T.lo_root[d] = (lo[d] + hi[d]) / 2.0 - r0;
  // K1 quantise + K2 stable radix sort (ties keep input order)
  uint64_t *d_key_in, *d_skey;
  int32_t* d_idx;
  if (dalloc(&d_key_in, N) || dalloc(&d_skey, N) || dalloc(&d_idx, N) || dalloc(&T.d_perm, N)) return -3;
  k_quantize<<<nblk(N), 256, 0, st>>>(d_points, N, T.lo_root[0], T.lo_root[1], T.lo_root[2], T.scale, d_key_in, d_idx);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_key_in, d_skey, d_idx, T.d_perm, (int)N, 0, 63, st);
  void* d_tmp;
  KIFMM_CUDA(cudaMalloc(&d_tmp, tmp_bytes));
  cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_key_in, d_skey, d_idx, T.d_perm, (int)N, 0, 63, st);
  KIFMM_CUDA(cudaGetLastError());
  cudaFree(d_tmp);
  cudaFree(d_key_in);
  cudaFree(d_idx);
  if (dalloc(&T.d_pts, N) || dalloc(&T.d_iperm, N)) return -3;
  k_gather_points<<<nblk(N), 256, 0, st>>>(d_points, T.d_perm, N, T.d_pts);
  k_invert_perm<<<nblk(N), 256, 0, st>>>(T.d_perm, N, T.d_iperm);
  // K3 levels
  uint8_t *d_active, *d_head;
  int *d_nsel, *d_sel;
  if (dalloc(&d_active, N) || dalloc(&d_head, N) || dalloc(&d_nsel, 1) || dalloc(&d_sel, N)) return -3;
  KIFMM_CUDA(cudaMemsetAsync(d_active, 1, N, st));
  struct Lev { int nb; int *beg, *end, *par; uint64_t* key; uint8_t* leaf; };
  std::vector<Lev> levs;
  {
    Lev L0{1, nullptr, nullptr, nullptr, nullptr, nullptr};
    if (dalloc(&L0.beg, 1) || dalloc(&L0.end, 1) || dalloc(&L0.par, 1) || dalloc(&L0.key, 1) || dalloc(&L0.leaf, 1)) return -3;
    int zero = 0, nn = (int)N, m1 = -1;
    uint64_t kz = 0;
    uint8_t lf = !((int64_t)N > P.leaf_size);
    KIFMM_CUDA(cudaMemcpyAsync(L0.beg, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    KIFMM_CUDA(cudaMemcpyAsync(L0.end, &nn, sizeof(int), cudaMemcpyHostToDevice, st));
    KIFMM_CUDA(cudaMemcpyAsync(L0.par, &m1, sizeof(int), cudaMemcpyHostToDevice, st));
    KIFMM_CUDA(cudaMemcpyAsync(L0.key, &kz, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    KIFMM_CUDA(cudaMemcpyAsync(L0.leaf, &lf, 1, cudaMemcpyHostToDevice, st));
    KIFMM_CUDA(cudaStreamSynchronize(st));
    levs.push_back(L0);
    if (lf) goto done;
  }
  {
    cub::CountingInputIterator<int> cnt(0);
    size_t sel_bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, sel_bytes, cnt, d_head, (int*)nullptr, d_nsel, (int)N, st);
    void* d_sel_tmp;
    KIFMM_CUDA(cudaMalloc(&d_sel_tmp, sel_bytes));
    for (int l = 0; l < kMaxLevel; ++l) {
      Lev& prev = levs.back();
      k_deactivate<<<nblk(prev.nb), 256, 0, st>>>(prev.beg, prev.end, prev.leaf, prev.nb, d_active);
      k_heads<<<nblk(N), 256, 0, st>>>(d_skey, d_active, N, 3 * (kMaxLevel - (l + 1)), d_head);
      cub::DeviceSelect::Flagged(d_sel_tmp, sel_bytes, cnt, d_head, d_sel, d_nsel, (int)N, st);
      int nb = 0;
      KIFMM_CUDA(cudaMemcpyAsync(&nb, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
      KIFMM_CUDA(cudaStreamSynchronize(st));
      if (nb == 0) break;
      Lev L{nb, nullptr, nullptr, nullptr, nullptr, nullptr};
      if (dalloc(&L.beg, nb) || dalloc(&L.end, nb) || dalloc(&L.par, nb) || dalloc(&L.key, nb) || dalloc(&L.leaf, nb)) return -3;
      KIFMM_CUDA(cudaMemcpyAsync(L.beg, d_sel, sizeof(int) * nb, cudaMemcpyDeviceToDevice, st));
      k_parent<<<nblk(nb), 256, 0, st>>>(L.beg, nb, prev.beg, prev.nb, L.par);
      k_box_fill<<<nblk(nb), 256, 0, st>>>(L.beg, L.par, nb, prev.end, d_skey, l + 1, P.leaf_size, L.end, L.key, L.leaf);
      KIFMM_CUDA(cudaGetLastError());
      levs.push_back(L);
      // stop when every box of this level is a leaf
      int nleaf_l = 0;
      {
        std::vector<uint8_t> lf(nb);
        KIFMM_CUDA(cudaMemcpyAsync(lf.data(), L.leaf, nb, cudaMemcpyDeviceToHost, st));
        KIFMM_CUDA(cudaStreamSynchronize(st));
        for (uint8_t v : lf) nleaf_l += v;
      }
      if (nleaf_l == nb) break;
    }
    cudaFree(d_sel_tmp);
  }
done:
  // concatenate levels (level-major)
  T.nlevels = (int)levs.size();
  T.level_begin.assign(T.nlevels + 1, 0);
  for (int l = 0; l < T.nlevels; ++l) T.level_begin[l + 1] = T.level_begin[l] + levs[l].nb;
  const int nb = T.level_begin.back();
  T.nboxes = nb;
  if (dalloc(&T.d_key, nb) || dalloc(&T.d_level, nb) || dalloc(&T.d_parent, nb) || dalloc(&T.d_pbeg, nb) ||
      dalloc(&T.d_pend, nb) || dalloc(&T.d_child_begin, nb) || dalloc(&T.d_nchild, nb) || dalloc(&T.d_leaf, nb) ||
      dalloc(&T.d_geom, nb))
    return -3;
  T.key.resize(nb); T.level.resize(nb); T.parent.resize(nb); T.pbeg.resize(nb); T.pend.resize(nb); T.leaf.resize(nb);
  for (int l = 0; l < T.nlevels; ++l) {
    const Lev& L = levs[l];
    int o = T.level_begin[l];
    KIFMM_CUDA(cudaMemcpyAsync(T.key.data() + o, L.key, sizeof(uint64_t) * L.nb, cudaMemcpyDeviceToHost, st));
    KIFMM_CUDA(cudaMemcpyAsync(T.pbeg.data() + o, L.beg, sizeof(int) * L.nb, cudaMemcpyDeviceToHost, st));
    KIFMM_CUDA(cudaMemcpyAsync(T.pend.data() + o, L.end, sizeof(int) * L.nb, cudaMemcpyDeviceToHost, st));
    KIFMM_CUDA(cudaMemcpyAsync(T.parent.data() + o, L.par, sizeof(int) * L.nb, cudaMemcpyDeviceToHost, st));
    KIFMM_CUDA(cudaMemcpyAsync(T.leaf.data() + o, L.leaf, L.nb, cudaMemcpyDeviceToHost, st));
  }
  KIFMM_CUDA(cudaStreamSynchronize(st));
  for (auto& L : levs) { cudaFree(L.beg); cudaFree(L.end); cudaFree(L.par); cudaFree(L.key); cudaFree(L.leaf); }
  for (int l = 0; l < T.nlevels; ++l)
    for (int b = T.level_begin[l]; b < T.level_begin[l + 1]; ++b) {
      T.level[b] = l;
      T.parent[b] = l == 0 ? -1 : T.parent[b] + T.level_begin[l - 1];
    }
  T.nleaves = 0;
  for (uint8_t v : T.leaf) T.nleaves += v;
  KIFMM_CUDA(cudaMemcpyAsync(T.d_key, T.key.data(), sizeof(uint64_t) * nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.d_level, T.level.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.d_parent, T.parent.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.d_pbeg, T.pbeg.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.d_pend, T.pend.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.d_leaf, T.leaf.data(), nb, cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemsetAsync(T.d_child_begin, 0xff, sizeof(int) * nb, st));
  KIFMM_CUDA(cudaMemsetAsync(T.d_nchild, 0, sizeof(int) * nb, st));
  k_children<<<nblk(nb), 256, 0, st>>>(T.d_parent, T.d_level, nb, T.d_child_begin, T.d_nchild);
  k_geom<<<nblk(nb), 256, 0, st>>>(T.d_key, T.d_level, nb, T.lo_root[0], T.lo_root[1], T.lo_root[2], T.r0, T.d_geom);
  KIFMM_CUDA(cudaGetLastError());
  T.child_begin.resize(nb);
  T.nchild.resize(nb);
  KIFMM_CUDA(cudaMemcpyAsync(T.child_begin.data(), T.d_child_begin, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaMemcpyAsync(T.nchild.data(), T.d_nchild, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_skey);
  cudaFree(d_active);
  cudaFree(d_head);
  cudaFree(d_nsel);
  cudaFree(d_sel);
  return 0;
}

}  // namespace kifmm
