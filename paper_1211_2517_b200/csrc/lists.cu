// Device U/V/W/X interaction lists (definitions = reading O5):
//   V(B), level >= 2: children of the colleagues of parent(B) not adjacent to B, with
//         the offset id of (source - target) in the 316-entry table
//   U(B), leaf B:     all leaves adjacent to B (closed boxes intersect), incl. B
//   W(B), leaf B:     descendants A of colleagues of B with A not adjacent to B and
//                     parent(A) adjacent to B;   X(B) = {A : B in W(A)}
// Neighbour lookup = binary search of the Morton key in the level's sorted key range.
// Lists are emitted per target by one thread (count pass + fill pass), then put in
// canonical order with CUB radix sorts of 64-bit composite keys.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "fmm_internal.h"

namespace kifmm {

namespace {

__constant__ int c_level_begin[kMaxLevel + 3];
__constant__ short c_offset_id[343];  // (dx+3)*49 + (dy+3)*7 + (dz+3) -> id or -1

__device__ __forceinline__ uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
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

struct Anchor { int x, y, z, l; };

__device__ __forceinline__ Anchor anchor_of(const uint64_t* key, const int* level, int b) {
  uint64_t k = key[b];
  return Anchor{(int)compact3(k >> 2), (int)compact3(k >> 1), (int)compact3(k), level[b]};
}

// box at (level, anchor) or -1
__device__ int find_box(const uint64_t* __restrict__ key, int l, int ax, int ay, int az) {
  int lim = 1 << l;
  if (ax < 0 || ay < 0 || az < 0 || ax >= lim || ay >= lim || az >= lim) return -1;
  uint64_t k = (spread3(ax) << 2) | (spread3(ay) << 1) | spread3(az);
  int lo = c_level_begin[l], hi = c_level_begin[l + 1];
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    uint64_t km = key[mid];
    if (km == k) return mid;
    if (km < k) lo = mid + 1; else hi = mid;
  }
  return -1;
}

__device__ __forceinline__ bool adjacent(const Anchor& a, const Anchor& b) {
  int sa = kMaxLevel - a.l, sb = kMaxLevel - b.l;
  int64_t alo, ahi, blo, bhi;
  alo = (int64_t)a.x << sa; ahi = (int64_t)(a.x + 1) << sa; blo = (int64_t)b.x << sb; bhi = (int64_t)(b.x + 1) << sb;
  if (alo > bhi || blo > ahi) return false;
  alo = (int64_t)a.y << sa; ahi = (int64_t)(a.y + 1) << sa; blo = (int64_t)b.y << sb; bhi = (int64_t)(b.y + 1) << sb;
  if (alo > bhi || blo > ahi) return false;
  alo = (int64_t)a.z << sa; ahi = (int64_t)(a.z + 1) << sa; blo = (int64_t)b.z << sb; bhi = (int64_t)(b.z + 1) << sb;
  if (alo > bhi || blo > ahi) return false;
  return true;
}

struct TreeView {
  const uint64_t* key; const int* level; const int* parent; const int* child_begin; const int* nchild;
  const uint8_t* leaf; const int* pbeg; const int* pend;
};

// colleague table: coll[b*27 + dir], dir = (dx+1)*9 + (dy+1)*3 + (dz+1)
__global__ void k_colleagues(TreeView t, int nb, int* __restrict__ coll) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  Anchor a = anchor_of(t.key, t.level, b);
  int dir = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz, ++dir) coll[b * 27 + dir] = find_box(t.key, a.l, a.x + dx, a.y + dy, a.z + dz);
}

// V(B): FILL = false counts, FILL = true writes (tgt, src, off)
template <bool FILL>
__global__ void k_vlist(TreeView t, int nb, const int* __restrict__ coll, const int* __restrict__ off,
                        int* __restrict__ cnt, int4* __restrict__ out) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int lb = t.level[b];
  int c = 0;
  if (lb >= 2) {
    Anchor ab = anchor_of(t.key, t.level, b);
    int par = t.parent[b];
    int base = FILL ? off[b] : 0;
    for (int dir = 0; dir < 27; ++dir) {
      int cb = coll[par * 27 + dir];
      if (cb < 0) continue;
      int c0 = t.child_begin[cb], nc = t.nchild[cb];
      for (int ch = c0; ch < c0 + nc; ++ch) {
        Anchor aa = anchor_of(t.key, t.level, ch);
        if (adjacent(aa, ab)) continue;
        if (FILL) {
          int id = c_offset_id[(aa.x - ab.x + 3) * 49 + (aa.y - ab.y + 3) * 7 + (aa.z - ab.z + 3)];
          out[base + c] = make_int4(b, ch, id, 0);
        }
        ++c;
      }
    }
  }
  if (!FILL) cnt[b] = c;
}

// U(B) and W(B) for leaf B.  Stack-based descent into adjacent non-leaf colleagues.
template <bool FILL>
__global__ void k_uwlist(TreeView t, int nb, const int* __restrict__ coll, const int* __restrict__ offU,
                         const int* __restrict__ offW, int* __restrict__ cntU, int* __restrict__ cntW,
                         int2* __restrict__ outU, int2* __restrict__ outW) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int cu = 0, cw = 0;
  if (t.leaf[b]) {
    Anchor ab = anchor_of(t.key, t.level, b);
    int bu = FILL ? offU[b] : 0, bw = FILL ? offW[b] : 0;
    int coarse[27];
    int ncoarse = 0;
    int stack[8 * (kMaxLevel + 1)];
    int dir = 0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz, ++dir) {
          int ax = ab.x + dx, ay = ab.y + dy, az = ab.z + dz, lim = 1 << ab.l;
          if (ax < 0 || ay < 0 || az < 0 || ax >= lim || ay >= lim || az >= lim) continue;
          int c = coll[b * 27 + dir];
          if (c >= 0) {
            int sp = 0;
            stack[sp++] = c;
            while (sp > 0) {
              int x = stack[--sp];
              if (t.leaf[x]) {
                if (FILL) outU[bu + cu] = make_int2(b, x);
                ++cu;
                continue;
              }
              int c0 = t.child_begin[x], nc = t.nchild[x];
              for (int ch = c0; ch < c0 + nc; ++ch) {
                Anchor ac = anchor_of(t.key, t.level, ch);
                if (adjacent(ac, ab)) stack[sp++] = ch;
                else {
                  if (FILL) outW[bw + cw] = make_int2(b, ch);
                  ++cw;
                }
              }
            }
          } else {
            // coarser neighbour: the first existing ancestor of the same-level cell, if a leaf
            for (int l = ab.l - 1; l >= 0; --l) {
              int sh = ab.l - l;
              int y = find_box(t.key, l, ax >> sh, ay >> sh, az >> sh);
              if (y >= 0) {
                if (t.leaf[y]) {
                  bool seen = false;
                  for (int i = 0; i < ncoarse; ++i) seen |= coarse[i] == y;
                  if (!seen) {
                    coarse[ncoarse++] = y;
                    if (FILL) outU[bu + cu] = make_int2(b, y);
                    ++cu;
                  }
                }
                break;
              }
            }
          }
        }
  }
  if (!FILL) { cntU[b] = cu; cntW[b] = cw; }
}

__global__ void k_pair_keys(const int2* __restrict__ in, int n, bool swap, uint64_t* __restrict__ keys,
                            int* __restrict__ idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int2 v = in[i];
  keys[i] = swap ? ((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x : ((uint64_t)(uint32_t)v.x << 32) | (uint32_t)v.y;
  idx[i] = i;
}

__global__ void k_vkeys(const int4* __restrict__ in, int n, uint64_t* __restrict__ keys, int* __restrict__ idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((uint64_t)(uint32_t)in[i].z << 32) | (uint32_t)in[i].x;
  idx[i] = i;
}

__global__ void k_gather_v(const int4* __restrict__ in, const int* __restrict__ idx, int n, int4* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}

// decode sorted composite keys into (tgt, src, direct) records
__global__ void k_decode(const uint64_t* __restrict__ keys, int n, int mode, TreeView t, int wx, int2* __restrict__ outU,
                         int4* __restrict__ out4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int tg = (int)(keys[i] >> 32), sr = (int)(keys[i] & 0xffffffffu);
  if (mode == 0) { outU[i] = make_int2(tg, sr); return; }
  int direct;
  if (mode == 1) direct = (t.pend[sr] - t.pbeg[sr]) <= wx;                   // W: source subtree small
  else direct = t.leaf[tg] && (t.pend[tg] - t.pbeg[tg]) <= wx;               // X: target leaf small
  out4[i] = make_int4(tg, sr, direct, 0);
}

inline int nblk(int64_t n, int t = 256) { return std::max(1, (int)((n + t - 1) / t)); }

int exclusive_scan(const int* d_in, int* d_out, int n, cudaStream_t st, int* total) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_in, d_out, n, st);
  void* tmp;
  KIFMM_CUDA(cudaMalloc(&tmp, bytes));
  cub::DeviceScan::ExclusiveSum(tmp, bytes, d_in, d_out, n, st);
  int last_in = 0, last_out = 0;
  KIFMM_CUDA(cudaMemcpyAsync(&last_in, d_in + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaMemcpyAsync(&last_out, d_out + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  cudaFree(tmp);
  *total = last_in + last_out;
  return 0;
}

int sort_u64(uint64_t* keys, int* idx, int n, cudaStream_t st, uint64_t** keys_out, int** idx_out) {
  uint64_t* ko;
  int* io;
  KIFMM_CUDA(cudaMalloc(&ko, sizeof(uint64_t) * std::max(n, 1)));
  KIFMM_CUDA(cudaMalloc(&io, sizeof(int) * std::max(n, 1)));
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, ko, idx, io, n, 0, 64, st);
  void* tmp;
  KIFMM_CUDA(cudaMalloc(&tmp, std::max<size_t>(bytes, 1)));
  cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, ko, idx, io, n, 0, 64, st);
  KIFMM_CUDA(cudaGetLastError());
  cudaFree(tmp);
  *keys_out = ko;
  *idx_out = io;
  return 0;
}

}  // namespace

int build_lists_device(Plan& P, cudaStream_t st) {
  Tree& T = P.tree;
  Lists& L = P.lists;
  const int nb = T.nboxes;
  {
    int lb[kMaxLevel + 3] = {0};
    for (int l = 0; l <= T.nlevels && l < kMaxLevel + 3; ++l) lb[l] = T.level_begin[l];
    for (int l = T.nlevels + 1; l < kMaxLevel + 3; ++l) lb[l] = T.level_begin[T.nlevels];
    KIFMM_CUDA(cudaMemcpyToSymbolAsync(c_level_begin, lb, sizeof(lb), 0, cudaMemcpyHostToDevice, st));
    short ids[343];
    int id = 0;
    for (int i = 0; i < 343; ++i) {
      int dx = i / 49 - 3, dy = (i / 7) % 7 - 3, dz = i % 7 - 3;
      int m = std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz)));
      ids[i] = m > 1 ? (short)id++ : (short)-1;
    }
    KIFMM_CUDA(cudaMemcpyToSymbolAsync(c_offset_id, ids, sizeof(ids), 0, cudaMemcpyHostToDevice, st));
  }
  TreeView tv{T.d_key, T.d_level, T.d_parent, T.d_child_begin, T.d_nchild, T.d_leaf, T.d_pbeg, T.d_pend};
  int* d_coll;
  KIFMM_CUDA(cudaMalloc(&d_coll, sizeof(int) * 27 * (size_t)nb));
  k_colleagues<<<nblk(nb, 128), 128, 0, st>>>(tv, nb, d_coll);
  int *d_cnt, *d_off, *d_cnt2, *d_off2;
  KIFMM_CUDA(cudaMalloc(&d_cnt, sizeof(int) * nb));
  KIFMM_CUDA(cudaMalloc(&d_off, sizeof(int) * nb));
  KIFMM_CUDA(cudaMalloc(&d_cnt2, sizeof(int) * nb));
  KIFMM_CUDA(cudaMalloc(&d_off2, sizeof(int) * nb));
  // ---- V
  k_vlist<false><<<nblk(nb, 128), 128, 0, st>>>(tv, nb, d_coll, nullptr, d_cnt, nullptr);
  if (exclusive_scan(d_cnt, d_off, nb, st, &L.nV)) return -3;
  int4* d_vraw;
  KIFMM_CUDA(cudaMalloc(&d_vraw, sizeof(int4) * std::max(L.nV, 1)));
  k_vlist<true><<<nblk(nb, 128), 128, 0, st>>>(tv, nb, d_coll, d_off, nullptr, d_vraw);
  {
    uint64_t *k, *ko;
    int *ix, *io;
    KIFMM_CUDA(cudaMalloc(&k, sizeof(uint64_t) * std::max(L.nV, 1)));
    KIFMM_CUDA(cudaMalloc(&ix, sizeof(int) * std::max(L.nV, 1)));
    k_vkeys<<<nblk(L.nV), 256, 0, st>>>(d_vraw, L.nV, k, ix);
    if (sort_u64(k, ix, L.nV, st, &ko, &io)) return -3;
    KIFMM_CUDA(cudaMalloc(&L.d_V, sizeof(int4) * std::max(L.nV, 1)));
    k_gather_v<<<nblk(L.nV), 256, 0, st>>>(d_vraw, io, L.nV, L.d_V);
    KIFMM_CUDA(cudaStreamSynchronize(st));
    cudaFree(k); cudaFree(ko); cudaFree(ix); cudaFree(io); cudaFree(d_vraw);
  }
  // ---- U and W
  k_uwlist<false><<<nblk(nb, 64), 64, 0, st>>>(tv, nb, d_coll, nullptr, nullptr, d_cnt, d_cnt2, nullptr, nullptr);
  if (exclusive_scan(d_cnt, d_off, nb, st, &L.nU)) return -3;
  if (exclusive_scan(d_cnt2, d_off2, nb, st, &L.nW)) return -3;
  int2 *d_uraw, *d_wraw;
  KIFMM_CUDA(cudaMalloc(&d_uraw, sizeof(int2) * std::max(L.nU, 1)));
  KIFMM_CUDA(cudaMalloc(&d_wraw, sizeof(int2) * std::max(L.nW, 1)));
  k_uwlist<true><<<nblk(nb, 64), 64, 0, st>>>(tv, nb, d_coll, d_off, d_off2, nullptr, nullptr, d_uraw, d_wraw);
  KIFMM_CUDA(cudaGetLastError());
  L.nX = L.nW;
  KIFMM_CUDA(cudaMalloc(&L.d_U, sizeof(int2) * std::max(L.nU, 1)));
  KIFMM_CUDA(cudaMalloc(&L.d_W, sizeof(int4) * std::max(L.nW, 1)));
  KIFMM_CUDA(cudaMalloc(&L.d_X, sizeof(int4) * std::max(L.nX, 1)));
  for (int which = 0; which < 3; ++which) {
    int n = which == 0 ? L.nU : L.nW;
    const int2* src = which == 0 ? d_uraw : d_wraw;
    uint64_t *k, *ko;
    int *ix, *io;
    KIFMM_CUDA(cudaMalloc(&k, sizeof(uint64_t) * std::max(n, 1)));
    KIFMM_CUDA(cudaMalloc(&ix, sizeof(int) * std::max(n, 1)));
    k_pair_keys<<<nblk(n), 256, 0, st>>>(src, n, which == 2, k, ix);
    if (sort_u64(k, ix, n, st, &ko, &io)) return -3;
    k_decode<<<nblk(n), 256, 0, st>>>(ko, n, which, tv, P.wx, L.d_U, which == 1 ? L.d_W : L.d_X);
    KIFMM_CUDA(cudaStreamSynchronize(st));
    cudaFree(k); cudaFree(ko); cudaFree(ix); cudaFree(io);
  }
  cudaFree(d_uraw); cudaFree(d_wraw);
  cudaFree(d_coll); cudaFree(d_cnt); cudaFree(d_off); cudaFree(d_cnt2); cudaFree(d_off2);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace kifmm
