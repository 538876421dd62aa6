// Matvec kernels of the B200 KIFMM hot path.
//
// Two kernel families carry every step:
//  * k_ggs  — grouped gather-GEMM-scatter on the FP64 tensor pipe (DMMA.8x8x4):
//             Y[tgt] (+)= scale * Op[g] * X[src] over (src, tgt) pairs grouped by
//             operator g.  M2L (316 groups C_delta, P:136-144 compressed per
//             P:216-235), M2M (8 groups M~_o), L2L (8 groups L~_o),
//             and the projections S' (S2M), U^T (X list), T' (L2T),
//             U (W list) all run through it.
//  * k_eval — kernel evaluations target-set x source-segments, FP64 ALU + MUFU
//             rsqrt: near-field P2P (S2T), S2M / X check potentials,
//             L2T / W potentials from equivalent densities.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>

#include "bem.cuh"
#include "common.cuh"
#include "fmm_internal.h"

namespace kifmm {

// ----------------------------------------------------------------------------
// k_ggs: one CTA per tile of <= NT pairs sharing one operator.
//   Op  : M x K row-major (zero-padded), ops[op * op_stride]
//   X   : rows of K doubles (ldx), B operand columns gathered to shared memory
//   Y   : rows of M doubles (ldy); first `mvalid` entries written (store or atomic add)
// Warp w owns 8-row blocks rb = w, w+NW, ...; per k-step one DMMA per 8 pairs.
// ----------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(256) k_ggs(const GemmTile* __restrict__ tiles, const int2* __restrict__ pairs,
                                             const double* __restrict__ ops, int op_stride, int M, int K, int mvalid,
                                             const double* X, int ldx, double* Y, int ldy,
                                             int atomic) {
  extern __shared__ __align__(16) double sm[];
  const int SB = K + 4;   // B row stride: SB = 4 (mod 16)/12 -> conflict-free fragment loads
  const int SO = M + 2;   // output row stride
  double* Bs = sm;
  double* Os = sm + NT * SB;
  __shared__ int s_src[NT], s_tgt[NT];
  const GemmTile tile = tiles[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (threadIdx.x < NT) {
    int2 pr = threadIdx.x < tile.count ? pairs[tile.begin + threadIdx.x] : make_int2(-1, -1);
    s_src[threadIdx.x] = pr.x;
    s_tgt[threadIdx.x] = pr.y;
  }
  __syncthreads();
  // gather the B panel: column p = X[src_p][0:K) (zero for p >= count)
  const int K2 = K >> 1;
  for (int e = threadIdx.x; e < NT * K2; e += blockDim.x) {
    int p = e / K2, k2 = e - p * K2;
    int src = s_src[p];
    double2 v = make_double2(0.0, 0.0);
    if (src >= 0) v = reinterpret_cast<const double2*>(X + (size_t)src * ldx)[k2];
    reinterpret_cast<double2*>(Bs + p * SB)[k2] = v;
  }
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  const double* A0 = ops + (size_t)tile.op * op_stride;
  const double scale = tile.scale;
  for (int rb = warp; rb < (M >> 3); rb += nwarps) {
    double acc[NT / 8][2];
#pragma unroll
    for (int j = 0; j < NT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
    const double* Arow = A0 + (size_t)(rb * 8 + g) * K + t;
    for (int kc = 0; kc < K; kc += 64) {
      const int ksteps = min(16, (K - kc) >> 2);
      double a[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) a[s] = s < ksteps ? __ldg(Arow + kc + 4 * s) : 0.0;
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        if (s < ksteps) {
          const double* bp = Bs + g * SB + kc + 4 * s + t;
#pragma unroll
          for (int j = 0; j < NT / 8; ++j) dmma_8x8x4(acc[j][0], acc[j][1], a[s], bp[j * 8 * SB]);
        }
      }
    }
    // D(g, 2t + c) of n-block j = output row rb*8+g of pair j*8+2t+c
#pragma unroll
    for (int j = 0; j < NT / 8; ++j) {
      Os[(j * 8 + 2 * t) * SO + rb * 8 + g] = acc[j][0] * scale;
      Os[(j * 8 + 2 * t + 1) * SO + rb * 8 + g] = acc[j][1] * scale;
    }
  }
  __syncthreads();
  // scatter: one warp per pair row, coalesced over the M outputs
  for (int p = warp; p < tile.count; p += nwarps) {
    double* y = Y + (size_t)s_tgt[p] * ldy;
    const double* o = Os + p * SO;
    if (atomic) {
      for (int e = lane; e < mvalid; e += 32) atomicAdd(y + e, o[e]);
    } else {
      for (int e = lane; e < mvalid; e += 32) y[e] = o[e];
    }
  }
}

// ----------------------------------------------------------------------------
// k_ggs_sq: the square (M = K = KP) grouped GEMM of M2L / M2M / L2L, persistent.
// Each CTA walks a contiguous range of tiles (consecutive tiles mostly share the
// operator, so its DMMA A-fragments stay in registers).  The B panel of the next
// tile is gathered with cp.async (LDGSTS, L2 -> smem, 16 B per copy) while the
// current tile runs on the tensor pipe; results are staged in smem and
// scatter-added with coalesced RED.F64 rows.  Warp w owns output rows 8w..8w+7.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int KP, int NT>
__global__ void __launch_bounds__(KP * 4) k_ggs_sq(const GemmTile* __restrict__ tiles, int ntiles,
                                                 const int2* __restrict__ pairs, const double* __restrict__ ops,
                                                 int mvalid, const double* X, double* Y, int atomic) {
  constexpr int NW = KP / 8;        // warps: one 8-row block each
  constexpr int NTH = NW * 32;
  constexpr int SB = KP + 4;        // conflict-free B fragment loads
  constexpr int KS = KP / 4;        // k-steps
  constexpr int K2 = KP / 2;        // 16-byte chunks per row
  extern __shared__ __align__(16) double sm[];
  __shared__ int2 s_pair[3][NT];    // pair indices, two tiles ahead
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  if (t0 >= t1) return;

  // pair indices of tile ti -> s_pair[slot] (cp.async, 8 B each; -1 padding)
  auto load_pairs = [&](const GemmTile& tl, int slot) {
    for (int p = threadIdx.x; p < NT; p += NTH) {
      if (p < tl.count) cp_async8(&s_pair[slot][p], pairs + tl.begin + p);
      else s_pair[slot][p] = make_int2(-1, -1);
    }
  };
  // B panel of a tile whose pairs are in s_pair[slot] -> buffer buf
  auto gather = [&](int slot, int buf) {
    double* B = sm + buf * NT * SB;
    for (int p = warp; p < NT; p += NW) {
      const int src = s_pair[slot][p].x;
      for (int c = lane; c < K2; c += 32) {
        double* dst = B + p * SB + 2 * c;
        if (src >= 0) cp_async16(dst, X + (size_t)src * KP + 2 * c);
        else { dst[0] = 0.0; dst[1] = 0.0; }
      }
    }
  };

  const GemmTile nil{0, 0, 0, 0, 0.0};
  GemmTile d0 = tiles[t0];
  GemmTile d1 = t0 + 1 < t1 ? tiles[t0 + 1] : nil;
  GemmTile d2 = t0 + 2 < t1 ? tiles[t0 + 2] : nil;
  load_pairs(d0, 0);
  load_pairs(d1, 1);
  cp_async_commit();
  cp_async_wait0();
  __syncthreads();
  gather(0, 0);
  cp_async_commit();

  double a[KS];
  int cur_op = -1;
  for (int ti = t0; ti < t1; ++ti) {
    const int k = ti - t0;
    const int buf = k & 1, slot = k % 3;
    cp_async_wait0();
    __syncthreads();  // B(ti), pairs(ti), pairs(ti+1) landed; zero fills visible
    GemmTile d3 = ti + 3 < t1 ? tiles[ti + 3] : nil;  // register prefetch, used next iteration
    if (ti + 1 < t1) gather((k + 1) % 3, buf ^ 1);
    if (ti + 2 < t1) load_pairs(d2, (k + 2) % 3);
    cp_async_commit();
    if (d0.op != cur_op) {
      cur_op = d0.op;
      const double* Arow = ops + (size_t)cur_op * KP * KP + (size_t)(warp * 8 + g) * KP + t;
#pragma unroll
      for (int s = 0; s < KS; ++s) a[s] = __ldg(Arow + 4 * s);
    }
    const double* B = sm + buf * NT * SB;
    double acc[NT / 8][2];
#pragma unroll
    for (int j = 0; j < NT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const double* bp = B + g * SB + 4 * s + t;
#pragma unroll
      for (int j = 0; j < NT / 8; ++j) dmma_8x8x4(acc[j][0], acc[j][1], a[s], bp[j * 8 * SB]);
    }
    // scatter straight from the accumulators: lane (g, t) holds rows warp*8+g of
    // pairs j*8+2t and j*8+2t+1 (fire-and-forget RED.F64, 64 B contiguous per pair)
    const double scale = d0.scale;
    const int row = warp * 8 + g;
    if (row < mvalid) {
#pragma unroll
      for (int j = 0; j < NT / 8; ++j) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int tg = s_pair[slot][j * 8 + 2 * t + c].y;
          if (tg >= 0) {
            double* y = Y + (size_t)tg * KP + row;
            if (atomic) atomicAdd(y, acc[j][c] * scale);
            else *y = acc[j][c] * scale;
          }
        }
      }
    }
    d0 = d1; d1 = d2; d2 = d3;
  }
}

// ----------------------------------------------------------------------------
// k_m2l_sib16: M2L grouped by sibling structure.  Every V pair (B, A) joins child a
// of P = parent(B) with child b of a colleague Q = P + delta of P, and
// its operator is C_{2 delta + b - a}.  A column = (target B, source parent Q);
// a tile = up to NT columns of one class (delta, a).  For each non-adjacent b the
// CTA gathers q^'(child b of Q) (zero if absent) and accumulates
// C_{2 delta + b - a} q^' in the DMMA accumulators, so each target receives one
// RED per (target, delta) instead of one per (target, offset).
//
// Pipeline (one "step" = one operator b of one tile):
//   * tiles are handed out dynamically (atomic counter; tiles sorted longest
//     first), the metadata of the next tile is fetched one tile ahead into a
//     3-slot ring;
//   * the B panel of step i+1 is gathered with cp.async (LDGSTS) while step i runs;
//   * the operator rows (A fragments) stream through registers in chunks of CH
//     k-steps, chunk c+1 (or chunk 0 of the next step's operator) loaded while
//     chunk c feeds the tensor pipe.
//
// The m16n8k8 FP64 MMA (kp = 32, 64, 104; SASS DMMA.8x8x4): each B fragment serves two
// 8-row halves, halving the shared-memory loads per DMMA.  RB = ceil(kp/16) row blocks
// (kp = 104: 7 blocks, rows 104..111 zero — 7.7% padded M, K unpadded); warp w owns rows
// 16 (w % RB) .. +16 and columns (w / RB) * NCW .. +NCW of a tile.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], const double (&a)[4], double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
}

template <int KP>
struct Sib16Shape {
  static constexpr int RB = (KP + 15) / 16;             // row blocks of 16 (rows >= KP are zero)
  static constexpr int CS = RB * 2 <= 8 ? 8 / RB : 1;   // column groups
  static constexpr int NW = RB * CS;                    // warps
};

template <int KP, int NT, int MINB>
__global__ void __launch_bounds__(Sib16Shape<KP>::NW * 32, MINB) k_m2l_sib16(
    const int4* __restrict__ tiles, int ntiles, const int* __restrict__ cols, const int* __restrict__ classes,
    const double* __restrict__ C, int mvalid, const double* X, double* Y, int* __restrict__ counter, int zero_row) {
  constexpr int RB = Sib16Shape<KP>::RB;
  constexpr int CS = Sib16Shape<KP>::CS;
  constexpr int NW = Sib16Shape<KP>::NW;
  constexpr int NTH = NW * 32;
  constexpr int SB = KP + 4;
  constexpr int K2 = KP / 2;
  constexpr int CW = 9;
  constexpr int NCW = NT / CS;       // columns per warp
  constexpr int NB = NCW / 8;        // n-blocks per warp
  constexpr int KS8 = KP / 8;        // k8-steps
  constexpr int CH = KS8 % 2 == 0 ? 2 : 1;  // k8-steps per A chunk
  constexpr int NCH = KS8 / CH;
  static_assert(KS8 % CH == 0 && NB >= 1, "tile shape");
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_meta[3][NT * CW];
  __shared__ int s_cls[3][17];  // each ring slot's class record (steps, children, offset ids)
  __shared__ int s_tile[3];
  __shared__ __align__(8) uint64_t s_full[2];  // one mbarrier per B-panel buffer
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp % RB) * 16;
  const int cbase = (warp / RB) * NCW;
  int ti = blockIdx.x;
  if (ti >= ntiles) return;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&s_full[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase[2] = {0u, 0u};  // parity of each buffer's next completion

  // a tile's column records and its class record into ring slot `slot` (read after the
  // next CTA barrier: no dependent global load at the tile boundary)
  // (4-byte cp.async: the warp does not wait for the records here; they are waited for
  // before the barrier of the current tile's last step, where they are first read)
  auto fetch_meta = [&](int tid, int slot) {
    const int4 tl = tiles[tid];
    for (int e = threadIdx.x; e < NT * CW; e += NTH) {
      const int c = e / CW;
      if (c < tl.z)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_meta[slot][e])),
                     "l"(cols + (size_t)tl.y * CW + e));
      else
        s_meta[slot][e] = -1;
    }
    if (threadIdx.x < 17)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_cls[slot][threadIdx.x])),
                   "l"(classes + tl.x * 17 + threadIdx.x));
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // B panel of one step: every column's source row (KP doubles, contiguous) is one
  // cp.async.bulk copy (SASS UBLKCP) issued by warp 0, completing on the buffer's mbarrier;
  // absent sources read the zero row of q^' (row zero_row, never written)
  auto gather = [&](int slot, int b, int buf) {
    if (warp != 0) return;
    const uint32_t bar = (unsigned)__cvta_generic_to_shared(&s_full[buf]);
    if (lane == 0) {
      // the buffer was last read through the generic proxy (all warps passed the barrier)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(NT * KP * 8) : "memory");
    }
    __syncwarp();
    double* Bd = sm + buf * NT * SB;
    for (int p = lane; p < NT; p += 32) {
      const int src = s_meta[slot][p * CW + 1 + b];
      const double* srow = X + (size_t)(src >= 0 ? src : zero_row) * KP;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (unsigned)__cvta_generic_to_shared(Bd + p * SB)),
          "l"(srow), "r"(KP * 8), "r"(bar)
          : "memory");
    }
  };
  auto wait_panel = [&](int buf) {
    const uint32_t bar = (unsigned)__cvta_generic_to_shared(&s_full[buf]);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar), "r"(phase[buf])
          : "memory");
    phase[buf] ^= 1u;
  };
  // A fragment of k8-step ks: rows r0+g, r0+g+8; columns 8 ks + t, 8 ks + t + 4
  auto op_rows = [&](int id) { return C + (size_t)id * KP * KP + (size_t)(r0 + g) * KP + t; };
  const bool lo_ok = r0 + g < KP, hi_ok = r0 + g + 8 < KP;  // padded rows (KP % 16 != 0) read as zero
  auto load_a = [&](const double* Ar, int ks, double (&a)[4]) {
    a[0] = lo_ok ? __ldg(Ar + 8 * ks) : 0.0;
    a[1] = hi_ok ? __ldg(Ar + 8 * KP + 8 * ks) : 0.0;
    a[2] = lo_ok ? __ldg(Ar + 8 * ks + 4) : 0.0;
    a[3] = hi_ok ? __ldg(Ar + 8 * KP + 8 * ks + 4) : 0.0;
  };

  int slot = 0;
  fetch_meta(ti, 0);
  if (threadIdx.x == 0) s_tile[1] = gridDim.x + atomicAdd(counter, 1);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int* cls = s_cls[0];
  gather(0, cls[1], 0);
  double a_cur[CH][4];
  const double* Aop = op_rows(cls[9]);
#pragma unroll
  for (int s = 0; s < CH; ++s) load_a(Aop, s, a_cur[s]);
  int buf = 0;
  double acc[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

  while (true) {
    const int nv = cls[0];
    const int nslot = slot == 2 ? 0 : slot + 1;
    const int tnext = s_tile[nslot];
    // thread 0 claims the tile after next at this tile's first step and publishes it just
    // before its last step's barrier: on multi-step tiles the atomic's round trip runs under
    // the MMAs instead of holding warp 0 (and so the CTA) at the first step's barrier
    int claimed = 0;
    for (int jb = 0; jb < nv; ++jb) {
      const bool last = jb + 1 == nv;
      if (jb == 0 && tnext < ntiles) {
        fetch_meta(tnext, nslot);
        if (threadIdx.x == 0) claimed = gridDim.x + atomicAdd(counter, 1);
      }
      if (last && threadIdx.x == 0 && tnext < ntiles) s_tile[nslot == 2 ? 0 : nslot + 1] = claimed;
      if (last) asm volatile("cp.async.wait_all;\n" ::: "memory");  // the next tile's records
      wait_panel(buf);  // this step's B panel has landed
      __syncthreads();  // every warp is done with the other buffer (and the new s_meta is visible)
      const double* Anext = nullptr;
      if (!last) {
        gather(slot, cls[2 + jb], buf ^ 1);
        Anext = op_rows(cls[9 + jb + 1]);
      } else if (tnext < ntiles) {
        const int* ncls = s_cls[nslot];
        gather(nslot, ncls[1], buf ^ 1);
        Anext = op_rows(ncls[9]);
      }
      // B fragment (k8-step ks, n-block j): b0 = B[8ks + t][col], b1 = B[8ks + t + 4][col], col = cbase + 8j + g
      const double* B = sm + buf * NT * SB + (size_t)(cbase + g) * SB + t;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        double a_nxt[CH][4];
        const bool more = c + 1 < NCH;
        if (more || Anext) {
#pragma unroll
          for (int s = 0; s < CH; ++s) load_a(more ? Aop : Anext, more ? (c + 1) * CH + s : s, a_nxt[s]);
        }
#pragma unroll
        for (int s = 0; s < CH; ++s) {
          const int ks = c * CH + s;
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            const double* bp = B + (size_t)j * 8 * SB + 8 * ks;
            dmma_16x8x8(acc[j], a_cur[s], bp[0], bp[4]);
          }
        }
#pragma unroll
        for (int s = 0; s < CH; ++s)
#pragma unroll
          for (int e = 0; e < 4; ++e) a_cur[s][e] = a_nxt[s][e];
      }
      Aop = Anext;
      buf ^= 1;
      if (last) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int tg = s_meta[slot][(cbase + j * 8 + 2 * t + c) * CW];
            if (tg >= 0) {
              if (r0 + g < mvalid) atomicAdd(Y + (size_t)tg * KP + r0 + g, acc[j][c]);
              if (r0 + g + 8 < mvalid) atomicAdd(Y + (size_t)tg * KP + r0 + g + 8, acc[j][2 + c]);
            }
          }
          acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        }
      }
    }
    if (tnext >= ntiles) break;
    ti = tnext;
    slot = nslot;
    cls = s_cls[slot];
  }
}

// ----------------------------------------------------------------------------
// k_eval: one CTA per target item.  Targets are either the points of a box
// (SURF_TGT = false; result stored to out[pbeg + i]) or the n surface points
// c_B + rad * e_i of a box (SURF_TGT = true; result stored to out[row * ldo + i]).
// Sources are a list of segments per item: (kind, a, b, len):
//   kind 0: points pts[a .. a+len)                       (P2P / S2M / X sources)
//   kind 1: surface of box b, radius r_b * f_out, densities eqd1[a * ldq + m]   (L2T)
//   kind 2: surface of box b, radius r_b * f_in,  densities eqd2[a * ldq + m]   (W)
// Thread t handles target t % mm over source slice t / mm (mm = targets in this
// pass); the slices are summed in shared memory; the sum is scaled by 1/(4 pi).
// ----------------------------------------------------------------------------
struct EvalArgs {
  const double4* pts;
  const double4* geom;
  const int* pbeg;
  const int* pend;
  const int4* items;     // (box, out row, 0, 0)
  const int* seg_off;    // CSR over items
  const int4* segs;      // (kind, a, b, len)
  const double* eqd1;
  const double* eqd2;
  const double* surf;    // unit surface grid, n x 3
  int ldq;               // equivalent-density row stride
  int n;                 // surface points
  double f_in, f_out;
  double tgt_f;          // surface factor of SURF_TGT targets
  double* out;
  int ldo;
  int accumulate;        // k_eval: out += result (leaf-op mode: L2T already stored)
  const double4* nrm;    // sorted source normals (double layer), else NULL
  const double4* tri;    // sorted triangles (BEM elements), else NULL
};

// Double-layer source term: q_j (x - y_j).n_j / r^3 with the source staged
// as (y, q n_x) and (q n_y, q n_z); 1/(4 pi) applied once per sum.
template <bool CHECK>
__device__ __forceinline__ double dl_term(double dx, double dy, double dz, double wx, double wy, double wz) {
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double ri = CHECK ? rinv_or_zero(r2) : rinv_nonzero(r2);
  const double dot = fma(dz, wz, fma(dy, wy, dx * wx));
  return dot * ri * (ri * ri);
}

constexpr int EV_SEG = 128;   // segments per batch (= 32 lanes x 4)
constexpr int EV_TB = 4;      // targets per thread (register blocking)

// Sum over sources sbuf[j0, j1) step G into TB accumulators; CHECK: pairs with
// r^2 == 0 contribute 0 (reading Q1), else r > 0 is known.
template <int TB, bool CHECK, bool DL = false>
__device__ __forceinline__ void eval_sources(const double4* sbuf, const double2* sbufw, int j0, int j1, int G,
                                             const double (&x)[TB][3], double (&acc)[TB]) {
#pragma unroll 2
  for (int j = j0; j < j1; j += G) {
    const double4 sv = sbuf[j];
    if (DL) {
      const double2 sw = sbufw[j];
#pragma unroll
      for (int u = 0; u < TB; ++u)
        acc[u] += dl_term<CHECK>(x[u][0] - sv.x, x[u][1] - sv.y, x[u][2] - sv.z, sv.w, sw.x, sw.y);
    } else {
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        acc[u] = fma(sv.w, CHECK ? rinv_or_zero(r2) : rinv_nonzero(r2), acc[u]);
      }
    }
  }
}

// One pass over up to TB * NT targets [t0, t0 + mm) of item `it`: thread (ti, gi)
// owns targets t0 + ti + u * mq (u < TB, mq = ceil(mm / TB)) and sweeps source slice
// gi (stride G = NT / mq); slices are summed in shared memory.  Sources are the
// concatenated segments, staged EV_CH at a time into a double buffer (point sources
// by cp.async, so chunk c + 1 lands while chunk c is evaluated); the first `nchk`
// sources are tested for r = 0.
template <int TB, int EV_CH, bool DL>
__device__ __forceinline__ void eval_pass(const EvalArgs& A, const int4& it, int tbeg, int t0, int mm, int sb, int se,
                                          int nchk, double4 (*sbuf)[EV_CH], double2 (*sbufw)[EV_CH], double* red,
                                          int* s_pref, int4* s_seg) {
  const int NT = blockDim.x;
  const int lane = threadIdx.x & 31;
  const int mq = (mm + TB - 1) / TB;
  const int G = NT / mq;
  const int ti = threadIdx.x % mq, gi = threadIdx.x / mq;
  const bool act = gi < G;
  double x[TB][3], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    const int i = ti + u * mq;
    acc[u] = 0.0;
    if (act && i < mm) {
      const double4 p = A.pts[tbeg + t0 + i];
      x[u][0] = p.x; x[u][1] = p.y; x[u][2] = p.z;
    } else {  // padding target far from everything (result discarded)
      x[u][0] = 1e100; x[u][1] = 0.0; x[u][2] = 0.0;
    }
  }
  // stage sources [c0, c0 + cn) of the current segment batch into buffer b
  auto stage = [&](int ns, int c0, int cn, int b) {
    for (int f = threadIdx.x; f < cn; f += NT) {
      const int fi = c0 + f;
      int lo = 0, hi = ns;  // last segment with prefix <= fi
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= fi) lo = mid; else hi = mid;
      }
      const int4 sg = s_seg[lo];
      const int j = fi - s_pref[lo];
      if (sg.x == 0 && DL) {  // double-layer source: (y, q n_x), (q n_y, q n_z)
        const double4 p = A.pts[sg.y + j], nv = A.nrm[sg.y + j];
        sbuf[b][f] = make_double4(p.x, p.y, p.z, p.w * nv.x);
        sbufw[b][f] = make_double2(p.w * nv.y, p.w * nv.z);
      } else if (sg.x == 0) {
        const double* src = reinterpret_cast<const double*>(A.pts + sg.y + j);
        double* dst = reinterpret_cast<double*>(&sbuf[b][f]);
        cp_async16(dst, src);
        cp_async16(dst + 2, src + 2);
      } else {
        const double4 gs = A.geom[sg.z];
        const double rad = gs.w * (sg.x == 1 ? A.f_out : A.f_in);
        const double* q = (sg.x == 1 ? A.eqd1 : A.eqd2) + (size_t)sg.y * A.ldq;
        sbuf[b][f] = make_double4(gs.x + rad * A.surf[3 * j], gs.y + rad * A.surf[3 * j + 1],
                                  gs.z + rad * A.surf[3 * j + 2], q[j]);
      }
    }
  };
  int base = 0;  // sources consumed before this segment batch
  for (int s0 = sb; s0 < se; s0 += EV_SEG) {
    const int ns = min(EV_SEG, se - s0);
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: segment table + exclusive prefix of lengths
      int len[4], run = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int sidx = lane * 4 + u;
        len[u] = 0;
        if (sidx < ns) {
          int4 sg = A.segs[s0 + sidx];
          s_seg[sidx] = sg;
          len[u] = sg.w;
        }
        run += len[u];
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int excl = incl - run;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int sidx = lane * 4 + u;
        if (sidx < ns) s_pref[sidx] = excl;
        excl += len[u];
      }
      if (lane == 31) s_pref[ns] = incl;
    }
    __syncthreads();
    const int total = s_pref[ns];
    stage(ns, 0, min(EV_CH, total), 0);
    cp_async_commit();
    int b = 0;
    for (int c0 = 0; c0 < total; c0 += EV_CH) {
      const int cn = min(EV_CH, total - c0);
      cp_async_wait0();
      __syncthreads();  // chunk c0 staged by every thread; buffer b ^ 1 free
      if (c0 + EV_CH < total) stage(ns, c0 + EV_CH, min(EV_CH, total - c0 - EV_CH), b ^ 1);
      cp_async_commit();
      if (act) {
        const int split = min(cn, max(0, nchk - (base + c0)));  // checked prefix of this chunk
        const int j0 = gi;
        int jc = j0;
        if (split > 0) {
          eval_sources<TB, true, DL>(sbuf[b], sbufw[b], j0, split, G, x, acc);
          jc = j0 + ((split - j0 + G - 1) / G) * G;  // first j >= split in this slice
        }
        eval_sources<TB, false, DL>(sbuf[b], sbufw[b], jc, cn, G, x, acc);
      }
      b ^= 1;
    }
    base += total;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < TB; ++u) red[u * NT + threadIdx.x] = acc[u];
  __syncthreads();
  for (int i = threadIdx.x; i < mm; i += NT) {
    const int u = i / mq, tl = i - u * mq;
    double sum = 0;
    for (int gg = 0; gg < G; ++gg) sum += red[u * NT + gg * mq + tl];
    double* o = A.out + tbeg + t0 + i;
    *o = A.accumulate ? *o + sum * kInv4Pi : sum * kInv4Pi;
  }
}

// ----------------------------------------------------------------------------
// k_p2p_sym: symmetric near field.  G is symmetric, so an unordered pair of
// leaves {B, A} (a U pair, or a direct W / X pair whose source is a leaf) is
// evaluated ONCE for both directions:  p_i += sum_j G_ij q_j (i in B) and
// p_j += sum_i G_ij q_i (j in A), i.e. ~13 FP64 ops per pair instead of 24.
// One warp per pair.  Lane l holds TB targets of B (l + 32 u); A's points stream
// through a per-warp shared buffer 32 at a time; lane l accumulates, for each of
// the 32 sources j, s_j = sum_u q_u G(x_u, y_j), and a butterfly reduce-scatter
// across the warp leaves sum_l s_j on lane j (31 shuffles per 32 x 32 TB pairs).
// Both sides are added to the potential with RED (the pair's leaves also receive
// other contributions).  Distinct leaves never share a point position.
// ----------------------------------------------------------------------------
constexpr int SYM_WARPS = 4;
constexpr int SYM_SB = 16;    // sources per batch (partial sums per lane)
constexpr int SYM_CH = 256;   // source points staged per warp

// targets pts[tb0, tb0 + mt) (TB per lane) against the staged sources sbuf[0, cn)
// (global index sb0 + j); both sides' sums go to pot with RED
template <int TB>
__device__ __forceinline__ void p2p_sym_pass(const double4* __restrict__ pts, int tb0, int mt, int sb0, int cn,
                                             const double4* sbuf, double* __restrict__ pot) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double x[TB][3], q[TB], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    const int i = lane + 32 * u;
    acc[u] = 0.0;
    if (i < mt) {
      const double4 p = pts[tb0 + i];
      x[u][0] = p.x; x[u][1] = p.y; x[u][2] = p.z; q[u] = p.w;
    } else {
      x[u][0] = 1e100; x[u][1] = 0.0; x[u][2] = 0.0; q[u] = 0.0;
    }
  }
  for (int j0 = 0; j0 < cn; j0 += SYM_SB) {
    double v[SYM_SB];
#pragma unroll
    for (int j = 0; j < SYM_SB; ++j) {
      const double4 sv = sbuf[j0 + j];
      double sj = 0.0;
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
        const double r = rinv_nonzero(fma(dz, dz, fma(dy, dy, dx * dx)));
        acc[u] = fma(sv.w, r, acc[u]);
        sj = fma(q[u], r, sj);
      }
      v[j] = sj;
    }
    // reduce-scatter within each 16-lane half, then fold the halves: lane l ends with
    // the sum over all lanes of the original v[l % 16]
#pragma unroll
    for (int off = SYM_SB / 2; off >= 1; off >>= 1) {
      const bool up = lane & off;
#pragma unroll
      for (int i = 0; i < off; ++i) {
        const double send = up ? v[i] : v[i + off];
        const double keep = up ? v[i + off] : v[i];
        v[i] = keep + __shfl_xor_sync(FULL, send, off);
      }
    }
    v[0] += __shfl_xor_sync(FULL, v[0], 16);
    if (lane < SYM_SB && j0 + lane < cn) atomicAdd(pot + sb0 + j0 + lane, v[0] * kInv4Pi);
  }
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    const int i = lane + 32 * u;
    if (i < mt) atomicAdd(pot + tb0 + i, acc[u] * kInv4Pi);
  }
}

template <int MINB>
__global__ void __launch_bounds__(SYM_WARPS * 32, MINB) k_p2p_sym(const int2* __restrict__ pairs, int npairs,
                                                              const double4* __restrict__ pts,
                                                              const int* __restrict__ pbeg, const int* __restrict__ pend,
                                                              double* __restrict__ pot) {
  __shared__ __align__(16) double4 sbuf[SYM_WARPS][SYM_CH];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pi = blockIdx.x * SYM_WARPS + w;
  if (pi >= npairs) return;
  const int2 pr = pairs[pi];
  const int tb0 = pbeg[pr.x], mt_all = pend[pr.x] - tb0;
  const int sb0 = pbeg[pr.y], ms = pend[pr.y] - sb0;
  for (int c0 = 0; c0 < ms; c0 += SYM_CH) {
    const int cn = min(SYM_CH, ms - c0);
    const int cpad = (cn + SYM_SB - 1) / SYM_SB * SYM_SB;
    __syncwarp();
    for (int j = lane; j < cpad; j += 32)  // padding sources: zero density, far away
      sbuf[w][j] = j < cn ? pts[sb0 + c0 + j] : make_double4(-1e100, 0.0, 0.0, 0.0);
    __syncwarp();
    for (int t0 = 0; t0 < mt_all; t0 += 96) {
      const int mt = min(96, mt_all - t0);
      if (mt > 64) p2p_sym_pass<3>(pts, tb0 + t0, mt, sb0 + c0, cn, sbuf[w], pot);
      else if (mt > 32) p2p_sym_pass<2>(pts, tb0 + t0, mt, sb0 + c0, cn, sbuf[w], pot);
      else p2p_sym_pass<1>(pts, tb0 + t0, mt, sb0 + c0, cn, sbuf[w], pot);
    }
  }
}

// k_eval: one CTA per target leaf (item (box, row, 0, 0)): potentials of the leaf's
// points from its source segments (kind, a, b, len):
//   kind 0: points pts[a .. a+len)                       (P2P: U, direct W / X)
//   kind 1: surface of box b, radius r_b * f_out, densities eqd1[a * ldq + m]   (L2T)
//   kind 2: surface of box b, radius r_b * f_in,  densities eqd2[a * ldq + m]   (W)
// chk_self: the first m_B sources are the leaf's own points (r = 0 possible).
template <int NT, int CH, bool DL = false>
__global__ void __launch_bounds__(NT) k_eval(EvalArgs A, int chk_self) {
  __shared__ __align__(16) double4 sbuf[2][CH];
  __shared__ __align__(16) double2 sbufw[2][DL ? CH : 1];
  __shared__ double red[EV_TB * NT];
  __shared__ int s_pref[EV_SEG + 1];
  __shared__ int4 s_seg[EV_SEG];
  const int4 it = A.items[blockIdx.x];
  const int tbeg = A.pbeg[it.x], m = A.pend[it.x] - tbeg;
  const int sb = A.seg_off[blockIdx.x], se = A.seg_off[blockIdx.x + 1];
  const int nchk = chk_self ? m : 0;
  for (int t0 = 0; t0 < m; t0 += EV_TB * NT) {
    const int mm = min(m - t0, EV_TB * NT);
    // (single layer: the weight buffer is a 1-element placeholder, never indexed)
    double2 (*sw)[CH] = reinterpret_cast<double2 (*)[CH]>(&sbufw[0][0]);
    if (mm >= 12) eval_pass<EV_TB, CH, DL>(A, it, tbeg, t0, mm, sb, se, nchk, sbuf, sw, red, s_pref, s_seg);
    else eval_pass<2, CH, DL>(A, it, tbeg, t0, mm, sb, se, nchk, sbuf, sw, red, s_pref, s_seg);
  }
}

// ----------------------------------------------------------------------------
// k_chk: check potentials of S2M (UC of a leaf at (3-2d) r, sources =
// the leaf's points) and of the X list (DC of the target at (1+d) r, sources = the
// X source leaf).  One warp per item, no block barriers: the warp stages 32 sources
// at a time in shared memory and every lane accumulates CHK_TB check points.
// ----------------------------------------------------------------------------
constexpr int CHK_WARPS = 8;
#ifndef KIFMM_CHK_MINB
#define KIFMM_CHK_MINB 3  // 80 registers: 3 CTAs per SM (the default heuristic took 92: 2 CTAs)
#endif

// BEM X-list check potentials (P:445-456 restated for S2L): one warp per item, each lane
// CHK_TB check points, the source elements' integrals by bem_integral
template <int CHK_TB>
__global__ void __launch_bounds__(CHK_WARPS * 32) k_chk_bem(EvalArgs A, int nitems) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int item = blockIdx.x * CHK_WARPS + w;
  if (item >= nitems) return;
  const int4 it = A.items[item];
  const double4 gb = A.geom[it.x];
  const int4 sg = A.segs[A.seg_off[item]];
  const double rad = gb.w * A.tgt_f;
  for (int r0 = 0; r0 < A.n; r0 += 32 * CHK_TB)
    for (int u = 0; u < CHK_TB; ++u) {
      const int i = r0 + lane + 32 * u;
      if (i >= A.n) continue;
      const double x[3] = {gb.x + rad * A.surf[3 * i], gb.y + rad * A.surf[3 * i + 1], gb.z + rad * A.surf[3 * i + 2]};
      double acc = 0.0;
      for (int j = 0; j < sg.w; ++j)
        acc += bem_integral(load_tri(A.tri + 3 * (int64_t)(sg.y + j)), x, false) * A.pts[sg.y + j].w;
      A.out[(size_t)it.y * A.ldo + i] = acc;
    }
}

template <int CHK_TB, bool DL = false>
__global__ void __launch_bounds__(CHK_WARPS * 32, KIFMM_CHK_MINB) k_chk(EvalArgs A, int nitems) {
  __shared__ double4 ssrc[CHK_WARPS][32];
  __shared__ double2 ssrcw[CHK_WARPS][DL ? 32 : 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int item = blockIdx.x * CHK_WARPS + w;
  if (item >= nitems) return;
  const int4 it = A.items[item];
  const double4 gb = A.geom[it.x];
  const int4 sg = A.segs[A.seg_off[item]];  // one point segment per item
  const double rad = gb.w * A.tgt_f;
  const int n = A.n;
  for (int r0 = 0; r0 < n; r0 += 32 * CHK_TB) {
    double x[CHK_TB][3], acc[CHK_TB];
#pragma unroll
    for (int u = 0; u < CHK_TB; ++u) {
      const int i = r0 + lane + 32 * u;
      acc[u] = 0.0;
      if (i < n) {
        x[u][0] = gb.x + rad * A.surf[3 * i];
        x[u][1] = gb.y + rad * A.surf[3 * i + 1];
        x[u][2] = gb.z + rad * A.surf[3 * i + 2];
      } else {
        x[u][0] = gb.x; x[u][1] = gb.y; x[u][2] = gb.z;
      }
    }
    for (int c0 = 0; c0 < sg.w; c0 += 32) {
      const int cnt = min(32, sg.w - c0);
      __syncwarp();
      if (lane < cnt) {
        const double4 p = A.pts[sg.y + c0 + lane];
        if (DL) {  // double-layer source: (y, q n_x), (q n_y, q n_z)
          const double4 nv = A.nrm[sg.y + c0 + lane];
          ssrc[w][lane] = make_double4(p.x, p.y, p.z, p.w * nv.x);
          ssrcw[w][lane] = make_double2(p.w * nv.y, p.w * nv.z);
        } else {
          ssrc[w][lane] = p;
        }
      }
      __syncwarp();
      for (int j = 0; j < cnt; ++j) {
        const double4 sv = ssrc[w][j];
        if (DL) {
          const double2 sw = ssrcw[w][j];
#pragma unroll
          for (int u = 0; u < CHK_TB; ++u)
            acc[u] += dl_term<true>(x[u][0] - sv.x, x[u][1] - sv.y, x[u][2] - sv.z, sv.w, sw.x, sw.y);
        } else {
#pragma unroll
          for (int u = 0; u < CHK_TB; ++u) {
            const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
            const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            acc[u] = fma(sv.w, rinv_or_zero(r2), acc[u]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CHK_TB; ++u) {
      const int i = r0 + lane + 32 * u;
      if (i < n) A.out[(size_t)it.y * A.ldo + i] = acc[u] * kInv4Pi;
    }
  }
}

// ----------------------------------------------------------------------------
// Per-leaf operators (leaf-op mode).  The S2M check potential and the L2T
// equivalent density are linear in the leaf's densities / compressed local
// expansion, so the two stages fold into one k x m (S2M) and m x k (L2T) operator
// per leaf, built once at setup (Step 1) — the same products
// S' (G q) and G (T' l^) with the sums reassociated:
//   S2M:  q^'_B = S_B q_B,   S_B = S' G(c_B + r_B (3-2d) e, x_B)
//   L2T:  p_B  = T_B l^_B,  T_B = r_B G(x_B, c_B + r_B (3-2d) e) T'
// so a matvec streams 2 x kp doubles per point from HBM instead of evaluating
// 2 n kernel values per point on the FP64 pipe.
// k_leafop_build: out(j, a) = scale * sum_i Op[a * sa + i * si] * G(surface_i, x_j),
//   MODE 0 (S2M): point-major rows  out[(pbeg + j - own_lo) * kp + a]
//   MODE 1 (L2T): point-major rows  out[(pbeg + j - own_lo) * kp + a], scale r_B
// ----------------------------------------------------------------------------
constexpr int LO_CH = 32;

template <int MODE, bool DL = false, bool BEM = false>
__global__ void __launch_bounds__(256) k_leafop_build(const int4* __restrict__ items, const double4* __restrict__ pts,
                                                      const double4* __restrict__ geom, const int* __restrict__ pbeg,
                                                      const int* __restrict__ pend, const double* __restrict__ surf,
                                                      int n, int kp, double f, const double* __restrict__ Op, int sa,
                                                      int si, int own_lo, double* __restrict__ out,
                                                      const double4* __restrict__ nrm = nullptr,
                                                      const double4* __restrict__ tri = nullptr,
                                                      const int4* __restrict__ xsegs = nullptr,
                                                      const int64_t* __restrict__ xmoff = nullptr) {
  extern __shared__ double Gs[];  // n x (LO_CH + 1)
  // MODE 0/1: the check surface and the sources are the leaf's; MODE 2 (X operator of row
  // blockIdx.x): the check surface is the target box's, the sources the X source leaf's
  const int b = items[blockIdx.x].x;
  const double4 gb = geom[b];
  const int p0 = MODE == 2 ? xsegs[blockIdx.x].y : pbeg[b];
  const int m = MODE == 2 ? xsegs[blockIdx.x].w : pend[b] - p0;
  const double rad = gb.w * f;
  const double scale = MODE == 1 ? gb.w : 1.0;
  for (int c0 = 0; c0 < m; c0 += LO_CH) {
    const int cm = min(LO_CH, m - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < n * LO_CH; e += blockDim.x) {
      const int i = e / LO_CH, jj = e - i * LO_CH;
      double v = 0.0;
      if (jj < cm) {
        const double4 x = pts[p0 + c0 + jj];
        const double dx = gb.x + rad * surf[3 * i] - x.x;
        const double dy = gb.y + rad * surf[3 * i + 1] - x.y;
        const double dz = gb.z + rad * surf[3 * i + 2] - x.z;
        if (BEM) {  // S2M by element integration (eq s2meval)
          const double cx[3] = {gb.x + rad * surf[3 * i], gb.y + rad * surf[3 * i + 1], gb.z + rad * surf[3 * i + 2]};
          v = bem_integral(load_tri(tri + 3 * (int64_t)(p0 + c0 + jj)), cx, false);
        } else if (DL) {  // S2M of double-layer sources (eq-doubles2m): dG/dn(x_j) at the check point
          const double4 nv = nrm[p0 + c0 + jj];
          v = kInv4Pi * dl_term<false>(dx, dy, dz, nv.x, nv.y, nv.z);
        } else {
          v = kInv4Pi * rinv_nonzero(fma(dz, dz, fma(dy, dy, dx * dx)));  // surface outside the leaf: r > 0
        }
      }
      Gs[i * (LO_CH + 1) + jj] = v;
    }
    __syncthreads();
    // 4 x 4 register blocks (rows a0.., points j0..): 8 loads per 16 FMAs; each entry keeps
    // the sequential sum over i
    constexpr int JB = LO_CH / 4;
    for (int e = threadIdx.x; e < (kp / 4) * JB; e += blockDim.x) {
      const int a0 = (e / JB) * 4, j0 = (e - (e / JB) * JB) * 4;
      if (j0 >= cm) continue;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      const double* op = Op + (size_t)a0 * sa;
      for (int i = 0; i < n; ++i) {
        double o[4], g[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] = op[(size_t)u * sa + (size_t)i * si];
#pragma unroll
        for (int v = 0; v < 4; ++v) g[v] = Gs[i * (LO_CH + 1) + j0 + v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(o[u], g[v], acc[u][v]);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (j0 + v >= cm) break;
        const int j = c0 + j0 + v;
        double* row = MODE == 2 ? out + xmoff[blockIdx.x] + (size_t)j * kp
                                : out + (size_t)(p0 + j - own_lo) * kp;  // point-major rows (S2M, L2T)
#pragma unroll
        for (int u = 0; u < 4; ++u) row[a0 + u] = acc[u][v] * scale;
      }
    }
  }
}

// Leaf-operator GEMVs (HBM-bound: each operator entry is read once per matvec).  Operators
// are point-major rows of kp doubles.  A warp covers a row with R = kp / 4 lanes, each
// loading 32 bytes (2 x 16-byte streaming loads), and RPW = 32 / R rows at a time (RPW = 1
// when R is not a power of two); rows are unrolled 2-deep per lane for bytes in flight.
struct RowMap {
  int R, RPW, rsub, c4;
  bool act;
  __device__ RowMap(int kp, int lane) {
    R = kp >> 2;
    RPW = (R & (R - 1)) == 0 ? 32 / R : 1;
    rsub = lane / R;
    c4 = lane - rsub * R;
    act = rsub < RPW;
  }
};
__device__ __forceinline__ void ld_row4(const double* p, double (&v)[4]) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// acc[e] += sum over this lane's rows j < m of q_j M[j][4 c4 + e] (rows rsub, rsub + RPW, ...;
// the loop is uniform over the warp: the shuffles need every lane)
template <int U>
__device__ __forceinline__ void gemv_rows_t(const double* __restrict__ M, const double4* __restrict__ pts, int p0,
                                            int m, int kp, const RowMap& rm, int lane, double (&acc)[4]) {
  for (int j0 = 0; j0 < m; j0 += 32) {  // densities 32 at a time, fetched by shuffle
    const double qv = j0 + lane < m ? pts[p0 + j0 + lane].w : 0.0;
    const int jn = min(32, m - j0);
    for (int jb = 0; jb < jn; jb += U * rm.RPW) {  // U rows per lane in flight
      double qu[U], v[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = jb + rm.rsub + u * rm.RPW;
        qu[u] = __shfl_sync(0xffffffffu, qv, min(j, 31));
        if (rm.act && j < jn) ld_row4(M + (size_t)(j0 + j) * kp + 4 * rm.c4, v[u]);
        else v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fma(qu[u], v[u][e], acc[e]);
    }
  }
}
// sum acc over the warp's RPW row groups: the totals land on the lanes with rsub = 0
__device__ __forceinline__ void gemv_rows_reduce(const RowMap& rm, double (&acc)[4]) {
  for (int o = rm.R; o < 32 && rm.RPW > 1; o <<= 1)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e] += __shfl_down_sync(0xffffffffu, acc[e], o);
}

// S2M with leaf operators: q^'_B[a] = sum_j q_j S_B[j][a]; one warp per leaf; stored (a
// leaf's multipole is written only here)
template <int U>
__global__ void __launch_bounds__(256) k_s2m_leafop(const int4* __restrict__ items, int nitems,
                                                    const double4* __restrict__ pts, const int* __restrict__ pbeg,
                                                    const int* __restrict__ pend, const double* __restrict__ S, int kp,
                                                    int own_lo, double* __restrict__ qhat) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nitems) return;
  const int b = items[w].x;
  const int p0 = pbeg[b], m = pend[b] - p0;
  const RowMap rm(kp, lane);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  gemv_rows_t<U>(S + (size_t)(p0 - own_lo) * kp, pts, p0, m, kp, rm, lane, acc);
  gemv_rows_reduce(rm, acc);
  if (rm.rsub == 0) {
    double* o = qhat + (size_t)b * kp + 4 * rm.c4;
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = acc[e];
  }
}

// X list with its operators: l^_B[a] += sum over B's X rows, sum_j q_j X_row[j][a]; one warp
// per target box (its rows are contiguous); M2L into l^ finished earlier on the stream and a
// target belongs to one warp: plain read-add-write
template <int U>
__global__ void __launch_bounds__(256) k_x_gemv(const int4* __restrict__ xt, int nxt, const int4* __restrict__ xsegs,
                                                const int64_t* __restrict__ xmoff, const double4* __restrict__ pts,
                                                const double* __restrict__ X, int kp, double* __restrict__ lhat) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nxt) return;
  const int4 t = xt[w];
  const RowMap rm(kp, lane);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r = t.y; r < t.z; ++r) {
    const int4 sg = xsegs[r];
    gemv_rows_t<U>(X + xmoff[r], pts, sg.y, sg.w, kp, rm, lane, acc);
  }
  gemv_rows_reduce(rm, acc);
  if (rm.rsub == 0) {
    double* o = lhat + (size_t)t.x * kp + 4 * rm.c4;
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] += acc[e];
  }
}

// L2T with leaf operators: pot[p0 + j] = sum_a T_B[j][a] l^_B[a] for every owned target
// leaf (leaves above level 2 have no far field: 0); one warp per leaf, the lane's four
// l^ entries in registers, each row's dot product reduced over its R lanes
constexpr int L2T_WARPS = 8;
__global__ void __launch_bounds__(L2T_WARPS * 32) k_l2t_leafop(const int4* __restrict__ items, int nitems,
                                                             const int* __restrict__ level, const int* __restrict__ pbeg,
                                                             const int* __restrict__ pend, const double* __restrict__ Tm,
                                                             const double* __restrict__ lhat, int kp, int own_lo,
                                                             double* __restrict__ pot) {
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * L2T_WARPS + wl;
  if (w >= nitems) return;
  const int b = items[w].x;
  const int p0 = pbeg[b], m = pend[b] - p0;
  if (level[b] < 2) {
    for (int j = lane; j < m; j += 32) pot[p0 + j] = 0.0;
    return;
  }
  const RowMap rm(kp, lane);
  double lh[4] = {0.0, 0.0, 0.0, 0.0};
  if (rm.act) {
#pragma unroll
    for (int e = 0; e < 4; ++e) lh[e] = lhat[(size_t)b * kp + 4 * rm.c4 + e];
  }
  const double* base = Tm + (size_t)(p0 - own_lo) * kp + 4 * rm.c4;
  const int wid = rm.RPW > 1 ? rm.R : 32;  // reduction span: the row's lanes
  for (int j0 = 0; j0 < m; j0 += 4 * rm.RPW) {  // 4 rows per lane in flight
    double d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + rm.rsub + u * rm.RPW;
      double v[4];
      d[u] = 0.0;
      if (rm.act && j < m) {
        ld_row4(base + (size_t)j * kp, v);
        d[u] = fma(v[3], lh[3], fma(v[2], lh[2], fma(v[1], lh[1], v[0] * lh[0])));
      }
    }
    for (int o = wid >> 1; o >= 1; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
    if (rm.act && rm.c4 == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + rm.rsub + u * rm.RPW;
        if (j < m) pot[p0 + j] = d[u];
      }
    }
  }
}

// densities into the sorted points (and, slim plans, a contiguous sorted copy: the weights
// the streamed S2M / X GEMVs bulk-copy)
__global__ void k_set_density(double4* __restrict__ pts, const int32_t* __restrict__ perm, const double* __restrict__ q,
                              int64_t N, double* __restrict__ qs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    const double v = q[perm[i]];
    double4 p = pts[i];  // whole 32-byte points: full-sector stores, no partial writes
    p.w = v;
    pts[i] = p;
    if (qs) qs[i] = v;
  }
}

__global__ void k_set_density_owned(double4* __restrict__ pts, const double* __restrict__ q, int lo, int cnt,
                                    double* __restrict__ qs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) {
    pts[lo + i].w = q[i];
    if (qs) qs[lo + i] = q[i];
  }
}

// potentials to caller order: pot[c] = near[iperm[c]] (+ far[iperm[c]]) — a gather, so the
// stores are coalesced and the random accesses are 8-byte reads (a scatter of 8-byte
// stores would make every 32-byte sector a partial write)
__global__ void k_gather_output(const double* __restrict__ pnear, const double* __restrict__ pfar,
                                const int32_t* __restrict__ iperm, int64_t N, double* __restrict__ pot) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < N) {
    const int32_t i = iperm[c];
    pot[c] = pfar ? pnear[i] + pfar[i] : pnear[i];
  }
}

// owned output in sorted order: pot[i] = near[lo + i] (+ far[lo + i])
__global__ void k_owned_output(const double* __restrict__ pnear, const double* __restrict__ pfar, int lo, int cnt,
                               double* __restrict__ pot) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) pot[i] = pfar ? pnear[lo + i] + pfar[lo + i] : pnear[lo + i];
}

// sorted normals: nrm[i] = (n[perm[i]], 0)
__global__ void k_sort_normals(const double* __restrict__ n, const int32_t* __restrict__ perm, int64_t N,
                               double4* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    const int64_t j = perm[i];
    out[i] = make_double4(n[3 * j], n[3 * j + 1], n[3 * j + 2], 0.0);
  }
}

int sort_normals(Plan& P, const double* d_normals, cudaStream_t st) {
  const int64_t N = P.tree.N;
  KIFMM_CUDA(cudaMalloc(&P.d_nrm, sizeof(double4) * N));
  P.allocations.push_back(P.d_nrm);
  k_sort_normals<<<(int)((N + 255) / 256), 256, 0, st>>>(d_normals, P.tree.d_perm, N, P.d_nrm);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

__global__ void k_combine(double* __restrict__ pnear, const double* __restrict__ pfar, int lo, int cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) pnear[lo + i] += pfar[lo + i];
}

// exchange packing: buf[i][c] = src[idx[i] * ld + c] (c < row), and the inverse store
__global__ void k_pack_rows(const double* __restrict__ src, int ld, const int* __restrict__ idx, int nrows, int row,
                            double* __restrict__ buf) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < (int64_t)nrows * row) {
    int i = (int)(e / row), c = (int)(e - (int64_t)i * row);
    buf[e] = src[(size_t)idx[i] * ld + c];
  }
}
__global__ void k_unpack_rows(double* __restrict__ dst, int ld, const int* __restrict__ idx, int nrows, int row,
                              const double* __restrict__ buf) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < (int64_t)nrows * row) {
    int i = (int)(e / row), c = (int)(e - (int64_t)i * row);
    dst[(size_t)idx[i] * ld + c] = buf[e];
  }
}

// ----------------------------------------------------------------------------
// host-side launch helpers
// ----------------------------------------------------------------------------
int g_num_sms = 148;  // set at setup (cudaDevAttrMultiProcessorCount)
int g_launches = 0;   // kernels launched by the current matvec (fmm_info.gpu_launches)

namespace {

inline int nblk(int64_t n, int t = 256) { return std::max(1, (int)((n + t - 1) / t)); }

int ggs_nt(int M, int K) { return (size_t)(K + 4 + M + 2) * 64 * 8 <= 116 * 1024 ? 64 : 32; }

constexpr int sq_nt(int kp) { return kp <= 64 ? 64 : 32; }
size_t sq_smem(int kp) { return (size_t)sq_nt(kp) * 2 * (kp + 4) * sizeof(double); }

template <int KP>
int launch_sq(const GemmLaunch& g, const double* ops, int mvalid, const double* X, double* Y, bool atomic,
              cudaStream_t st) {
  constexpr int NT = sq_nt(KP);
  const size_t smem = sq_smem(KP);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ggs_sq<KP, NT>, KP * 4, smem);
  const int grid = std::min(g.ntiles, g_num_sms * std::max(1, per_sm));
  k_ggs_sq<KP, NT><<<grid, KP * 4, smem, st>>>(g.d_tiles, g.ntiles, g.d_pairs, ops, mvalid, X, Y, atomic);
  return 0;
}

int launch_ggs(const GemmLaunch& g, const double* ops, int op_stride, int M, int K, int mvalid, const double* X,
               int ldx, double* Y, int ldy, bool atomic, cudaStream_t st) {
  if (g.ntiles == 0) return 0;
  ++g_launches;
  if (M == K && ldx == K && ldy == K && op_stride == K * K && (K == 32 || K == 64 || K == 104)) {
    if (K == 32) launch_sq<32>(g, ops, mvalid, X, Y, atomic, st);
    else if (K == 64) launch_sq<64>(g, ops, mvalid, X, Y, atomic, st);
    else launch_sq<104>(g, ops, mvalid, X, Y, atomic, st);
    KIFMM_CUDA(cudaGetLastError());
    return 0;
  }
  const int NT = ggs_nt(M, K);
  const size_t smem = (size_t)NT * (K + 4 + M + 2) * sizeof(double);
  if (NT == 64)
    k_ggs<64><<<g.ntiles, 256, smem, st>>>(g.d_tiles, g.d_pairs, ops, op_stride, M, K, mvalid, X, ldx, Y, ldy, atomic);
  else
    k_ggs<32><<<g.ntiles, 256, smem, st>>>(g.d_tiles, g.d_pairs, ops, op_stride, M, K, mvalid, X, ldx, Y, ldy, atomic);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

// ----------------------------------------------------------------------------
// k_m2l_lr: the sibling-grouped M2L with the paper's stage-2 low-rank cores
// (eq-lra): C_o ~= U^_o V^_o with rank r_o, so each operator step of a
// tile is two skinny GEMMs instead of one k x k GEMM:
//   phase A  T = V^_o Q        (r_o x NT, inner k)   -> shared memory (column-major)
//   phase B  acc += U^_o T     (k x NT, inner r_o)   -> the per-(target, delta) accumulators
// 4 k r_o instead of 2 k^2 flops per column.  Same tiles, classes, dynamic scheduler,
// metadata ring and cp.async B-panel pipeline as k_m2l_sib16; m16n8k8 FP64 MMA in both
// phases.  Factor tables (zero padded): Vh[o] RP x KP, Uh[o] KP x RP; rank[o] = r_o.
// ----------------------------------------------------------------------------
template <int KP, int NT, int RP, int MINB>
__global__ void __launch_bounds__(Sib16Shape<KP>::NW * 32, MINB) k_m2l_lr(
    const int4* __restrict__ tiles, int ntiles, const int* __restrict__ cols, const int* __restrict__ classes,
    const double* __restrict__ Uh, const double* __restrict__ Vh, const int* __restrict__ rank, int mvalid,
    const double* X, double* Y, int* __restrict__ counter) {
  constexpr int RB = Sib16Shape<KP>::RB;
  constexpr int CS = Sib16Shape<KP>::CS;
  constexpr int NW = Sib16Shape<KP>::NW;
  constexpr int NTH = NW * 32;
  constexpr int SB = KP + 4;
  constexpr int ST = RP + 4;         // T: column-major, stride ST
  constexpr int K2 = KP / 2;
  constexpr int CW = 9;
  constexpr int NCW = NT / CS;
  constexpr int NB = NCW / 8;
  constexpr int NBT = NT / 8;        // n-blocks of a tile (phase A)
  constexpr int KS8 = KP / 8;
  extern __shared__ __align__(16) double sm[];
  double* Ts = sm + 2 * NT * SB;
  __shared__ int s_meta[3][NT * CW];
  __shared__ int s_tile[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp % RB) * 16;
  const int cbase = (warp / RB) * NCW;
  const bool lo_ok = r0 + g < KP, hi_ok = r0 + g + 8 < KP;
  int ti = blockIdx.x;
  if (ti >= ntiles) return;

  auto fetch_meta = [&](int tid, int slot) {
    const int4 tl = tiles[tid];
    for (int e = threadIdx.x; e < NT * CW; e += NTH) {
      const int c = e / CW;
      s_meta[slot][e] = c < tl.z ? cols[(size_t)tl.y * CW + e] : -1;
    }
  };
  auto gather = [&](int slot, int b, int buf) {
    double* Bd = sm + buf * NT * SB;
    for (int p = warp; p < NT; p += NW) {
      const int src = s_meta[slot][p * CW + 1 + b];
      for (int c = lane; c < K2; c += 32) {
        double* dst = Bd + p * SB + 2 * c;
        if (src >= 0) cp_async16(dst, X + (size_t)src * KP + 2 * c);
        else { dst[0] = 0.0; dst[1] = 0.0; }
      }
    }
  };

  int slot = 0;
  fetch_meta(ti, 0);
  if (threadIdx.x == 0) s_tile[1] = gridDim.x + atomicAdd(counter, 1);
  __syncthreads();
  const int* cls = classes + tiles[ti].x * 17;
  gather(0, cls[1], 0);
  cp_async_commit();
  int buf = 0;
  double acc[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

  while (true) {
    const int nv = cls[0];
    const int nslot = slot == 2 ? 0 : slot + 1;
    const int tnext = s_tile[nslot];
    for (int jb = 0; jb < nv; ++jb) {
      const bool last = jb + 1 == nv;
      if (jb == 0 && tnext < ntiles) {
        fetch_meta(tnext, nslot);
        if (threadIdx.x == 0) s_tile[nslot == 2 ? 0 : nslot + 1] = gridDim.x + atomicAdd(counter, 1);
      }
      cp_async_wait0();
      __syncthreads();  // B panel of this step landed; T free; next metadata visible
      if (!last) gather(slot, cls[2 + jb], buf ^ 1);
      else if (tnext < ntiles) gather(nslot, classes[tiles[tnext].x * 17 + 1], buf ^ 1);
      cp_async_commit();
      const int op = cls[9 + jb];
      const int r = rank[op];
      const int ra = (r + 15) >> 4, rk8 = (r + 7) >> 3;
      // ---- phase A: T = V^_o Q   (tiles (row block, n-block) over the warps)
      {
        const double* Vo = Vh + (size_t)op * RP * KP;
        const double* B = sm + buf * NT * SB;
        for (int tile = warp; tile < ra * NBT; tile += NW) {
          const int rb = tile / NBT, nb = tile - rb * NBT;
          const double* Ar = Vo + (size_t)(16 * rb + g) * KP + t;
          const double* Bp = B + (size_t)(nb * 8 + g) * SB + t;
          double c4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
          for (int ks = 0; ks < KS8; ++ks) {
            double a[4];
            a[0] = __ldg(Ar + 8 * ks);
            a[1] = __ldg(Ar + 8 * KP + 8 * ks);
            a[2] = __ldg(Ar + 8 * ks + 4);
            a[3] = __ldg(Ar + 8 * KP + 8 * ks + 4);
            dmma_16x8x8(c4, a, Bp[8 * ks], Bp[8 * ks + 4]);
          }
          // c0,c1: T[16 rb + g][nb 8 + 2t (+1)], c2,c3: row + 8
          double* T0 = Ts + (size_t)(nb * 8 + 2 * t) * ST + 16 * rb + g;
          T0[0] = c4[0];
          T0[ST] = c4[1];
          T0[8] = c4[2];
          T0[ST + 8] = c4[3];
        }
      }
      __syncthreads();  // T complete
      // ---- phase B: acc += U^_o T   (warp: rows r0..r0+16, columns cbase..cbase+NCW)
      {
        const double* Ar = Uh + (size_t)op * KP * RP + (size_t)(r0 + g) * RP + t;
        const double* Bp = Ts + (size_t)(cbase + g) * ST + t;
        for (int ks = 0; ks < rk8; ++ks) {
          double a[4];
          a[0] = lo_ok ? __ldg(Ar + 8 * ks) : 0.0;
          a[1] = hi_ok ? __ldg(Ar + 8 * RP + 8 * ks) : 0.0;
          a[2] = lo_ok ? __ldg(Ar + 8 * ks + 4) : 0.0;
          a[3] = hi_ok ? __ldg(Ar + 8 * RP + 8 * ks + 4) : 0.0;
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            const double* bp = Bp + (size_t)j * 8 * ST + 8 * ks;
            dmma_16x8x8(acc[j], a, bp[0], bp[4]);
          }
        }
      }
      buf ^= 1;
      if (last) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int tg = s_meta[slot][(cbase + j * 8 + 2 * t + c) * CW];
            if (tg >= 0) {
              if (r0 + g < mvalid) atomicAdd(Y + (size_t)tg * KP + r0 + g, acc[j][c]);
              if (r0 + g + 8 < mvalid) atomicAdd(Y + (size_t)tg * KP + r0 + g + 8, acc[j][2 + c]);
            }
          }
          acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        }
      }
    }
    if (tnext >= ntiles) break;
    ti = tnext;
    slot = nslot;
    cls = classes + tiles[ti].x * 17;
  }
}

// ----------------------------------------------------------------------------
// k_m2l_lr2: stage-2 sibling M2L, factors staged in shared memory (kp <= 64).
// All 8 warps step through the same tile (64 columns, warp w owns columns 8w..8w+7).
// Per operator step the B panel AND the factors V^_o (r8 x kp) and U^_o (kp x r8) are
// copied with cp.async one step ahead into double buffers, so every MMA operand comes
// from shared memory.  Phase A computes T^T (8 columns x r8) = Q^T V^_o^T with
// DMMA.8x8x4 (operands: panel, V^); phase B accumulates acc (kp x 8) += U^_o T with the
// m16n8k8 MMA, its B fragments moved out of phase A's accumulators by 4 shuffles per
// k8-step (no shared T, one barrier per step).
// ----------------------------------------------------------------------------
template <int KP, int RP, int NT_ = 128>
struct Lr2Smem {
  static constexpr int NT = NT_;
  static constexpr int SB = KP + 4;  // panel row (column-major panel)
  static constexpr int SV = KP + 4;  // V^ row
  static constexpr int SU = RP + 4;  // U^ row
  static constexpr int PANEL = NT * SB, VS = RP * SV, US = KP * SU;
  static constexpr int BUF = PANEL + VS + US;  // doubles per buffer
};

template <int KP, int RP, int NTC, int CB>
__global__ void __launch_bounds__(NTC * 4 / CB, 1) k_m2l_lr2(
    const int4* __restrict__ tiles, int ntiles, const int* __restrict__ cols, const int* __restrict__ classes,
    const double* __restrict__ Uh, const double* __restrict__ Vh, const int* __restrict__ rank, int mvalid,
    const double* X, double* Y, int* __restrict__ counter) {
  // warp w owns CB column blocks of 8: columns 8 CB w .. 8 CB w + 8 CB - 1
  using S = Lr2Smem<KP, RP, NTC>;
  constexpr int NT = S::NT, NW = NT / (8 * CB), NTH = NW * 32, CW = 9, K2 = KP / 2, KS4 = KP / 4;
  constexpr int RB = KP / 16;          // output row blocks (m16)
  constexpr int NRB = RP / 8;          // max rank blocks of 8
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_meta[3][NT * CW];
  __shared__ int s_tile[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int col0 = 8 * CB * warp;
  int ti = blockIdx.x;
  if (ti >= ntiles) return;

  auto fetch_meta = [&](int tid, int slot) {
    const int4 tl = tiles[tid];
    for (int e = threadIdx.x; e < NT * CW; e += NTH) {
      const int c = e / CW;
      s_meta[slot][e] = c < tl.z ? cols[(size_t)tl.y * CW + e] : -1;
    }
  };
  // stage step (child b of the columns in meta slot, operator op) into buffer buf
  auto stage = [&](int slot, int b, int op, int buf) {
    double* base = sm + (size_t)buf * S::BUF;
    double* Bd = base;
    for (int p = warp; p < NT; p += NW) {
      const int src = s_meta[slot][p * CW + 1 + b];
      for (int c = lane; c < K2; c += 32) {
        double* dst = Bd + p * S::SB + 2 * c;
        if (src >= 0) cp_async16(dst, X + (size_t)src * KP + 2 * c);
        else { dst[0] = 0.0; dst[1] = 0.0; }
      }
    }
    const int r8 = (rank[op] + 7) & ~7;
    double* Vd = base + S::PANEL;
    const double* Vg = Vh + (size_t)op * RP * KP;
    for (int e = threadIdx.x; e < r8 * K2; e += NTH) {
      const int row = e / K2, c = e - row * K2;
      cp_async16(Vd + row * S::SV + 2 * c, Vg + (size_t)row * KP + 2 * c);
    }
    double* Ud = base + S::PANEL + S::VS;
    const double* Ug = Uh + (size_t)op * KP * RP;
    const int r2 = r8 / 2;
    for (int e = threadIdx.x; e < KP * r2; e += NTH) {
      const int row = e / r2, c = e - row * r2;
      cp_async16(Ud + row * S::SU + 2 * c, Ug + (size_t)row * RP + 2 * c);
    }
  };

  int slot = 0;
  fetch_meta(ti, 0);
  if (threadIdx.x == 0) s_tile[1] = gridDim.x + atomicAdd(counter, 1);
  __syncthreads();
  const int* cls = classes + tiles[ti].x * 17;
  stage(0, cls[1], cls[9], 0);
  cp_async_commit();
  int buf = 0;
  double acc[RB][CB][4];
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int c = 0; c < CB; ++c) acc[i][c][0] = acc[i][c][1] = acc[i][c][2] = acc[i][c][3] = 0.0;

  while (true) {
    const int nv = cls[0];
    const int nslot = slot == 2 ? 0 : slot + 1;
    const int tnext = s_tile[nslot];
    for (int jb = 0; jb < nv; ++jb) {
      const bool last = jb + 1 == nv;
      if (jb == 0 && tnext < ntiles) {
        fetch_meta(tnext, nslot);
        if (threadIdx.x == 0) s_tile[nslot == 2 ? 0 : nslot + 1] = gridDim.x + atomicAdd(counter, 1);
      }
      cp_async_wait0();
      __syncthreads();  // this step's panel + factors landed; the other buffer is free
      if (!last) stage(slot, cls[2 + jb], cls[9 + jb + 1], buf ^ 1);
      else if (tnext < ntiles) {
        const int* ncls = classes + tiles[tnext].x * 17;
        stage(nslot, ncls[1], ncls[9], buf ^ 1);
      }
      cp_async_commit();
      const double* base = sm + (size_t)buf * S::BUF;
      const int op = cls[9 + jb];
      const int nrb = (rank[op] + 7) >> 3;
      // phase A: T^T[col][rank 8 rb + 2t (+1)] of column block cb in d[rb][cb]; each V^
      // fragment feeds the CB column blocks
      double d[NRB][CB][2];
      {
        const double* Pa = base + (size_t)(col0 + g) * S::SB + t;   // a = panel[col][4s + t]
        const double* Vb = base + S::PANEL + (size_t)g * S::SV + t;  // b = V^[8 rb + g][4s + t]
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) {
#pragma unroll
          for (int c = 0; c < CB; ++c) d[rb][c][0] = d[rb][c][1] = 0.0;
          if (rb < nrb) {
            const double* vb = Vb + (size_t)8 * rb * S::SV;
#pragma unroll
            for (int s4 = 0; s4 < KS4; ++s4) {
              const double bv = vb[4 * s4];
#pragma unroll
              for (int c = 0; c < CB; ++c) dmma_8x8x4(d[rb][c][0], d[rb][c][1], Pa[(size_t)8 * c * S::SB + 4 * s4], bv);
            }
          }
        }
      }
      // phase B: acc += U^ T; each U^ fragment feeds the CB column blocks
      {
        const double* Ua = base + S::PANEL + S::VS + (size_t)g * S::SU + t;
        const int src0 = 4 * g + (t >> 1), src1 = src0 + 2;
        const bool odd = t & 1;
#pragma unroll
        for (int ks = 0; ks < NRB; ++ks) {
          if (ks < nrb) {
            double b0[CB], b1[CB];
#pragma unroll
            for (int c = 0; c < CB; ++c) {
              const double x0 = __shfl_sync(FULL, d[ks][c][0], src0), x1 = __shfl_sync(FULL, d[ks][c][1], src0);
              const double y0 = __shfl_sync(FULL, d[ks][c][0], src1), y1 = __shfl_sync(FULL, d[ks][c][1], src1);
              b0[c] = odd ? x1 : x0;
              b1[c] = odd ? y1 : y0;
            }
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
              const double* ua = Ua + (size_t)16 * rb * S::SU + 8 * ks;
              double a[4];
              a[0] = ua[0];
              a[1] = ua[8 * S::SU];
              a[2] = ua[4];
              a[3] = ua[8 * S::SU + 4];
#pragma unroll
              for (int c = 0; c < CB; ++c) dmma_16x8x8(acc[rb][c], a, b0[c], b1[c]);
            }
          }
        }
      }
      buf ^= 1;
      if (last) {
#pragma unroll
        for (int cb = 0; cb < CB; ++cb)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int tg = s_meta[slot][(col0 + 8 * cb + 2 * t + c) * CW];
            if (tg >= 0) {
#pragma unroll
              for (int rb = 0; rb < RB; ++rb) {
                const int row = 16 * rb + g;
                if (row < mvalid) atomicAdd(Y + (size_t)tg * KP + row, acc[rb][cb][c]);
                if (row + 8 < mvalid) atomicAdd(Y + (size_t)tg * KP + row + 8, acc[rb][cb][2 + c]);
              }
            }
          }
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int c = 0; c < CB; ++c) acc[i][c][0] = acc[i][c][1] = acc[i][c][2] = acc[i][c][3] = 0.0;
      }
    }
    if (tnext >= ntiles) break;
    ti = tnext;
    slot = nslot;
    cls = classes + tiles[ti].x * 17;
  }
}

constexpr int kLr2Cols = 128;  // columns per stage-2 sibling tile (kp <= 64)

template <int KP, int RP, int CB>
int launch_lr2_cb(const SibLaunch& g, const LowRank& lr, int mvalid, const double* X, double* Y, cudaStream_t st) {
  using S = Lr2Smem<KP, RP, kLr2Cols>;
  constexpr int NTH = kLr2Cols * 4 / CB;
  const size_t smem = (size_t)2 * S::BUF * sizeof(double);
  static bool attr = false;
  if (!attr) {
    KIFMM_CUDA(cudaFuncSetAttribute(k_m2l_lr2<KP, RP, kLr2Cols, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_m2l_lr2<KP, RP, kLr2Cols, CB>, NTH, smem);
  const int grid = std::min(g.ntiles, g_num_sms * std::max(1, per_sm));
  KIFMM_CUDA(cudaMemsetAsync(g.d_counter, 0, sizeof(int), st));
  k_m2l_lr2<KP, RP, kLr2Cols, CB><<<grid, NTH, smem, st>>>(g.d_tiles, g.ntiles, g.d_cols, g.d_classes, lr.d_Uh,
                                                           lr.d_Vh, lr.d_rank, mvalid, X, Y, g.d_counter);
  return 0;
}

template <int KP, int RP>
int launch_lr2(const SibLaunch& g, const LowRank& lr, int mvalid, const double* X, double* Y, cudaStream_t st) {
  return launch_lr2_cb<KP, RP, 1>(g, lr, mvalid, X, Y, st);  // (two column blocks per warp measured slower)
}

template <int KP, int RP>
int launch_lr(const SibLaunch& g, const LowRank& lr, int mvalid, const double* X, double* Y, cudaStream_t st) {
  constexpr int NT = sq_nt(KP);
  constexpr int NTH = Sib16Shape<KP>::NW * 32;
  const size_t smem = ((size_t)NT * 2 * (KP + 4) + (size_t)NT * (RP + 4)) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    KIFMM_CUDA(cudaFuncSetAttribute(k_m2l_lr<KP, NT, RP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_m2l_lr<KP, NT, RP, 2>, NTH, smem);
  const int grid = std::min(g.ntiles, g_num_sms * std::max(1, per_sm));
  KIFMM_CUDA(cudaMemsetAsync(g.d_counter, 0, sizeof(int), st));
  k_m2l_lr<KP, NT, RP, 2><<<grid, NTH, smem, st>>>(g.d_tiles, g.ntiles, g.d_cols, g.d_classes, lr.d_Uh, lr.d_Vh,
                                                   lr.d_rank, mvalid, X, Y, g.d_counter);
  return 0;
}

template <int KP>
int launch_lr_rp(const SibLaunch& g, const LowRank& lr, int mvalid, const double* X, double* Y, cudaStream_t st) {
  switch (lr.rp) {
    case 16: return launch_lr<KP, 16>(g, lr, mvalid, X, Y, st);
    case 32: return launch_lr<KP, 32>(g, lr, mvalid, X, Y, st);
    case 48: return launch_lr<KP, 48>(g, lr, mvalid, X, Y, st);
    case 64: return launch_lr<KP, 64>(g, lr, mvalid, X, Y, st);
    default: return launch_lr<KP, (KP + 15) / 16 * 16>(g, lr, mvalid, X, Y, st);
  }
}

int launch_m2l_lowrank(const SibLaunch& g, const LowRank& lr, int kp, int mvalid, const double* X, double* Y,
                       cudaStream_t st) {
  if (g.ntiles == 0) return 0;
  ++g_launches;
  int rc = 0;
  if (kp == 64 && (lr.rp == 16 || lr.rp == 32)) {
    rc = lr.rp == 16 ? launch_lr2<64, 16>(g, lr, mvalid, X, Y, st) : launch_lr2<64, 32>(g, lr, mvalid, X, Y, st);
    if (rc) return rc;
    KIFMM_CUDA(cudaGetLastError());
    return 0;
  }
  if (kp == 32 && (lr.rp == 16 || lr.rp == 32)) {
    rc = lr.rp == 16 ? launch_lr2<32, 16>(g, lr, mvalid, X, Y, st) : launch_lr2<32, 32>(g, lr, mvalid, X, Y, st);
    if (rc) return rc;
    KIFMM_CUDA(cudaGetLastError());
    return 0;
  }
  if (kp == 32) rc = launch_lr_rp<32>(g, lr, mvalid, X, Y, st);
  else if (kp == 64) rc = launch_lr_rp<64>(g, lr, mvalid, X, Y, st);
  else rc = launch_lr_rp<104>(g, lr, mvalid, X, Y, st);
  if (rc) return rc;
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

template <int KP, int MINB>
int launch_sib16(const SibLaunch& g, const double* C, int mvalid, const double* X, double* Y, int zero_row,
                 cudaStream_t st) {
  constexpr int NT = sq_nt(KP);
  constexpr int NTH = Sib16Shape<KP>::NW * 32;
  const size_t smem = (size_t)NT * 2 * (KP + 4) * sizeof(double);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_m2l_sib16<KP, NT, MINB>, NTH, smem);
  const int grid = std::min(g.ntiles, g_num_sms * std::max(1, per_sm));
  KIFMM_CUDA(cudaMemsetAsync(g.d_counter, 0, sizeof(int), st));
  k_m2l_sib16<KP, NT, MINB><<<grid, NTH, smem, st>>>(g.d_tiles, g.ntiles, g.d_cols, g.d_classes, C, mvalid, X, Y,
                                                     g.d_counter, zero_row);
  return 0;
}

int launch_m2l_sib(const SibLaunch& g, const double* C, int kp, int mvalid, const double* X, double* Y, int zero_row,
                   cudaStream_t st) {
  if (g.ntiles == 0) return 0;
  ++g_launches;
  if (kp == 32) launch_sib16<32, 3>(g, C, mvalid, X, Y, zero_row, st);
  else if (kp == 64) launch_sib16<64, 3>(g, C, mvalid, X, Y, zero_row, st);
  else if (kp == 104) launch_sib16<104, 3>(g, C, mvalid, X, Y, zero_row, st);
  else return -3;  // kp = round_up(k_eff, 8) with k_eff <= 100 at p <= 8: 32, 64 or 104 only
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

int build_leaf_ops(Plan& P, cudaStream_t st) {
  if (P.n_s2m == 0) return 0;
  const Tree& T = P.tree;
  const size_t smem = (size_t)P.n * (LO_CH + 1) * sizeof(double);
  KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double f = 3.0 - 2.0 * P.d;  // UC and DE halfwidth factor
  if (P.leaf_s2m) {
    if (P.bem)
      k_leafop_build<0, false, true><<<P.n_s2m, 256, smem, st>>>(
          P.d_s2m_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf, P.n, P.kp, f, P.d_S, P.np, 1, P.dist.own_lo,
          P.d_s2m_mat, nullptr, P.d_tri);
    else if (P.d_nrm)
      k_leafop_build<0, true><<<P.n_s2m, 256, smem, st>>>(P.d_s2m_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf,
                                                          P.n, P.kp, f, P.d_S, P.np, 1, P.dist.own_lo, P.d_s2m_mat,
                                                          P.d_nrm);
    else
      k_leafop_build<0><<<P.n_s2m, 256, smem, st>>>(P.d_s2m_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf, P.n,
                                                    P.kp, f, P.d_S, P.np, 1, P.dist.own_lo, P.d_s2m_mat);
    KIFMM_CUDA(cudaGetLastError());
  }
  if (P.leaf_l2t) {
    k_leafop_build<1><<<P.n_s2m, 256, smem, st>>>(P.d_s2m_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf, P.n,
                                                  P.kp, f, P.d_T, 1, P.kp, P.dist.own_lo, P.d_l2t_mat);
    KIFMM_CUDA(cudaGetLastError());
  }
  return 0;
}

// X operators: row r = (target B, source leaf A): U^T G_src(c_B + r_B (1 + d) e, sources of A)
int build_x_ops(Plan& P, cudaStream_t st) {
  if (P.n_xnd == 0) return 0;
  const Tree& T = P.tree;
  const size_t smem = (size_t)P.n * (LO_CH + 1) * sizeof(double);
  const double f = 1.0 + P.d;  // DC halfwidth factor
  if (P.bem) {
    KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_leafop_build<2, false, true><<<P.n_xnd, 256, smem, st>>>(P.d_x_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend,
                                                               P.d_surf, P.n, P.kp, f, P.d_Ut, P.np, 1, 0, P.d_x_mat,
                                                               nullptr, P.d_tri, P.d_x_seg, P.d_x_moff);
  } else if (P.d_nrm) {
    KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_leafop_build<2, true><<<P.n_xnd, 256, smem, st>>>(P.d_x_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf,
                                                        P.n, P.kp, f, P.d_Ut, P.np, 1, 0, P.d_x_mat, P.d_nrm, nullptr,
                                                        P.d_x_seg, P.d_x_moff);
  } else {
    KIFMM_CUDA(cudaFuncSetAttribute(k_leafop_build<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_leafop_build<2><<<P.n_xnd, 256, smem, st>>>(P.d_x_items, T.d_pts, T.d_geom, T.d_pbeg, T.d_pend, P.d_surf, P.n,
                                                  P.kp, f, P.d_Ut, P.np, 1, 0, P.d_x_mat, nullptr, nullptr, P.d_x_seg,
                                                  P.d_x_moff);
  }
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

int sib_tile_width(int kp, bool lowrank) {
  return lowrank && kp <= 64 ? kLr2Cols : sq_nt(kp);
}

int ggs_tile_width(int M, int K) {
  if (M == K && (K == 32 || K == 64 || K == 104)) return sq_nt(K);
  return ggs_nt(M, K);
}

int kernels_init() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs_sq<32, sq_nt(32)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs_sq<64, sq_nt(64)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs_sq<104, sq_nt(104)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_m2l_sib16<32, sq_nt(32), 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_m2l_sib16<64, sq_nt(64), 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_m2l_sib16<104, sq_nt(104), 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  return 0;
}


// Evaluation work lists live in the plan; see build_schedules (schedule.cpp).
// k_eval with 128 threads per target leaf (measured best of 128 / 256 threads and
// a warp-per-leaf variant)
static void launch_eval(const Plan& P, EvalArgs a, int chk_self, cudaStream_t st, bool dl = false, int nitems = -1) {
  if (nitems < 0) {
    a.items = P.d_tleaf_items;
    nitems = P.n_tleaf;
  }
  if (nitems == 0) return;
  if (dl) k_eval<128, 256, true><<<nitems, 128, 0, st>>>(a, chk_self);
  else k_eval<128, 256><<<nitems, 128, 0, st>>>(a, chk_self);
}

static int launch_sym(const Plan& P, cudaStream_t st);

// near field into pot_near: one-sided segments (own leaf first, U, direct W/X) + symmetric pairs
static int launch_near(const Plan& P, const EvalArgs& ea, cudaStream_t st) {
  if (P.nr_on) {  // mutual leaf pairs (near.cu): every result added with RED
    KIFMM_CUDA(cudaMemsetAsync(P.d_pot_near, 0, sizeof(double) * P.tree.N, st));
    return near_launch(P, P.d_pot_near, st);
  }
  if (P.n_tleaf > 0) {
    EvalArgs a = ea;
    a.seg_off = P.d_near_off; a.segs = P.d_near_seg; a.out = P.d_pot_near;
    launch_eval(P, a, 1, st, P.d_nrm != nullptr);  // the near-field sources are input points
    ++g_launches;
    KIFMM_CUDA(cudaGetLastError());
  }
  return launch_sym(P, st);
}

static int launch_sym(const Plan& P, cudaStream_t st) {
  if (P.n_sym == 0) return 0;
  ++g_launches;
  const int grid = (P.n_sym + SYM_WARPS - 1) / SYM_WARPS;
  k_p2p_sym<5><<<grid, SYM_WARPS * 32, 0, st>>>(P.d_sym, P.n_sym, P.tree.d_pts, P.tree.d_pbeg, P.tree.d_pend, P.d_pot_near);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

// check points per lane: one round of 32*TB when n <= 160, else rounds of 32*ceil(n/64)
void launch_chk(const EvalArgs& a, int nitems, int n, cudaStream_t st) {
  const int tb = n <= 160 ? (n + 31) / 32 : (n + 63) / 64;
  const int grid = (nitems + CHK_WARPS - 1) / CHK_WARPS, thr = CHK_WARPS * 32;
  if (a.tri) {  // BEM elements: element integrals
    k_chk_bem<2><<<grid, thr, 0, st>>>(a, nitems);
    return;
  }
  if (a.nrm) {  // double-layer sources
    switch (std::min(5, std::max(1, tb))) {
      case 1: k_chk<1, true><<<grid, thr, 0, st>>>(a, nitems); break;
      case 2: k_chk<2, true><<<grid, thr, 0, st>>>(a, nitems); break;
      case 3: k_chk<3, true><<<grid, thr, 0, st>>>(a, nitems); break;
      case 4: k_chk<4, true><<<grid, thr, 0, st>>>(a, nitems); break;
      default: k_chk<5, true><<<grid, thr, 0, st>>>(a, nitems); break;
    }
    return;
  }
  switch (std::min(5, std::max(1, tb))) {
    case 1: k_chk<1><<<grid, thr, 0, st>>>(a, nitems); break;
    case 2: k_chk<2><<<grid, thr, 0, st>>>(a, nitems); break;
    case 3: k_chk<3><<<grid, thr, 0, st>>>(a, nitems); break;
    case 4: k_chk<4><<<grid, thr, 0, st>>>(a, nitems); break;
    default: k_chk<5><<<grid, thr, 0, st>>>(a, nitems); break;
  }
}

namespace {
int pack(const double* src, int ld, const int* idx, int nrows, int row, double* buf, cudaStream_t st) {
  if (nrows == 0) return 0;
  ++g_launches;
  const int64_t e = (int64_t)nrows * row;
  k_pack_rows<<<(int)((e + 255) / 256), 256, 0, st>>>(src, ld, idx, nrows, row, buf);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}
int unpack(double* dst, int ld, const int* idx, int nrows, int row, const double* buf, cudaStream_t st) {
  if (nrows == 0) return 0;
  ++g_launches;
  const int64_t e = (int64_t)nrows * row;
  k_unpack_rows<<<(int)((e + 255) / 256), 256, 0, st>>>(dst, ld, idx, nrows, row, buf);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}
}  // namespace

// Diagnostics (KIFMM_TRACE=1, stderr only): events on both streams around the launches of
// one matvec, printed relative to its start after the matvec completes — the only view of
// the two-stream timeline without a tracing tool in this image.
namespace {
struct Trace {
  Plan* P = nullptr;
  int n = 0;
  const char* names[32];
  void begin(Plan& p) {
    static const bool on = std::getenv("KIFMM_TRACE") != nullptr;
    P = nullptr;
    n = 0;
    if (!on) return;
    if (p.ev_trace.empty()) {
      p.ev_trace.resize(32);
      for (auto& e : p.ev_trace) cudaEventCreate(&e);
    }
    P = &p;
  }
  void mark(const char* name, cudaStream_t s) {
    if (!P || n >= 32) return;
    names[n] = name;
    cudaEventRecord(P->ev_trace[n++], s);
  }
  void dump() {
    if (!P || n == 0) return;
    cudaDeviceSynchronize();
    std::fprintf(stderr, "kifmm trace:");
    for (int i = 0; i < n; ++i) {
      float ms = -1;
      cudaError_t e = cudaEventElapsedTime(&ms, P->ev_trace[0], P->ev_trace[i]);
      std::fprintf(stderr, " %s=%.3f%s", names[i], ms, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    std::fprintf(stderr, "\n");
    (void)cudaGetLastError();
    P = nullptr;
  }
};
Trace g_trace;
}  // namespace

int launch_m2l(const Plan& P, const SibLaunch& g, cudaStream_t st);

// Profile events (fmm_info.phase_ms): 0 density (+ghost densities) | 1 S2M | 2 M2M |
// 3 exchange (straddlers + ghost q^') | 4 M2L | 5 X | 6 L2L | 7 evaluation (L2T, W, P2P) | 8 output
int matvec_stage(Plan& P, int stage, const double* d_density, double* d_pot, bool owned, cudaStream_t st) {
  Tree& T = P.tree;
  const int64_t N = T.N;
  const int kp = P.kp, np = P.np, k = P.k, n = P.n;
  const DistPlan& Dp = P.dist;
  auto mark = [&](int i) { if (P.profile) cudaEventRecord(P.ev_phase[i], st); };
  // profiled plans also time the near-field launches alone (fmm_info.near_ms)
  auto mark_near = [&](int i) {
    if (P.profile && P.ev_near[i]) {
      cudaEventRecord(P.ev_near[i], st);
      P.near_timed = true;
    }
  };
  double* pts_w = reinterpret_cast<double*>(T.d_pts) + 3;  // the q column of the (x, y, z, q) points
  EvalArgs ea{};
  ea.pts = T.d_pts; ea.geom = T.d_geom; ea.pbeg = T.d_pbeg; ea.pend = T.d_pend;
  ea.surf = P.d_surf; ea.n = n; ea.f_in = 1.0 + P.d; ea.f_out = 3.0 - 2.0 * P.d; ea.ldq = np;
  ea.nrm = P.d_nrm;  // S2M / X check potentials and the near field use it (double layer)
  ea.tri = P.d_tri;  // BEM: X check potentials by element integration
  // NVTX range per stage (tracing; free without an attached tool)
  static const char* const kStageName[kNumStages] = {"fmm/density", "fmm/upward", "fmm/ghosts", "fmm/downward",
                                                     "fmm/output"};
  struct NvtxRange {
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
  } nvtx_range(stage >= 0 && stage < kNumStages ? kStageName[stage] : "fmm/stage");
  // per-plan launch count across stages (plans of a loopback group interleave)
  struct LaunchCount {
    Plan& P;
    LaunchCount(Plan& p, int stage) : P(p) { g_launches = stage == 0 ? 0 : P.launch_acc; }
    ~LaunchCount() { P.launch_acc = g_launches; P.launches = g_launches; }
  } counter(P, stage);
  switch (stage) {
    case 0: {  // densities into the Morton-ordered points
      mark(0);
      ++g_launches;
      if (owned) {
        const int cnt = Dp.own_hi - Dp.own_lo;
        if (cnt > 0)
          k_set_density_owned<<<nblk(cnt), 256, 0, st>>>(T.d_pts, d_density, Dp.own_lo, cnt,
                                                         P.stream_ok ? P.d_q_sorted : nullptr);
        if (pack(pts_w, 4, P.xd.d_send_idx, P.xd.nsend, 1, P.xd.d_send, st)) return -3;
      } else {
        k_set_density<<<nblk(N), 256, 0, st>>>(T.d_pts, T.d_perm, d_density, N, P.stream_ok ? P.d_q_sorted : nullptr);
      }
      KIFMM_CUDA(cudaGetLastError());
      return 0;
    }
    case 1: {  // upward pass (partial multipoles of straddling boxes)
      if (owned && unpack(pts_w, 4, P.xd.d_recv_idx, P.xd.nrecv, 1, P.xd.d_recv, st)) return -3;
      if (P.overlap == 1) {  // near field on its own stream, concurrent with the far field
        KIFMM_CUDA(cudaEventRecord(P.ev_fork, st));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_near, P.ev_fork, 0));
        if (launch_near(P, ea, P.stream_near)) return -3;
        KIFMM_CUDA(cudaEventRecord(P.ev_join, P.stream_near));
      }
      // near field on the near stream from here, beside the far field.  NCCL-connected
      // plans fork after the ghost exchange instead (stage 3): k_near's persistent CTAs
      // hold every SM slot, and the NCCL kernels enqueued behind the M2M would wait for
      // them, serialising the far field behind the whole near field
      if (P.overlap == 3 && !(P.nccl_comm && !P.bem)) {
        KIFMM_CUDA(cudaEventRecord(P.ev_fork, st));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_near, P.ev_fork, 0));
        if (P.bem) {  // BEM: the element-integral block SpMV (HBM-bound) beside the M2L (tensor)
          ++g_launches;
          if (bem_near_matvec(P, P.stream_near)) return -3;
          KIFMM_CUDA(cudaEventRecord(P.ev_join, P.stream_near));
        } else {
          KIFMM_CUDA(cudaMemsetAsync(P.d_pot_near, 0, sizeof(double) * N, P.stream_near));
          if (near_launch(P, P.d_pot_near, P.stream_near, 1, P.nr_spare)) return -3;
        }
      }
      KIFMM_CUDA(cudaMemsetAsync(P.d_qhat, 0, sizeof(double) * (size_t)T.nboxes * kp, st));
      KIFMM_CUDA(cudaMemsetAsync(P.d_lhat, 0, sizeof(double) * (size_t)T.nboxes * kp, st));
      mark(1);
      g_trace.mark("s2m_begin", st);
      if (P.stream_ok) {  // S2M streamed by bulk copies (stream.cu), stored into q^'
        if (stream_s2m(P, st)) return -3;
      } else if (P.leaf_s2m) {  // S2M as one GEMV per leaf with its precomputed operator
        if (P.n_s2m > 0) {
          ++g_launches;
          // 4 rows per lane in flight when a row is a power-of-two number of 32-byte lane
          // loads (kp <= 64, several rows per warp), else 2 (registers: occupancy)
          if (kp <= 64 && ((kp / 4) & (kp / 4 - 1)) == 0)
            k_s2m_leafop<4><<<(P.n_s2m + 7) / 8, 256, 0, st>>>(P.d_s2m_items, P.n_s2m, T.d_pts, T.d_pbeg, T.d_pend,
                                                               P.d_s2m_mat, kp, Dp.own_lo, P.d_qhat);
          else
            k_s2m_leafop<2><<<(P.n_s2m + 7) / 8, 256, 0, st>>>(P.d_s2m_items, P.n_s2m, T.d_pts, T.d_pbeg, T.d_pend,
                                                               P.d_s2m_mat, kp, Dp.own_lo, P.d_qhat);
          KIFMM_CUDA(cudaGetLastError());
        }
      } else if (P.n_s2m > 0) {  // S2M stage 1: check potentials of leaves at level >= 2
        EvalArgs a = ea;
        a.items = P.d_s2m_items; a.seg_off = P.d_s2m_off; a.segs = P.d_s2m_seg; a.tgt_f = 3.0 - 2.0 * P.d;
        a.out = P.d_chk_s2m; a.ldo = np;
        launch_chk(a, P.n_s2m, n, st);
        ++g_launches;
        KIFMM_CUDA(cudaGetLastError());
      }
      // S2M stage 2: q^'_B = S' c  (store)
      if (!P.leaf_s2m && launch_ggs(P.g_s2m, P.d_S, 0, kp, np, k, P.d_chk_s2m, np, P.d_qhat, kp, false, st)) return -3;
      mark(2);
      // M2M, finest child level first: q^'_P += 1/2 M~_o q^'_c
      for (auto& g : P.g_m2m)
        if (launch_ggs(g, P.d_M, kp * kp, kp, kp, k, P.d_qhat, kp, P.d_qhat, kp, true, st)) return -3;
      mark(3);
      return pack(P.d_qhat, kp, P.d_straddle, P.n_straddle, kp, P.d_straddle_buf, st);
    }
    case 2:  // complete straddlers, then the ghost multipoles other ranks need
      if (unpack(P.d_qhat, kp, P.d_straddle, P.n_straddle, kp, P.d_straddle_buf, st)) return -3;
      return pack(P.d_qhat, kp, P.xq.d_send_idx, P.xq.nsend, kp, P.xq.d_send, st);
    case 3: {  // interactions and downward pass for the owned targets
      if (unpack(P.d_qhat, kp, P.xq.d_recv_idx, P.xq.nrecv, kp, P.xq.d_recv, st)) return -3;
      if (P.overlap == 3 && P.nccl_comm && !P.bem) {  // the near stream's fork, after the exchanges (see stage 1)
        KIFMM_CUDA(cudaEventRecord(P.ev_fork, st));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_near, P.ev_fork, 0));
        KIFMM_CUDA(cudaMemsetAsync(P.d_pot_near, 0, sizeof(double) * N, P.stream_near));
        if (near_launch(P, P.d_pot_near, P.stream_near, 1, P.nr_spare)) return -3;
      }
      g_trace.mark("m2m_end", st);
      mark(4);
      // M2L, all levels in one launch per kernel: l^_B += C_delta q^'_A
      //   dense sibling groups (one RED per (target, delta)), then the sparse remainder by offset
      // overlap mode 2: M2L on the plan's high-priority stream (its persistent CTAs are
      // dispatched first), the near field on the low-priority near stream filling the rest
      cudaStream_t sm2l = st;
      if (P.overlap == 2) {
        KIFMM_CUDA(cudaEventRecord(P.ev_fork, st));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_m2l, P.ev_fork, 0));
        sm2l = P.stream_m2l;
      }
      // the local-source tiles (unless matvec_device ran them beside the exchanges), then the
      // tiles with ghost / straddling sources
      if (!P.m2l_local_done && launch_m2l(P, P.g_m2l_sib, sm2l)) return -3;
      P.m2l_local_done = false;
      if (launch_m2l(P, P.g_m2l_sib_ghost, sm2l)) return -3;
      if (P.overlap == 2) {
        KIFMM_CUDA(cudaEventRecord(P.ev_m2l, P.stream_m2l));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_near, P.ev_fork, 0));
        if (launch_near(P, ea, P.stream_near)) return -3;
        KIFMM_CUDA(cudaEventRecord(P.ev_join, P.stream_near));
        KIFMM_CUDA(cudaStreamWaitEvent(st, P.ev_m2l, 0));
      }
      if (P.overlap == 3 && !P.bem) {  // k_near part 2 after the M2L, beside X / L2L / L2T / the far pass
        KIFMM_CUDA(cudaEventRecord(P.ev_m2l, st));
        KIFMM_CUDA(cudaStreamWaitEvent(P.stream_near, P.ev_m2l, 0));
        if (near_launch(P, P.d_pot_near, P.stream_near, 2, P.nr_spare)) return -3;
        KIFMM_CUDA(cudaEventRecord(P.ev_join, P.stream_near));
      }
      g_trace.mark("m2l_end", st);
      mark(5);
      // X list (S2L): check potentials on DC of the target, then U^T projection (atomic)
      g_trace.mark("x_begin", st);
      if (P.stream_ok) {  // streamed by bulk copies, added into l^ with RED
        if (stream_x(P, st)) return -3;
      } else if (P.leaf_x && P.n_xt > 0) {
        ++g_launches;
        if (kp <= 64 && ((kp / 4) & (kp / 4 - 1)) == 0)
          k_x_gemv<4><<<(P.n_xt + 7) / 8, 256, 0, st>>>(P.d_xt_items, P.n_xt, P.d_x_seg, P.d_x_moff, T.d_pts, P.d_x_mat,
                                                        kp, P.d_lhat);
        else
          k_x_gemv<2><<<(P.n_xt + 7) / 8, 256, 0, st>>>(P.d_xt_items, P.n_xt, P.d_x_seg, P.d_x_moff, T.d_pts, P.d_x_mat, kp,
                                                   P.d_lhat);
        KIFMM_CUDA(cudaGetLastError());
      } else if (P.n_xnd > 0) {
        EvalArgs a = ea;
        a.items = P.d_x_items; a.seg_off = P.d_x_off; a.segs = P.d_x_seg; a.tgt_f = 1.0 + P.d;
        a.out = P.d_chk_x; a.ldo = np;
        launch_chk(a, P.n_xnd, n, st);
        ++g_launches;
        KIFMM_CUDA(cudaGetLastError());
        if (launch_ggs(P.g_x, P.d_Ut, 0, kp, np, k, P.d_chk_x, np, P.d_lhat, kp, true, st)) return -3;
      }
      mark(6);
      // L2L, coarsest parent level first: l^_c += L~_o l^_P
      for (auto& g : P.g_l2l)
        if (launch_ggs(g, P.d_L, kp * kp, kp, kp, k, P.d_lhat, kp, P.d_lhat, kp, true, st)) return -3;
      mark(7);
      // near field as its own pass (split_phases: phase exports; double layer: its own
      // kernel) unless it runs on the overlapped near stream
      const bool sep = P.split_phases || P.overlap || P.d_nrm || P.bem;
      g_trace.mark("l2l_end", st);
      if (P.bem) {  // BEM near field: the precomputed element-integral blocks
        if (P.overlap != 3) {  // (overlapped: launched on the near stream at the fork)
          ++g_launches;
          if (bem_near_matvec(P, st)) return -3;
        }
      } else if (sep && !P.overlap) {
        mark_near(0);
        if (launch_near(P, ea, st)) return -3;
        mark_near(1);
      }
      // L2T stage 1: q_d = r_l T' l^_B ; W stage 1: q_u = r_A U q^'_A  (store)
      if (launch_ggs(P.g_l2t, P.d_T, 0, np, kp, n, P.d_lhat, kp, P.d_eqd_l2t, np, false, st)) return -3;
      if (launch_ggs(P.g_w, P.d_Ue, 0, np, kp, n, P.d_qhat, kp, P.d_eqd_w, np, false, st)) return -3;
      // far field of the targets into pot_far when the near field is separate (split or
      // overlapped on the near stream), else everything fused into pot_near
      double* far_out = sep ? P.d_pot_far : P.d_pot_near;
      // leaf-op mode: L2T as one GEMV per leaf, stored; the evaluation pass below adds to it
      if (P.leaf_l2t && P.n_tleaf > 0) {
        ++g_launches;
        k_l2t_leafop<<<(P.n_tleaf + L2T_WARPS - 1) / L2T_WARPS, L2T_WARPS * 32, 0, st>>>(
            P.d_tleaf_items, P.n_tleaf, T.d_level, T.d_pbeg, T.d_pend, P.d_l2t_mat, P.d_lhat, kp, Dp.own_lo, far_out);
        KIFMM_CUDA(cudaGetLastError());
      }
      // mutual near field fused into pot_near: after the stored L2T (else on zeros), before
      // the far segments (k_eval below adds to the result)
      const bool nr_fused = P.nr_on && !sep;
      if (nr_fused) {
        if (!P.leaf_l2t) KIFMM_CUDA(cudaMemsetAsync(P.d_pot_near, 0, sizeof(double) * N, st));
        mark_near(0);
        if (near_launch(P, P.d_pot_near, st)) return -3;
        mark_near(1);
      }
      // L2T + W stage 2 (and, fused, the near field): potentials at the targets of each leaf
      if (P.n_tleaf > 0 && !(sep && P.leaf_l2t && P.n_far_seg == 0) && !(nr_fused && P.n_far_seg == 0)) {
        EvalArgs a = ea;
        a.items = P.d_tleaf_items;
        a.accumulate = P.leaf_l2t || nr_fused ? 1 : 0;
        a.nrm = nullptr;  // far sources are equivalent surfaces: single layer
        a.tri = nullptr;
        if (sep || nr_fused) { a.seg_off = P.d_far_off; a.segs = P.d_far_seg; }
        else { a.seg_off = P.d_all_off; a.segs = P.d_all_seg; }
        a.out = far_out;
        a.eqd1 = P.d_eqd_l2t; a.eqd2 = P.d_eqd_w;
        int nitems = -1;  // adding to stored results: only the leaves that have far segments
        if ((sep || nr_fused) && a.accumulate) {
          a.items = P.d_fitems; a.seg_off = P.d_fitem_off; a.segs = P.d_fitem_seg;
          nitems = P.n_fitems;
        }
        launch_eval(P, a, sep || nr_fused ? 0 : 1, st, false, nitems);
        ++g_launches;
        KIFMM_CUDA(cudaGetLastError());
      }
      if (!sep && launch_sym(P, st)) return -3;
      if (sep && !P.split_phases) {  // [join the near stream,] then pot_near += pot_far on the owned points
        if (P.overlap) KIFMM_CUDA(cudaStreamWaitEvent(st, P.ev_join, 0));
        const int cnt = Dp.own_hi - Dp.own_lo;
        if (cnt > 0) {
          ++g_launches;
          k_combine<<<nblk(cnt), 256, 0, st>>>(P.d_pot_near, P.d_pot_far, Dp.own_lo, cnt);
          KIFMM_CUDA(cudaGetLastError());
        }
      }
      g_trace.mark("joined", st);
      mark(8);
      if (owned) {
        const int cnt = Dp.own_hi - Dp.own_lo;
        ++g_launches;
        if (cnt > 0)
          k_owned_output<<<nblk(cnt), 256, 0, st>>>(P.d_pot_near, P.split_phases ? P.d_pot_far : nullptr, Dp.own_lo,
                                                     cnt, d_pot);
        KIFMM_CUDA(cudaGetLastError());
        mark(9);
        if (P.profile) P.profiled = true;
      }
      return 0;
    }
    case 4: {  // caller order (replicated mode; the owned ranges were allgathered into pot_near)
      if (owned) return 0;
      k_gather_output<<<nblk(N), 256, 0, st>>>(P.d_pot_near, P.split_phases ? P.d_pot_far : nullptr, T.d_iperm, N, d_pot);
      ++g_launches;
      KIFMM_CUDA(cudaGetLastError());
      mark(9);
      if (P.profile) P.profiled = true;
      return 0;
    }
  }
  return -1;
}

// M2L, all levels in one launch per kernel (the dense cores or the stage-2 factors)
int launch_m2l(const Plan& P, const SibLaunch& g, cudaStream_t st) {
  if (P.lr.on) return launch_m2l_lowrank(g, P.lr, P.kp, P.k, P.d_qhat, P.d_lhat, st);
  return launch_m2l_sib(g, P.d_C, P.kp, P.k, P.d_qhat, P.d_lhat, P.tree.nboxes, st);
}

// One matvec of a single-GPU plan, or of one rank of an NCCL-connected plan.  NCCL plans
// (not profiled) overlap the exchanges with compute: after the upward pass the straddler
// allreduce, the ghost-q^' pack and the exchange run on the plan's comm stream while the
// main stream runs the M2L tiles whose sources are complete locally (they touch neither
// the straddling rows the allreduce rewrites nor the ghost rows still in flight); the
// main stream then waits for the exchange and continues with the ghost-source tiles.
int matvec_device(Plan& P, const double* d_density, double* d_pot, bool owned, cudaStream_t st) {
  const bool dist = P.nccl_comm != nullptr;
  g_trace.begin(P);
  g_trace.mark("start", st);
  struct Dump {
    ~Dump() { g_trace.dump(); }
  } dump_at_exit;
  if (matvec_stage(P, 0, d_density, d_pot, owned, st)) return -3;
  if (dist && owned && nccl_exchange(P, P.xd, st)) return -5;
  if (matvec_stage(P, 1, d_density, d_pot, owned, st)) return -3;
  if (dist && P.stream_comm && !P.profile) {
    cudaStream_t sc = P.stream_comm;
    KIFMM_CUDA(cudaEventRecord(P.ev_up, st));
    KIFMM_CUDA(cudaStreamWaitEvent(sc, P.ev_up, 0));
    if (nccl_allreduce_sum(P, P.d_straddle_buf, (size_t)P.n_straddle * P.kp, sc)) return -5;
    if (matvec_stage(P, 2, d_density, d_pot, owned, sc)) return -3;
    if (nccl_exchange(P, P.xq, sc)) return -5;
    KIFMM_CUDA(cudaEventRecord(P.ev_comm, sc));
    g_trace.mark("m2l_local_begin", st);
    if (launch_m2l(P, P.g_m2l_sib, st)) return -3;
    g_trace.mark("m2l_local_end", st);
    P.m2l_local_done = true;
    KIFMM_CUDA(cudaStreamWaitEvent(st, P.ev_comm, 0));
  } else {
    if (dist && nccl_allreduce_sum(P, P.d_straddle_buf, (size_t)P.n_straddle * P.kp, st)) return -5;
    if (matvec_stage(P, 2, d_density, d_pot, owned, st)) return -3;
    if (dist && nccl_exchange(P, P.xq, st)) return -5;
  }
  if (matvec_stage(P, 3, d_density, d_pot, owned, st)) return -3;
  if (dist && !owned && nccl_allgather_ranges(P, P.d_pot_near, st)) return -5;
  return matvec_stage(P, 4, d_density, d_pot, owned, st);
}

}  // namespace kifmm
