// Near field (P2P) with mutual leaf pairs: k_near.
//
// G(x, y) = 1 / (4 pi |x - y|) is symmetric, so the unordered pair of leaves
// {B, A} of a U pair (or of a direct W pair whose mirror is the direct X pair) is
// evaluated ONCE for both directions: p_i += sum_j G_ij q_j (i in B) and
// p_j += sum_i G_ij q_i (j in A).  The host assigns each such pair to one of its two
// leaves (schedule.cpp, mut_target) as a "mutual" source segment; the leaf's own
// points (r = 0 possible: checked) and the remaining one-sided point segments (pairs
// with a leaf of another rank) complete its source list.  About 13 FP64 instructions
// per unordered pair instead of 2 x 12 one-sided.
//
// Work unit: a pass of up to TB x MQ targets of one leaf against at most 4 chunks of its
// source list; a chunk is <= near_ch(TB MQ) source slots of a host-built point-index
// table (no per-source search, no segment scan on the device).  Thread (ti, gi) holds
// targets ti + MQ u (u < TB) and sweeps sources gi, gi + G, ... of each chunk (G = NT / MQ
// slices).  MQ is a power of two, so a slice's MQ lanes are adjacent lanes of one warp:
// for mutual sources each lane forms s_j = sum_u q_u G(x_u, y_j) and every SB steps a
// butterfly reduce-scatter over the slice leaves sum_i q_i G(x_i, y_j) on one lane, which
// adds it to p_j with one RED.  Target sums are reduced over the G slices in shared memory
// at the end of the unit and added with RED (other CTAs deposit mutual contributions into
// the same potentials).  Double-layer sources take the same path with their normals
// (k_near<TB, MQ, true>).
//
// Persistent CTAs, one launch per pass shape; units are taken from a global counter
// (longest first), two ahead of use.  Software-pipelined: while chunk c is evaluated,
// chunk c + 1 — possibly the first chunk of the CTA's next unit, with that unit's targets —
// is already in flight into the other buffer (cp.async from slot indices loaded one chunk
// earlier), so no load of the critical path waits on metadata.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fmm_internal.h"

namespace kifmm {

namespace {

__device__ __forceinline__ void nr_cp16(void* smem_dst, const void* gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void nr_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void nr_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

constexpr int NR_NT = 128;

struct NearArgs {
  const int4* items;    // work units: (first target point, targets <= TB MQ, chunk begin, chunk end)
  int nitems;
  const int4* chunks;   // (first source slot, n | nchk << 10 | ml << 20, mh, 0)
  const int* src;       // per chunk: the point index of each source slot
  const double4* pts;   // sorted (x, y, z, q)
  double* out;          // potentials (sorted order), added to with RED
  const double4* nrm;   // double layer: sorted source normals (else null)
  int* counter;         // items handed out beyond the first gridDim.x (zeroed per launch)
};

// one-sided sum over sources [j0, j1) step G into acc; CHECK: r = 0 contributes 0 (Q1)
template <int TB, bool CHECK>
__device__ __forceinline__ void nr_onesided(const double4* sbuf, int j0, int j1, int G, const double (&x)[TB][3],
                                            double (&acc)[TB]) {
#pragma unroll 2
  for (int j = j0; j < j1; j += G) {
    const double4 sv = sbuf[j];
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      acc[u] = fma(sv.w, CHECK ? rinv_or_zero(r2) : rinv_nonzero(r2), acc[u]);
    }
  }
}

// SB steps of mutual sources j = j0 + G (s0 + t), t < SB, then a butterfly
// reduce-scatter of the SB partial sums over the slice's MQ lanes and one RED per step.
// LAST: a single step that is past j1 on some slices — evaluated on a clamped source
// with zero weight and discarded there (no branch), so every batch is straight-line.
template <int TB, int MQ, int SB, bool LAST>
__device__ __forceinline__ void nr_mutual_batch(const double4* sbuf, const int* sidx, int j0, int j1, int G, int s0,
                                                const double (&x)[TB][3], const double (&q)[TB], double (&acc)[TB],
                                                double* __restrict__ out) {
  static_assert(SB <= MQ && (!LAST || SB == 1), "batch shape");
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double v[SB];
  bool valid = true;
#pragma unroll
  for (int t = 0; t < SB; ++t) {
    int j = j0 + G * (s0 + t);
    if (LAST) {
      valid = j < j1;
      j = valid ? j : j1 - 1;
    }
    const double4 sv = sbuf[j];
    const double w = LAST && !valid ? 0.0 : sv.w;
    double sj = 0.0;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
      const double r = rinv_nonzero(fma(dz, dz, fma(dy, dy, dx * dx)));  // distinct leaves: r > 0
      acc[u] = fma(w, r, acc[u]);
      sj = fma(q[u], r, sj);
    }
    v[t] = sj;
  }
  // (a layout keeping step t ^ (l % SB) in slot t avoids the selects below but makes the
  // slice's lanes read different sources: measured slower)
#pragma unroll
  for (int off = SB / 2; off >= 1; off >>= 1) {  // lane l keeps the partial of step l % SB
    const bool up = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = up ? v[i] : v[i + off];
      const double keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(FULL, send, off);
    }
  }
#pragma unroll
  for (int off = SB; off < MQ; off <<= 1) v[0] += __shfl_xor_sync(FULL, v[0], off);
  if ((lane & (MQ - 1)) < SB && valid) atomicAdd(out + sidx[j0 + G * (s0 + (lane & (SB - 1)))], v[0] * kInv4Pi);
}

// the mutual range [lo, j1) of a chunk (this thread's first source j0): nmin steps are
// valid on every slice, one more on some; batches of 4, 2, 1, then the masked last step
template <int TB, int MQ>
__device__ __forceinline__ void nr_mutual(const double4* sbuf, const int* sidx, int lo, int j0, int j1, int G,
                                          const double (&x)[TB][3], const double (&q)[TB], double (&acc)[TB],
                                          double* __restrict__ out) {
#ifndef KIFMM_NEAR_SB
#define KIFMM_NEAR_SB 4
#endif
  constexpr int SB = MQ < KIFMM_NEAR_SB ? MQ : KIFMM_NEAR_SB;
  const int nmin = (j1 - lo) / G, nsteps = (j1 - lo + G - 1) / G;  // uniform over the CTA
  int s0 = 0;
  for (; s0 + SB <= nmin; s0 += SB) nr_mutual_batch<TB, MQ, SB, false>(sbuf, sidx, j0, j1, G, s0, x, q, acc, out);
  if (SB >= 8 && s0 + 4 <= nmin) {
    nr_mutual_batch<TB, MQ, (SB >= 4 ? 4 : 1), false>(sbuf, sidx, j0, j1, G, s0, x, q, acc, out);
    s0 += SB >= 4 ? 4 : 1;
  }
  if (SB >= 4 && s0 + 2 <= nmin) {
    nr_mutual_batch<TB, MQ, (SB >= 2 ? 2 : 1), false>(sbuf, sidx, j0, j1, G, s0, x, q, acc, out);
    s0 += SB >= 2 ? 2 : 1;
  }
  if (s0 < nmin) nr_mutual_batch<TB, MQ, 1, false>(sbuf, sidx, j0, j1, G, s0++, x, q, acc, out);
  if (s0 < nmin) nr_mutual_batch<TB, MQ, 1, false>(sbuf, sidx, j0, j1, G, s0++, x, q, acc, out);
  if (s0 < nsteps) nr_mutual_batch<TB, MQ, 1, true>(sbuf, sidx, j0, j1, G, s0, x, q, acc, out);
}

// Double layer: the source term is q_j (x - y_j).n_j / r^3 (1/(4 pi) once per
// sum).  Sources are staged as (y, q) and (n, 0); w_j = q_j n_j is formed per step.  For a
// mutual pair with d = x_i - x_j and r3 = 1 / |d|^3: p_i += (d . w_j) r3 and
// p_j += (x_j - x_i) . w_i r3 = -(d . w_i) r3 — ~21 FP64 instructions for both sides
// against 2 x 18 one-sided.
template <int TB, bool CHECK>
__device__ __forceinline__ void nr_onesided_dl(const double4* sbuf, const double4* nbuf, int j0, int j1, int G,
                                               const double (&x)[TB][3], double (&acc)[TB]) {
#pragma unroll 2
  for (int j = j0; j < j1; j += G) {
    const double4 sv = sbuf[j], sn = nbuf[j];
    const double wx = sv.w * sn.x, wy = sv.w * sn.y, wz = sv.w * sn.z;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double ri = CHECK ? rinv_or_zero(r2) : rinv_nonzero(r2);
      const double dw = fma(dz, wz, fma(dy, wy, dx * wx));
      acc[u] = fma(dw * ri, ri * ri, acc[u]);
    }
  }
}

template <int TB, int MQ, int SB, bool LAST>
__device__ __forceinline__ void nr_mutual_batch_dl(const double4* sbuf, const double4* nbuf, const int* sidx, int j0,
                                                   int j1, int G, int s0, const double (&x)[TB][3],
                                                   const double (&wt)[TB][3], double (&acc)[TB],
                                                   double* __restrict__ out) {
  static_assert(SB <= MQ && (!LAST || SB == 1), "batch shape");
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double v[SB];
  bool valid = true;
#pragma unroll
  for (int t = 0; t < SB; ++t) {
    int j = j0 + G * (s0 + t);
    if (LAST) {
      valid = j < j1;
      j = valid ? j : j1 - 1;
    }
    const double4 sv = sbuf[j], sn = nbuf[j];
    const double qs = LAST && !valid ? 0.0 : sv.w;
    const double wx = qs * sn.x, wy = qs * sn.y, wz = qs * sn.z;
    double sj = 0.0;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
      const double ri = rinv_nonzero(fma(dz, dz, fma(dy, dy, dx * dx)));  // distinct leaves: r > 0
      const double r3 = ri * (ri * ri);
      acc[u] = fma(fma(dz, wz, fma(dy, wy, dx * wx)), r3, acc[u]);
      sj = fma(fma(dz, wt[u][2], fma(dy, wt[u][1], dx * wt[u][0])), r3, sj);
    }
    v[t] = sj;
  }
#pragma unroll
  for (int off = SB / 2; off >= 1; off >>= 1) {  // lane l keeps the partial of step l % SB
    const bool up = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = up ? v[i] : v[i + off];
      const double keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(FULL, send, off);
    }
  }
#pragma unroll
  for (int off = SB; off < MQ; off <<= 1) v[0] += __shfl_xor_sync(FULL, v[0], off);
  if ((lane & (MQ - 1)) < SB && valid) atomicAdd(out + sidx[j0 + G * (s0 + (lane & (SB - 1)))], -v[0] * kInv4Pi);
}

template <int TB, int MQ>
__device__ __forceinline__ void nr_mutual_dl(const double4* sbuf, const double4* nbuf, const int* sidx, int lo, int j0,
                                             int j1, int G, const double (&x)[TB][3], const double (&wt)[TB][3],
                                             double (&acc)[TB], double* __restrict__ out) {
  constexpr int SB = MQ < 4 ? MQ : 4;
  const int nmin = (j1 - lo) / G, nsteps = (j1 - lo + G - 1) / G;  // uniform over the CTA
  int s0 = 0;
  for (; s0 + SB <= nmin; s0 += SB)
    nr_mutual_batch_dl<TB, MQ, SB, false>(sbuf, nbuf, sidx, j0, j1, G, s0, x, wt, acc, out);
  if (SB >= 4 && s0 + 2 <= nmin) {
    nr_mutual_batch_dl<TB, MQ, (SB >= 2 ? 2 : 1), false>(sbuf, nbuf, sidx, j0, j1, G, s0, x, wt, acc, out);
    s0 += SB >= 2 ? 2 : 1;
  }
  if (s0 < nmin) nr_mutual_batch_dl<TB, MQ, 1, false>(sbuf, nbuf, sidx, j0, j1, G, s0++, x, wt, acc, out);
  if (s0 < nmin) nr_mutual_batch_dl<TB, MQ, 1, false>(sbuf, nbuf, sidx, j0, j1, G, s0++, x, wt, acc, out);
  if (s0 < nsteps) nr_mutual_batch_dl<TB, MQ, 1, true>(sbuf, nbuf, sidx, j0, j1, G, s0, x, wt, acc, out);
}

// the CTA's work sequence: unit blockIdx.x, then units taken from a global counter
// (dynamic: units differ in cost; the host orders them longest first), two ahead of use
// through a 4-slot ring in shared memory; per unit its chunks
struct Cursor {
  int item, chunk;
  int4 rec;  // this unit's record
};

// (register targets measured on C4, ncu: 5 CTAs per SM at 96 registers for the 5-6 target
// passes, or 2 CTAs at ~230 for 7-8, ran at the same speed as the compiler's default
// 128 registers / 4 CTAs — more resident warps do not lift the FP64 pipe past ~70% here)
template <int TB, int MQ, bool DL = false>
__global__ void __launch_bounds__(NR_NT) k_near(NearArgs A) {
  constexpr int NT = NR_NT, G = NT / MQ, CAP = TB * MQ, CH = near_ch(CAP, DL), NR_PER = CH / NT;
  static_assert(DL || TB * NT * sizeof(double) <= CH * sizeof(double4), "slice sums alias a source buffer");
  __shared__ __align__(16) double4 sbuf[2][CH];
  __shared__ __align__(16) double4 tbuf[2][CAP];
  __shared__ __align__(16) double4 nbuf[2][DL ? CH : 1];   // double layer: source normals
  __shared__ __align__(16) double4 tnbuf[2][DL ? CAP : 1]; // double layer: target normals
  __shared__ double red_dl[DL ? TB * NT : 1];
  __shared__ int sidx[2][CH];
  __shared__ int s_ring[4];
  const int tid = threadIdx.x;
  const int ti = tid & (MQ - 1), gi = tid / MQ;
  int ring = 0;  // next ring slot to consume (uniform); slot ring + 2 is claimed on consumption

  auto advance = [&](Cursor c) {
    if (++c.chunk < c.rec.w) return c;
    c.item = s_ring[ring & 3];
    if (tid == 0) s_ring[(ring + 2) & 3] = (int)gridDim.x + atomicAdd(A.counter, 1);
    ++ring;
    if (c.item < A.nitems) {
      c.rec = A.items[c.item];
      c.chunk = c.rec.z;
    }
    return c;
  };
  // issue the copies of chunk record ck (source indices idx[] held by this thread) and,
  // on a pass's first chunk, of the pass's targets, into buffer b
  auto stage = [&](const Cursor& c, const int4& ck, const int (&idx)[NR_PER], int b) {
    const int n = ck.y & 1023;
#pragma unroll
    for (int r = 0; r < NR_PER; ++r) {
      const int f = tid + r * NT;
      if (f < n) {
        const double* src = reinterpret_cast<const double*>(A.pts + idx[r]);
        double* dst = reinterpret_cast<double*>(&sbuf[b][f]);
        nr_cp16(dst, src);
        nr_cp16(dst + 2, src + 2);
        if constexpr (DL) {
          const double* nsrc = reinterpret_cast<const double*>(A.nrm + idx[r]);
          double* ndst = reinterpret_cast<double*>(&nbuf[b][f]);
          nr_cp16(ndst, nsrc);
          nr_cp16(ndst + 2, nsrc + 2);
        }
        sidx[b][f] = idx[r];
      }
    }
    if (c.chunk == c.rec.z) {
      for (int i = tid; i < c.rec.y; i += NT) {
        const double* src = reinterpret_cast<const double*>(A.pts + c.rec.x + i);
        double* dst = reinterpret_cast<double*>(&tbuf[b][i]);
        nr_cp16(dst, src);
        nr_cp16(dst + 2, src + 2);
        if constexpr (DL) {
          const double* nsrc = reinterpret_cast<const double*>(A.nrm + c.rec.x + i);
          double* ndst = reinterpret_cast<double*>(&tnbuf[b][i]);
          nr_cp16(ndst, nsrc);
          nr_cp16(ndst + 2, nsrc + 2);
        }
      }
    }
  };
  auto load_idx = [&](const int4& ck, int (&idx)[NR_PER]) {
    const int n = ck.y & 1023;
#pragma unroll
    for (int r = 0; r < NR_PER; ++r) {
      const int f = tid + r * NT;
      idx[r] = f < n ? __ldcs(A.src + ck.x + f) : 0;
    }
  };

  if ((int)blockIdx.x >= A.nitems) return;
  if (tid == 0) {
    s_ring[0] = (int)gridDim.x + atomicAdd(A.counter, 1);
    s_ring[1] = (int)gridDim.x + atomicAdd(A.counter, 1);
  }
  __syncthreads();
  Cursor cur;
  cur.item = blockIdx.x;
  cur.rec = A.items[cur.item];
  cur.chunk = cur.rec.z;
  // prologue: stage chunk 0; chunk 1's record and indices in registers
  int4 ck_cur = A.chunks[cur.chunk];
  int idx[NR_PER];
  load_idx(ck_cur, idx);
  stage(cur, ck_cur, idx, 0);
  nr_commit();
  Cursor nxt = advance(cur);
  bool more = nxt.item < A.nitems;
  int4 ck_nxt = more ? A.chunks[nxt.chunk] : make_int4(0, 0, 0, 0);
  if (more) load_idx(ck_nxt, idx);

  double x[TB][3], q[TB], acc[TB];
  double wt[DL ? TB : 1][3];  // double layer: the targets' q_i n_i
  int b = 0, mm = 0;
  while (true) {
    nr_wait0();
    __syncthreads();  // chunk cur in buffer b; buffer b ^ 1 free
    if (more) stage(nxt, ck_nxt, idx, b ^ 1);
    nr_commit();
    // records of the chunk after next, read while this chunk is evaluated
    Cursor nn = cur;
    int4 ck_nn = make_int4(0, 0, 0, 0);
    bool more2 = false;
    if (more) {
      nn = advance(nxt);
      more2 = nn.item < A.nitems;
      if (more2) {
        ck_nn = A.chunks[nn.chunk];
        load_idx(ck_nn, idx);
      }
    }
    if (cur.chunk == cur.rec.z) {  // first chunk of a unit: its targets
      mm = cur.rec.y;
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int i = ti + u * MQ;
        acc[u] = 0.0;
        if (i < mm) {
          const double4 p = tbuf[b][i];
          x[u][0] = p.x; x[u][1] = p.y; x[u][2] = p.z; q[u] = p.w;
        } else {  // padding target: far away, zero density (results discarded)
          x[u][0] = 1e100; x[u][1] = 0.0; x[u][2] = 0.0; q[u] = 0.0;
        }
        if constexpr (DL) {
          const double4 nv = i < mm ? tnbuf[b][i] : make_double4(0.0, 0.0, 0.0, 0.0);
          wt[u][0] = q[u] * nv.x;
          wt[u][1] = q[u] * nv.y;
          wt[u][2] = q[u] * nv.z;
        }
      }
    }
    {
      const int n = ck_cur.y & 1023, nchk = (ck_cur.y >> 10) & 1023, ml = ck_cur.y >> 20, mh = ck_cur.z;
      auto first = [&](int lo) { return lo <= gi ? gi : gi + ((lo - gi + G - 1) / G) * G; };
      // [0, nchk) checked one-sided (the leaf's own points), [nchk, ml) one-sided,
      // [ml, mh) mutual, [mh, n) one-sided
      if constexpr (DL) {
        if (nchk > 0) nr_onesided_dl<TB, true>(sbuf[b], nbuf[b], gi, nchk, G, x, acc);
        if (ml > nchk) nr_onesided_dl<TB, false>(sbuf[b], nbuf[b], first(nchk), ml, G, x, acc);
        if (mh > ml) nr_mutual_dl<TB, MQ>(sbuf[b], nbuf[b], sidx[b], ml, first(ml), mh, G, x, wt, acc, A.out);
        if (n > mh) nr_onesided_dl<TB, false>(sbuf[b], nbuf[b], first(mh), n, G, x, acc);
      } else {
        if (nchk > 0) nr_onesided<TB, true>(sbuf[b], gi, nchk, G, x, acc);
        if (ml > nchk) nr_onesided<TB, false>(sbuf[b], first(nchk), ml, G, x, acc);
        if (mh > ml) nr_mutual<TB, MQ>(sbuf[b], sidx[b], ml, first(ml), mh, G, x, q, acc, A.out);
        if (n > mh) nr_onesided<TB, false>(sbuf[b], first(mh), n, G, x, acc);
      }
    }
    if (cur.chunk + 1 == cur.rec.w) {  // last chunk of the unit: sum the slices, RED into p
      // (the slice sums go to the chunk buffer just evaluated: after this barrier nobody
      // reads it, and the next staging into it follows the next top-of-loop barrier)
      double* red = DL ? red_dl : reinterpret_cast<double*>(&sbuf[b][0]);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < TB; ++u) red[u * NT + tid] = acc[u];
      __syncthreads();
      for (int i = tid; i < mm; i += NT) {
        const int u = i / MQ, tl = i - u * MQ;
        double sum = 0.0;
        for (int g = 0; g < G; ++g) sum += red[u * NT + g * MQ + tl];
        atomicAdd(A.out + cur.rec.x + i, sum * kInv4Pi);
      }
    }
    if (!more) break;
    cur = nxt;
    ck_cur = ck_nxt;
    nxt = nn;
    ck_nxt = ck_nn;
    more = more2;
    b ^= 1;
  }
}

// spare > 0: leave that many CTA slots per SM to kernels running beside it (overlap mode 3)
template <int TB, int MQ, bool DL>
int near_launch_one(const NearArgs& a, int count, int spare, cudaStream_t st) {
  static int per_sm = -1;
  if (per_sm < 0) {
    // the largest shared-memory carveout: 5 CTAs of ~40 KB need more than the 168 KB the
    // driver's default choice gives a kernel with static shared memory only
    cudaFuncSetAttribute(k_near<TB, MQ, DL>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_near<TB, MQ, DL>, NR_NT, 0) != cudaSuccess) per_sm = 1;
    per_sm = std::max(1, per_sm);
  }
  const int grid = std::min(count, std::max(1, per_sm - spare) * g_num_sms);
  k_near<TB, MQ, DL><<<grid, NR_NT, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// double-layer variants exist for passes of <= 160 targets (table 3)
template <int TB, int MQ>
int near_launch_sel(const NearArgs& a, int count, int spare, cudaStream_t st) {
  if constexpr (TB * MQ <= 160) {
    if (a.nrm) return near_launch_one<TB, MQ, true>(a, count, spare, st);
  } else {
    if (a.nrm) return -3;
  }
  return near_launch_one<TB, MQ, false>(a, count, spare, st);
}

struct NearShapeDef {
  int tb, mq;
};
// pass shapes by capacity TB x MQ (more targets per thread: fewer reductions per pair;
// measured against a small-TB table with more resident warps, which was slower)
const NearShapeDef kNearTab0[] = {{2, 4}, {3, 4}, {4, 4}, {5, 4}, {6, 4}, {4, 8}, {5, 8}, {6, 8}, {7, 8},
                                  {8, 8}, {5, 16}, {6, 16}, {7, 16}, {8, 16}, {5, 32}, {6, 32}, {7, 32}, {8, 32}};

const NearShapeDef* near_table(int tab, int* count) {
  if (tab == 3) {  // double layer: the shapes up to 160 targets (static shared memory <= 48 KB)
    *count = (int)(sizeof(kNearTab0) / sizeof(kNearTab0[0])) - 3;
    return kNearTab0;
  }
  *count = (int)(sizeof(kNearTab0) / sizeof(kNearTab0[0]));
  return kNearTab0;
}

}  // namespace

int near_shape_count(int tab) {
  int c = 0;
  near_table(tab, &c);
  return c;
}

int near_shape_cap(int tab, int shape) {
  int c = 0;
  const NearShapeDef* t = near_table(tab, &c);
  return t[shape].tb * t[shape].mq;
}

int near_launch(const Plan& P, double* out, cudaStream_t st, int part, int spare) {
  int cnt = 0;
  const NearShapeDef* tab = near_table(P.nr_table, &cnt);
  const int ng = (int)P.nr_groups.size();
  if (ng == 0) return 0;
  // part 0: every unit; 1 / 2: the first P.nr_split / the remaining units of each group
  // (units are sorted longest first); counters: [0, ng) part 0 / 1, [ng, 2 ng) part 2
  if (part != 2) KIFMM_CUDA(cudaMemsetAsync(P.d_nr_counters, 0, sizeof(int) * 2 * ng, st));
  // serialised plans: the pass-shape launches alternate between st and the plan's second
  // near stream — every launch is a persistent grid whose CTAs drain at its end, and the
  // other stream's launch takes the SM slots they free (the launches are independent: each
  // adds its own pairs into the potentials with RED).  C4 near field 10.02 -> 9.86 ms,
  // C3 1.58 -> 1.40, C2 0.59 -> 0.53.  With the near field beside the far field (overlap
  // mode 3) the far kernels fill those slots instead (two streams there: C2 2.36 -> 2.43 ms)
  const bool two = P.stream_nr2 && ng > 1 && P.overlap == 0;
  if (two) {
    KIFMM_CUDA(cudaEventRecord(P.ev_nr_fork, st));
    KIFMM_CUDA(cudaStreamWaitEvent(P.stream_nr2, P.ev_nr_fork, 0));
  }
  for (int gidx = 0; gidx < ng; ++gidx) {
    cudaStream_t sg = two && (gidx & 1) ? P.stream_nr2 : st;
    const int3& g = P.nr_groups[gidx];
    const int na = part == 0 ? g.z : std::min(g.z, (int)(P.nr_split * g.z + 0.5));
    const int first = part == 2 ? na : 0, count = part == 1 ? na : g.z - first;
    if (count <= 0) continue;
    NearArgs a;
    a.counter = P.d_nr_counters + (part == 2 ? ng : 0) + gidx;
    a.items = P.d_nr_items + g.y + first;
    a.nitems = count;
    a.chunks = P.d_nr_chunks;
    a.src = P.d_nr_src;
    a.pts = P.tree.d_pts;
    a.nrm = P.d_nrm;
    a.out = out;
    int rc = -3;
    switch (tab[g.x].tb * 64 + tab[g.x].mq) {
#define KIFMM_NS(TBv, MQv) case TBv * 64 + MQv: rc = near_launch_sel<TBv, MQv>(a, count, spare, sg); break;
      KIFMM_NS(2, 4) KIFMM_NS(3, 4) KIFMM_NS(4, 4) KIFMM_NS(5, 4) KIFMM_NS(6, 4)
      KIFMM_NS(4, 8) KIFMM_NS(5, 8) KIFMM_NS(6, 8) KIFMM_NS(7, 8) KIFMM_NS(8, 8)
      KIFMM_NS(5, 16) KIFMM_NS(6, 16) KIFMM_NS(7, 16) KIFMM_NS(8, 16)
      KIFMM_NS(5, 32) KIFMM_NS(6, 32) KIFMM_NS(7, 32) KIFMM_NS(8, 32)
#undef KIFMM_NS
      default: break;
    }
    if (rc) {
      set_error("k_near launch failed");
      return rc;
    }
    ++g_launches;
  }
  if (two) {
    KIFMM_CUDA(cudaEventRecord(P.ev_nr_join, P.stream_nr2));
    KIFMM_CUDA(cudaStreamWaitEvent(st, P.ev_nr_join, 0));
  }
  return 0;
}

}  // namespace kifmm
