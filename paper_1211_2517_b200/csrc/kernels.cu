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
};

constexpr int EV_NT = 256;
constexpr int EV_CH = 512;
constexpr int EV_SEG = 128;

template <bool SURF_TGT>
__global__ void __launch_bounds__(EV_NT) k_eval(EvalArgs A) {
  __shared__ double4 sbuf[EV_CH];
  __shared__ double red[EV_NT];
  __shared__ int s_pref[EV_SEG + 1];
  __shared__ int4 s_seg[EV_SEG];
  const int item = blockIdx.x;
  const int4 it = A.items[item];
  const int box = it.x;
  const double4 gb = A.geom[box];
  int m, tbeg = 0;
  if (SURF_TGT) m = A.n;
  else { tbeg = A.pbeg[box]; m = A.pend[box] - tbeg; }
  const int sb = A.seg_off[item], se = A.seg_off[item + 1];
  for (int t0 = 0; t0 < m; t0 += EV_NT) {
    const int mm = min(m - t0, EV_NT);
    const int G = EV_NT / mm;
    const int ti = threadIdx.x % mm, gi = threadIdx.x / mm;
    const bool act = gi < G;
    double x0 = 0, x1 = 0, x2 = 0;
    if (act) {
      if (SURF_TGT) {
        double rad = gb.w * A.tgt_f;
        x0 = gb.x + rad * A.surf[3 * (t0 + ti)];
        x1 = gb.y + rad * A.surf[3 * (t0 + ti) + 1];
        x2 = gb.z + rad * A.surf[3 * (t0 + ti) + 2];
      } else {
        double4 p = A.pts[tbeg + t0 + ti];
        x0 = p.x; x1 = p.y; x2 = p.z;
      }
    }
    double acc = 0.0;
    for (int s0 = sb; s0 < se; s0 += EV_SEG) {
      const int ns = min(EV_SEG, se - s0);
      __syncthreads();
      if (threadIdx.x == 0) {
        int run = 0;
        for (int s = 0; s < ns; ++s) {
          int4 sg = A.segs[s0 + s];
          s_seg[s] = sg;
          s_pref[s] = run;
          run += sg.w;
        }
        s_pref[ns] = run;
      }
      __syncthreads();
      const int total = s_pref[ns];
      for (int c0 = 0; c0 < total; c0 += EV_CH) {
        const int cn = min(EV_CH, total - c0);
        __syncthreads();
        for (int f = threadIdx.x; f < cn; f += EV_NT) {
          int fi = c0 + f;
          int lo = 0, hi = ns;  // last segment with prefix <= fi
          while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (s_pref[mid] <= fi) lo = mid; else hi = mid;
          }
          const int4 sg = s_seg[lo];
          const int j = fi - s_pref[lo];
          double4 v;
          if (sg.x == 0) {
            v = A.pts[sg.y + j];
          } else {
            const double4 gs = A.geom[sg.z];
            const double rad = gs.w * (sg.x == 1 ? A.f_out : A.f_in);
            const double* q = (sg.x == 1 ? A.eqd1 : A.eqd2) + (size_t)sg.y * A.ldq;
            v = make_double4(gs.x + rad * A.surf[3 * j], gs.y + rad * A.surf[3 * j + 1], gs.z + rad * A.surf[3 * j + 2], q[j]);
          }
          sbuf[f] = v;
        }
        __syncthreads();
        if (act) {
#pragma unroll 4
          for (int j = gi; j < cn; j += G) {
            const double4 s = sbuf[j];
            const double dx = x0 - s.x, dy = x1 - s.y, dz = x2 - s.z;
            const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            acc = fma(s.w, rinv_or_zero(r2), acc);
          }
        }
      }
    }
    __syncthreads();
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < mm) {
      double s = 0;
      for (int gg = 0; gg < G; ++gg) s += red[gg * mm + threadIdx.x];
      s *= kInv4Pi;
      if (SURF_TGT) A.out[(size_t)it.y * A.ldo + t0 + threadIdx.x] = s;
      else A.out[tbeg + t0 + threadIdx.x] = s;
    }
  }
}

__global__ void k_set_density(double4* __restrict__ pts, const int32_t* __restrict__ perm, const double* __restrict__ q,
                              int64_t N) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) pts[i].w = q[perm[i]];
}

__global__ void k_gather_output(const double* __restrict__ pnear, const double* __restrict__ pfar,
                                const int32_t* __restrict__ perm, int64_t N, double* __restrict__ pot) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) pot[perm[i]] = pnear[i] + pfar[i];
}

// ----------------------------------------------------------------------------
// host-side launch helpers
// ----------------------------------------------------------------------------
namespace {

inline int nblk(int64_t n, int t = 256) { return std::max(1, (int)((n + t - 1) / t)); }

int ggs_nt(int M, int K) { return (size_t)(K + 4 + M + 2) * 64 * 8 <= 116 * 1024 ? 64 : 32; }

int g_launches = 0;

int launch_ggs(const GemmLaunch& g, const double* ops, int op_stride, int M, int K, int mvalid, const double* X,
               int ldx, double* Y, int ldy, bool atomic, cudaStream_t st) {
  if (g.ntiles == 0) return 0;
  ++g_launches;
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

int ggs_tile_width(int M, int K) { return ggs_nt(M, K); }

int kernels_init() {
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  KIFMM_CUDA(cudaFuncSetAttribute(k_ggs<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  return 0;
}


// Evaluation work lists live in the plan; see build_schedules (schedule.cpp).
struct EvalLaunch;

int matvec_device(Plan& P, const double* d_density, double* d_pot, cudaStream_t st) {
  Tree& T = P.tree;
  const int64_t N = T.N;
  const int kp = P.kp, np = P.np, k = P.k, n = P.n;
  auto mark = [&](int i) { if (P.profile) cudaEventRecord(P.ev_phase[i], st); };
  g_launches = 0;
  mark(0);
  ++g_launches;
  k_set_density<<<nblk(N), 256, 0, st>>>(T.d_pts, T.d_perm, d_density, N);
  KIFMM_CUDA(cudaGetLastError());
  KIFMM_CUDA(cudaMemsetAsync(P.d_qhat, 0, sizeof(double) * (size_t)T.nboxes * kp, st));
  KIFMM_CUDA(cudaMemsetAsync(P.d_lhat, 0, sizeof(double) * (size_t)T.nboxes * kp, st));
  // near field (P2P: U + direct W/X), independent of the far field
  EvalArgs ea{};
  ea.pts = T.d_pts; ea.geom = T.d_geom; ea.pbeg = T.d_pbeg; ea.pend = T.d_pend;
  ea.surf = P.d_surf; ea.n = n; ea.f_in = 1.0 + P.d; ea.f_out = 3.0 - 2.0 * P.d; ea.ldq = np;
  if (P.n_tleaf > 0) {
    EvalArgs a = ea;
    a.items = P.d_tleaf_items; a.seg_off = P.d_near_off; a.segs = P.d_near_seg; a.out = P.d_pot_near;
    k_eval<false><<<P.n_tleaf, EV_NT, 0, st>>>(a);
    ++g_launches;
    KIFMM_CUDA(cudaGetLastError());
  }
  mark(1);
  // S2M stage 1: check potentials of leaves at level >= 2
  if (P.n_s2m > 0) {
    EvalArgs a = ea;
    a.items = P.d_s2m_items; a.seg_off = P.d_s2m_off; a.segs = P.d_s2m_seg; a.tgt_f = 3.0 - 2.0 * P.d;
    a.out = P.d_chk_s2m; a.ldo = np;
    k_eval<true><<<P.n_s2m, EV_NT, 0, st>>>(a);
    ++g_launches;
    KIFMM_CUDA(cudaGetLastError());
  }
  // S2M stage 2: q^'_B = S' c  (store)
  if (launch_ggs(P.g_s2m, P.d_S, 0, kp, np, k, P.d_chk_s2m, np, P.d_qhat, kp, false, st)) return -3;
  mark(2);
  // M2M, finest child level first: q^'_P += 1/2 M~_o q^'_c
  for (auto& g : P.g_m2m)
    if (launch_ggs(g, P.d_M, kp * kp, kp, kp, k, P.d_qhat, kp, P.d_qhat, kp, true, st)) return -3;
  mark(3);
  // M2L, all levels in one launch: l^_B += C_delta q^'_A
  if (launch_ggs(P.g_m2l, P.d_C, kp * kp, kp, kp, k, P.d_qhat, kp, P.d_lhat, kp, true, st)) return -3;
  mark(4);
  // X list (S2L): check potentials on DC of the target, then U^T projection (atomic)
  if (P.n_xnd > 0) {
    EvalArgs a = ea;
    a.items = P.d_x_items; a.seg_off = P.d_x_off; a.segs = P.d_x_seg; a.tgt_f = 1.0 + P.d;
    a.out = P.d_chk_x; a.ldo = np;
    k_eval<true><<<P.n_xnd, EV_NT, 0, st>>>(a);
    ++g_launches;
    KIFMM_CUDA(cudaGetLastError());
    if (launch_ggs(P.g_x, P.d_Ut, 0, kp, np, k, P.d_chk_x, np, P.d_lhat, kp, true, st)) return -3;
  }
  mark(5);
  // L2L, coarsest parent level first: l^_c += L~_o l^_P
  for (auto& g : P.g_l2l)
    if (launch_ggs(g, P.d_L, kp * kp, kp, kp, k, P.d_lhat, kp, P.d_lhat, kp, true, st)) return -3;
  mark(6);
  // L2T stage 1: q_d = r_l T' l^_B ; W stage 1: q_u = r_A U q^'_A  (store)
  if (launch_ggs(P.g_l2t, P.d_T, 0, np, kp, n, P.d_lhat, kp, P.d_eqd_l2t, np, false, st)) return -3;
  if (launch_ggs(P.g_w, P.d_Ue, 0, np, kp, n, P.d_qhat, kp, P.d_eqd_w, np, false, st)) return -3;
  // L2T + W stage 2: potentials at the targets of each leaf
  if (P.n_tleaf > 0) {
    EvalArgs a = ea;
    a.items = P.d_tleaf_items; a.seg_off = P.d_far_off; a.segs = P.d_far_seg; a.out = P.d_pot_far;
    a.eqd1 = P.d_eqd_l2t; a.eqd2 = P.d_eqd_w;
    k_eval<false><<<P.n_tleaf, EV_NT, 0, st>>>(a);
    ++g_launches;
    KIFMM_CUDA(cudaGetLastError());
  }
  mark(7);
  k_gather_output<<<nblk(N), 256, 0, st>>>(P.d_pot_near, P.d_pot_far, T.d_perm, N, d_pot);
  ++g_launches;
  P.launches = g_launches;
  KIFMM_CUDA(cudaGetLastError());
  mark(8);
  if (P.profile) P.profiled = true;
  return 0;
}

}  // namespace kifmm
