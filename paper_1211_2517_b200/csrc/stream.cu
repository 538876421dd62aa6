// Leaf-operator GEMVs of the upward side (S2M, X) streamed through shared memory by bulk
// copies.
//
// Both leaf-level translations with per-leaf operators (DESIGN.md §5 "leaf-op mode") read
// kp doubles per source point and do one FMA per double: HBM-bound (C4: 8.6 GB for S2M,
// 3.7 GB for X per matvec).  Each is a persistent grid of single-warp CTAs, kStreamCtaPerSm
// per SM: lane 0 issues cp.async.bulk copies (SASS UBLKCP) of contiguous operator rows plus
// the chunk's densities into an NS-stage shared-memory ring, each stage completing on its
// own mbarrier (expect_tx bytes); the warp consumes stage s while the other stage is in
// flight, then refills s.  ~200 KB in flight per SM keeps HBM busy with twelve warps per SM
// (C4 S2M 6.3 TB/s, 1.36 ms, against 5.1 TB/s for the register-path GEMV).  The waits are
// mbarrier.try_wait (suspended, not spinning).
//
// Work: an item = (first operator row, rows, first weight point, output box):
//   S2M  q^'_B  = sum_j q_j S_B[j]   store
//   X    l^_B  += sum_j q_j X_(B,A)[j]     (projection)       RED
// Each CTA streams a contiguous range of items (host-balanced by rows, stream_plan below).
// Measured and not kept: the L2T dot-product form (a reduce-scatter
// over the warp per 16 rows) reached 4.3 TB/s against 6.4 for k_l2t_leafop; single-warp
// CTAs sized to run BESIDE k_near (1 per SM, ~23 KB) reached only 1-2 TB/s and slowed
// k_near (C4 25.2 vs 21.8 ms).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fmm_internal.h"

namespace kifmm {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// 12 single-warp CTAs per SM, 2 stages each (~200 KB in flight per SM): measured on C4
// against 4 x 6 stages (S2M 1.40 / X 0.69 ms), 8 x 3 (1.37 / 0.60), 16 x 2 of 6 KB
// (1.35 / 0.58); 12 x 2: 1.36 / 0.57 ms
constexpr int kStreamCtaPerSm = 12;

// rows per stage (the stage also holds up to max(KP, RS + 2) doubles of weights);
// kStreamCtaPerSm CTAs x NS stages x ~8.7 KB (kp <= 64) / 7.5 KB (kp = 104) per SM
template <int KP>
struct StreamShape {
  static constexpr int RS = KP <= 64 ? 16 : 8;
  static constexpr int NS = 2;
  static constexpr int EXTRA = (KP > RS + 2 ? KP : RS + 2);
  static constexpr int STAGE = (RS * KP + EXTRA) * 8;  // bytes (multiple of 16)
  static constexpr int T = (KP + 63) / 64;            // double2 column units per lane
  static_assert(STAGE % 16 == 0, "bulk copies move multiples of 16 bytes");
};

struct StreamArgs {
  const int4* items;     // (first row, rows, first weight / output point, output box)
  const int* cta_begin;  // CTA c streams items [cta_begin[c], cta_begin[c + 1])
  const double* mat;     // operator rows, KP doubles each
  const double* q;       // densities in sorted order (contiguous copy of pts.w)
  double* out;           // per-box rows (q^' or l^)
};

// lane's double2 unit t covers columns 2 lane + 64 t, + 1
template <int KP>
__device__ __forceinline__ bool col_ok(int lane, int t) { return 2 * lane + 64 * t < KP; }

template <int KP, bool ATOMIC>
__global__ void __launch_bounds__(32, 1) k_stream(StreamArgs A) {
  using SS = StreamShape<KP>;
  constexpr int RS = SS::RS, NS = SS::NS, T = SS::T;
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[NS];
  const int lane = threadIdx.x;
  const int i0 = A.cta_begin[blockIdx.x], i1 = A.cta_begin[blockIdx.x + 1];
  if (i0 >= i1) return;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // ---- producer cursor (uniform over the warp; lane 0 issues)
  int iss_it = i0, iss_r = 0;
  int4 iss_rec = A.items[i0];
  auto issue = [&](int seq) {
    if (iss_it >= i1) return;
    const int s = seq % NS;
    const int nr = min(RS, iss_rec.y - iss_r);
    unsigned char* st = ring + (size_t)s * SS::STAGE;
    if (lane == 0) {
      const uint32_t bar = smem_u32(&full[s]);
      const uint32_t rbytes = (uint32_t)nr * KP * 8;
      // the chunk's densities (an aligned pair-superset: bulk copies move 16-byte units)
      const long w0 = (long)iss_rec.z + iss_r, a0 = w0 & ~1L, a1 = (w0 + nr + 1) & ~1L;
      const double* xsrc = A.q + a0;
      const uint32_t xbytes = (uint32_t)(a1 - a0) * 8;
      // the ring slot was last read through the generic proxy: order those reads before
      // the async-proxy writes of the refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rbytes + xbytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(st)),
          "l"(A.mat + ((size_t)iss_rec.x + iss_r) * KP), "r"(rbytes), "r"(bar)
          : "memory");
      asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(st + RS * KP * 8)),
            "l"(xsrc), "r"(xbytes), "r"(bar)
            : "memory");
    }
    iss_r += nr;
    if (iss_r >= iss_rec.y) {
      iss_r = 0;
      if (++iss_it < i1) iss_rec = A.items[iss_it];
    }
  };
  for (int s = 0; s < NS; ++s) issue(s);

  // ---- consumer
  int it = i0, r0 = 0;
  int4 rec = A.items[i0];
  double acc[4][T][2];  // four row phases of accumulators
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;
  for (int seq = 0; it < i1; ++seq) {
    const int s = seq % NS;
    const uint32_t par = (uint32_t)(seq / NS) & 1u;
    const uint32_t bar = smem_u32(&full[s]);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar), "r"(par)
          : "memory");
    const int nr = min(RS, rec.y - r0);
    const double* rows = reinterpret_cast<const double*>(ring + (size_t)s * SS::STAGE);
    const double* extra = rows + RS * KP;
    {
      const double* w = extra + (((long)rec.z + r0) & 1);
#pragma unroll 2
      for (int r = 0; r < nr; r += 4) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          if (r + a < nr) {
            const double wr = w[r + a];
#pragma unroll
            for (int t = 0; t < T; ++t)
              if (col_ok<KP>(lane, t)) {
                const double2 v = *reinterpret_cast<const double2*>(rows + (r + a) * KP + 2 * lane + 64 * t);
                acc[a][t][0] = fma(wr, v.x, acc[a][t][0]);
                acc[a][t][1] = fma(wr, v.y, acc[a][t][1]);
              }
          }
        }
      }
    }
    __syncwarp();  // every lane is done with stage s
    issue(seq + NS);
    r0 += nr;
    if (r0 >= rec.y) {  // item done
      const int nxt = it + 1;
      const int4 nrec = nxt < i1 ? A.items[nxt] : make_int4(0, 0, 0, -1);
      if (nrec.w != rec.w) {  // output box done (X: consecutive items may share it)
#pragma unroll
        for (int t = 0; t < T; ++t)
          if (col_ok<KP>(lane, t)) {
            double* o = A.out + (size_t)rec.w * KP + 2 * lane + 64 * t;
            const double s0 = (acc[0][t][0] + acc[1][t][0]) + (acc[2][t][0] + acc[3][t][0]);
            const double s1 = (acc[0][t][1] + acc[1][t][1]) + (acc[2][t][1] + acc[3][t][1]);
            if (ATOMIC) {
              atomicAdd(o, s0);
              atomicAdd(o + 1, s1);
            } else {
              o[0] = s0;
              o[1] = s1;
            }
          }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int t = 0; t < T; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;
      }
      it = nxt;
      r0 = 0;
      rec = nrec;
    }
  }
}

template <int KP, bool ATOMIC>
int launch_one(const StreamPlan& S, const double* mat, const double* q, double* out, cudaStream_t st) {
  if (S.nitems == 0) return 0;
  using SS = StreamShape<KP>;
  const int smem = SS::NS * SS::STAGE;
  static bool attr = false;
  if (!attr) {
    KIFMM_CUDA(cudaFuncSetAttribute(k_stream<KP, ATOMIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    KIFMM_CUDA(cudaFuncSetAttribute(k_stream<KP, ATOMIC>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    (int)cudaSharedmemCarveoutMaxShared));
    attr = true;
  }
  StreamArgs a{S.d_items, S.d_cta, mat, q, out};
  k_stream<KP, ATOMIC><<<S.ncta, 32, smem, st>>>(a);
  KIFMM_CUDA(cudaGetLastError());
  return 0;
}

template <bool ATOMIC>
int launch_kp(int kp, const StreamPlan& S, const double* mat, const double* q, double* out, cudaStream_t st) {
  switch (kp) {
    case 32: return launch_one<32, ATOMIC>(S, mat, q, out, st);
    case 64: return launch_one<64, ATOMIC>(S, mat, q, out, st);
    case 104: return launch_one<104, ATOMIC>(S, mat, q, out, st);
  }
  set_error("stream GEMV: unsupported kp " + std::to_string(kp));
  return -3;
}

}  // namespace

int stream_s2m(const Plan& P, cudaStream_t st) {
  if (P.sw_s2m.nitems == 0) return 0;
  ++g_launches;
  return launch_kp<false>(P.kp, P.sw_s2m, P.d_s2m_mat, P.d_q_sorted, P.d_qhat, st);
}
int stream_x(const Plan& P, cudaStream_t st) {
  if (P.sw_x.nitems == 0) return 0;
  ++g_launches;
  return launch_kp<true>(P.kp, P.sw_x, P.d_x_mat, P.d_q_sorted, P.d_lhat, st);
}

// Host: items in streaming order, cut into ncta contiguous ranges of ~equal rows (a range
// boundary never splits the items of one output box, so a CTA owns its boxes).
int stream_plan(Plan& P, StreamPlan& S, const std::vector<int4>& items, cudaStream_t st) {
  S.nitems = (int)items.size();
  S.ncta = 0;
  if (items.empty()) return 0;
  int64_t total = 0;
  for (const int4& it : items) total += it.y;
  const int ncta = std::max(1, std::min(kStreamCtaPerSm * g_num_sms, S.nitems));
  std::vector<int> cta(ncta + 1, S.nitems);
  cta[0] = 0;
  int64_t acc = 0;
  int c = 1;
  for (int i = 0; i < S.nitems && c < ncta; ++i) {
    acc += items[i].y;
    const bool box_end = i + 1 == S.nitems || items[i + 1].w != items[i].w;
    if (box_end && acc * ncta >= total * c) cta[c++] = i + 1;
  }
  for (; c < ncta; ++c) cta[c] = S.nitems;
  S.ncta = ncta;
  S.rows = total;
  int4* di = nullptr;
  int* dc = nullptr;
  KIFMM_CUDA(cudaMalloc(&di, sizeof(int4) * items.size()));
  P.allocations.push_back(di);
  KIFMM_CUDA(cudaMalloc(&dc, sizeof(int) * cta.size()));
  P.allocations.push_back(dc);
  KIFMM_CUDA(cudaMemcpyAsync(di, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaMemcpyAsync(dc, cta.data(), sizeof(int) * cta.size(), cudaMemcpyHostToDevice, st));
  KIFMM_CUDA(cudaStreamSynchronize(st));
  S.d_items = di;
  S.d_cta = dc;
  return 0;
}

}  // namespace kifmm
