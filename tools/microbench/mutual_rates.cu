// Issue-rate limits of the mutual near-field pair loop (k_near's inner batch) on B200:
// TB targets per thread in registers, sources broadcast from shared memory per slice of MQ
// lanes, each source step accumulating both the targets' sums and the source's reverse sum
// s_j = sum_u q_u G(x_u, y_j).  Variants (FP64 instructions per unordered pair in brackets):
//   0 one-sided                (12)  acc_u += w_j G
//   1 mutual, no reduction     (13)  + s_j, kept in a register
//   2 mutual + butterfly       (13)  + the SB = 4 reduce-scatter over MQ = 8 lanes per 4 steps
//   3 as 2 + k_near's RED of each reduced reverse sum to a random potential (index from
//     shared memory)
//   4 as 3 + a CTA barrier every 8 batches (k_near's chunk of 512 sources over 16 slices)
// Reports pairs/s and the FP64 instruction-lane rate against 148 x 64 x clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mutual_rates mutual_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double kC3 = 0.375;

__device__ __forceinline__ double rinv(double r2) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double t = r2 * y0, e = fma(-t, y0, 1.0), p = fma(e, kC3, 0.5), h = y0 * e;
  return fma(h, p, y0);
}

template <int TB, int VAR, int MINB, int MQ = 8>
__global__ void __launch_bounds__(128, MINB) k_mut(double* out, const double4* __restrict__ src, int ns, int reps,
                                                   double* pot) {
  constexpr int SB = 4, G = 128 / MQ;
  __shared__ double4 sb[1024];
  __shared__ int sidx[1024];
  for (int j = threadIdx.x; j < ns; j += blockDim.x) {
    sb[j] = src[j];
    sidx[j] = (int)(((unsigned)(j + 1) * 2654435761u + blockIdx.x * 40503u) & ((1u << 22) - 1));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, ti = threadIdx.x & (MQ - 1), gi = threadIdx.x / MQ;
  double x[TB][3], q[TB], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    // every coordinate differs per target (a shared coordinate lets the compiler drop that
    // difference for the other targets: 245 instead of 265 FP64 instructions per batch)
    x[u][0] = 0.5 + 1e-4 * (ti + 7 * u); x[u][1] = 0.25 + 1e-5 * gi + 3e-6 * u; x[u][2] = -0.125 * u + 1e-7 * ti;
    q[u] = 0.1 * u; acc[u] = 0;
  }
  double red = 0.0;
  for (int r = 0; r < reps; ++r) {
    int nb = 0;
    for (int j0 = gi; j0 + G * (SB - 1) < ns; j0 += G * SB) {
      if (VAR == 4 && ++nb == 8) {
        nb = 0;
        __syncthreads();
      }
      double v[SB];
#pragma unroll
      for (int t = 0; t < SB; ++t) {
        const double4 sv = sb[j0 + G * t];
        double sj = 0.0;
#pragma unroll
        for (int u = 0; u < TB; ++u) {
          const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
          const double g = rinv(fma(dz, dz, fma(dy, dy, dx * dx)));
          acc[u] = fma(sv.w, g, acc[u]);
          if (VAR >= 1) sj = fma(q[u], g, sj);
        }
        v[t] = sj;
      }
      if (VAR == 1) {
#pragma unroll
        for (int t = 0; t < SB; ++t) red += v[t];
      }
      if (VAR >= 2) {
#pragma unroll
        for (int off = SB / 2; off >= 1; off >>= 1) {
          const bool up = lane & off;
#pragma unroll
          for (int i = 0; i < off; ++i) {
            const double send = up ? v[i] : v[i + off];
            const double keep = up ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
#pragma unroll
        for (int off = SB; off < MQ; off <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        if (VAR >= 3) {
          if ((lane & (MQ - 1)) < SB) atomicAdd(pot + sidx[j0 + G * (lane & (SB - 1))], v[0] * 0.0795);
        } else {
          red += v[0];
        }
      }
    }
  }
  double s = red;
#pragma unroll
  for (int u = 0; u < TB; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// VAR 5 (k_mut_part): the reverse-sum partial of each step goes to shared memory
// part[ti][j] (no butterfly); every 4 batches (a 256-source chunk: 16 slices x 16 steps) one
// barrier, then each thread sums the MQ partials of 2 sources of the chunk just completed
// and adds them with RED (double-buffered partials: one barrier per chunk)
template <int TB, int MQ = 8>
__global__ void __launch_bounds__(128) k_mut_part(double* out, const double4* __restrict__ src, int ns, int reps,
                                                  double* pot) {
  constexpr int SB = 4, G = 128 / MQ, CHK = 256, PS = CHK + 4;
  __shared__ double4 sb[CHK];
  __shared__ int sidx[CHK];
  __shared__ double part[2][MQ][PS];
  for (int j = threadIdx.x; j < CHK; j += blockDim.x) {
    sb[j] = src[j];
    sidx[j] = (int)(((unsigned)(j + 1) * 2654435761u + blockIdx.x * 40503u) & ((1u << 22) - 1));
  }
  __syncthreads();
  const int ti = threadIdx.x & (MQ - 1), gi = threadIdx.x / MQ;
  double x[TB][3], q[TB], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    x[u][0] = 0.5 + 1e-4 * (ti + 7 * u); x[u][1] = 0.25 + 1e-5 * gi + 3e-6 * u; x[u][2] = -0.125 * u + 1e-7 * ti;
    q[u] = 0.1 * u; acc[u] = 0;
  }
  int pb = 0;
  for (int r = 0; r < reps * (ns / CHK); ++r) {
    double* pw = &part[pb][ti][0];
    for (int j0 = gi; j0 + G * (SB - 1) < CHK; j0 += G * SB) {
#pragma unroll
      for (int t = 0; t < SB; ++t) {
        const double4 sv = sb[j0 + G * t];
        double sj = 0.0;
#pragma unroll
        for (int u = 0; u < TB; ++u) {
          const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
          const double g = rinv(fma(dz, dz, fma(dy, dy, dx * dx)));
          acc[u] = fma(sv.w, g, acc[u]);
          sj = fma(q[u], g, sj);
        }
        pw[j0 + G * t] = sj;
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < CHK; j += blockDim.x) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < MQ; ++t) s += part[pb][t][j];
      atomicAdd(pot + sidx[j], s * 0.0795);
    }
    pb ^= 1;
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < TB; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// VAR 6 (k_mut_lane): the transposed layout — every lane of a warp holds the SAME TB
// targets (the warp's), the lanes take different sources (lane l: sources l, l + 32, ...),
// so a source's reverse sum over the warp's targets is complete in one lane: no
// reduce-scatter.  W warps hold W x TB targets; per 256-source chunk each warp stores its
// per-source partials to shared memory, one barrier, then each thread sums the W partials
// of 2 sources and adds them with RED (double-buffered partials).
template <int TB, int W>
__global__ void __launch_bounds__(W * 32) k_mut_lane(double* out, const double4* __restrict__ src, int ns, int reps,
                                                     double* pot) {
  constexpr int CHK = 256, NTH = W * 32;
  __shared__ double4 sb[CHK];
  __shared__ int sidx[CHK];
  __shared__ double part[2][W][CHK];
  for (int j = threadIdx.x; j < CHK; j += NTH) {
    sb[j] = src[j];
    sidx[j] = (int)(((unsigned)(j + 1) * 2654435761u + blockIdx.x * 40503u) & ((1u << 22) - 1));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double x[TB][3], q[TB], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    x[u][0] = 0.5 + 1e-4 * (w + 7 * u); x[u][1] = 0.25 + 3e-6 * u + 1e-5 * w; x[u][2] = -0.125 * u + 1e-7 * w;
    q[u] = 0.1 * u; acc[u] = 0;
  }
  int pb = 0;
  for (int r = 0; r < reps * (ns / CHK); ++r) {
    double* pw = &part[pb][w][0];
#pragma unroll 2
    for (int j = lane; j < CHK; j += 32) {
      const double4 sv = sb[j];
      double sj = 0.0;
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
        const double g = rinv(fma(dz, dz, fma(dy, dy, dx * dx)));
        acc[u] = fma(sv.w, g, acc[u]);
        sj = fma(q[u], g, sj);
      }
      pw[j] = sj;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < CHK; j += NTH) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) s += part[pb][t][j];
      atomicAdd(pot + sidx[j], s * 0.0795);
    }
    pb ^= 1;
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < TB; ++u) s += acc[u];
  out[blockIdx.x * NTH + threadIdx.x] = s;
}

template <int TB, int W>
void run_lane(double* out, const double4* src, int ns, double* pot) {
  const int reps = 40;
  int per_sm = 0;
  cudaFuncSetAttribute(k_mut_lane<TB, W>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mut_lane<TB, W>, W * 32, 0);
  const int grid = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i < 4; ++i) {
    cudaEventRecord(a);
    k_mut_lane<TB, W><<<grid, W * 32>>>(out, src, ns, reps, pot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  const double pairs = (double)grid * W * TB * 256.0 * (ns / 256) * reps;  // unordered target-source pairs
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double peak = 148.0 * 64 * clk * 1e3;
  printf("{\"TB\": %d, \"W\": %d, \"var\": 6, \"ctas_per_sm\": %d, \"pairs_per_s\": %.4g, \"fp64_instr_frac\": %.3f}\n",
         TB, W, per_sm, pairs / (best * 1e-3), pairs * 13.0 / (best * 1e-3) / peak);
}

template <int TB, int MQ = 8>
void run_part(double* out, const double4* src, int ns, double* pot) {
  const int reps = 40;
  int per_sm = 0;
  cudaFuncSetAttribute(k_mut_part<TB, MQ>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mut_part<TB, MQ>, 128, 0);
  const int grid = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i < 4; ++i) {
    cudaEventRecord(a);
    k_mut_part<TB, MQ><<<grid, 128>>>(out, src, ns, reps, pot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  constexpr int G = 128 / MQ;
  const double pairs = (double)grid * 128 * TB * (256.0 / G) * (ns / 256) * reps;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double peak = 148.0 * 64 * clk * 1e3;
  printf("{\"TB\": %d, \"MQ\": %d, \"var\": 5, \"ctas_per_sm\": %d, \"pairs_per_s\": %.4g, \"fp64_instr_frac\": %.3f}\n",
         TB, MQ, per_sm, pairs / (best * 1e-3), pairs * 13.0 / (best * 1e-3) / peak);
}

template <int TB, int VAR, int MINB, int MQ = 8>
void run(double* out, const double4* src, int ns, double* pot, int pad = 0) {
  const int reps = 40;
  int per_sm = 0;
  // pad: dynamic shared memory that caps the CTAs per SM (k_near runs 4 per SM)
  cudaFuncSetAttribute(k_mut<TB, VAR, MINB, MQ>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_mut<TB, VAR, MINB, MQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mut<TB, VAR, MINB, MQ>, 128, pad);
  const int grid = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i < 4; ++i) {
    cudaEventRecord(a);
    k_mut<TB, VAR, MINB, MQ><<<grid, 128, pad>>>(out, src, ns, reps, pot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  constexpr int SB = 4, G = 128 / MQ;
  const double steps = (double)((ns - G * (SB - 1) + G * SB - 1) / (G * SB)) * SB;  // per thread per rep
  const double pairs = (double)grid * 128 * TB * steps * reps;                     // thread-target-source
  const double instr = pairs * (VAR == 0 ? 12.0 : 13.0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double peak = 148.0 * 64 * clk * 1e3;
  printf("{\"TB\": %d, \"MQ\": %d, \"var\": %d, \"minb\": %d, \"ctas_per_sm\": %d, \"pairs_per_s\": %.4g, \"fp64_instr_frac\": %.3f}\n",
         TB, MQ, VAR, MINB, per_sm, pairs / (best * 1e-3), instr / (best * 1e-3) / peak);
}

int main() {
  const int ns = 1024;
  double4* h = new double4[ns];
  for (int j = 0; j < ns; ++j) h[j] = make_double4(0.01 * (j % 37), 0.02 * (j % 23), 0.03 * (j % 11) + 1.0, 1.0);
  double4* src;
  double* out;
  cudaMalloc(&src, sizeof(double4) * ns);
  cudaMalloc(&out, 64 << 20);
  cudaMemcpy(src, h, sizeof(double4) * ns, cudaMemcpyHostToDevice);
  double* pot;
  cudaMalloc(&pot, sizeof(double) << 22);
  cudaMemset(pot, 0, sizeof(double) << 22);
  run<5, 0, 1>(out, src, ns, pot);
  run<5, 1, 1>(out, src, ns, pot);
  run<5, 2, 1>(out, src, ns, pot);
  run<5, 3, 1>(out, src, ns, pot);
  run<5, 4, 1>(out, src, ns, pot);
  run<5, 2, 1>(out, src, ns, pot, 20 << 10);
  run<5, 3, 1>(out, src, ns, pot, 20 << 10);
  run<5, 4, 1>(out, src, ns, pot, 20 << 10);
  run<8, 4, 1>(out, src, ns, pot);
  run<4, 4, 1>(out, src, ns, pot);
  run_part<5>(out, src, ns, pot);
  run_part<6>(out, src, ns, pot);
  run_part<4>(out, src, ns, pot);
  run_part<5, 4>(out, src, ns, pot);
  run_lane<5, 8>(out, src, ns, pot);
  run_lane<8, 4>(out, src, ns, pot);
  run_lane<8, 5>(out, src, ns, pot);
  run_lane<7, 5>(out, src, ns, pot);
  run_lane<6, 4>(out, src, ns, pot);
  run_lane<4, 4>(out, src, ns, pot);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
