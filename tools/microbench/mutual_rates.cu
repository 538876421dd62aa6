// Issue-rate limits of the mutual near-field pair loop (k_near's inner batch) on B200:
// TB targets per thread in registers, sources broadcast from shared memory per slice of MQ
// lanes, each source step accumulating both the targets' sums and the source's reverse sum
// s_j = sum_u q_u G(x_u, y_j).  Variants (FP64 instructions per unordered pair in brackets):
//   0 one-sided                (12)  acc_u += w_j G
//   1 mutual, no reduction     (13)  + s_j, kept in a register
//   2 mutual + butterfly       (13)  + the SB = 4 reduce-scatter over MQ = 8 lanes per 4 steps
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
__global__ void __launch_bounds__(128, MINB) k_mut(double* out, const double4* __restrict__ src, int ns, int reps) {
  constexpr int SB = 4, G = 128 / MQ;
  __shared__ double4 sb[1024];
  for (int j = threadIdx.x; j < ns; j += blockDim.x) sb[j] = src[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, ti = threadIdx.x & (MQ - 1), gi = threadIdx.x / MQ;
  double x[TB][3], q[TB], acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    x[u][0] = 0.5 + 1e-4 * (ti + 7 * u); x[u][1] = 0.25 + 1e-5 * gi; x[u][2] = -0.125 * u; q[u] = 0.1 * u; acc[u] = 0;
  }
  double red = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (int j0 = gi; j0 + G * (SB - 1) < ns; j0 += G * SB) {
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
      if (VAR == 2) {
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
        red += v[0];
      }
    }
  }
  double s = red;
#pragma unroll
  for (int u = 0; u < TB; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int TB, int VAR, int MINB, int MQ = 8>
void run(double* out, const double4* src, int ns) {
  const int reps = 40;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mut<TB, VAR, MINB, MQ>, 128, 0);
  const int grid = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i < 4; ++i) {
    cudaEventRecord(a);
    k_mut<TB, VAR, MINB, MQ><<<grid, 128>>>(out, src, ns, reps);
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
  run<5, 2, 1>(out, src, ns);
  run<8, 2, 1>(out, src, ns);
  run<4, 2, 1, 4>(out, src, ns);
  run<6, 2, 1, 4>(out, src, ns);
  run<8, 2, 1, 4>(out, src, ns);
  run<10, 2, 1, 4>(out, src, ns);
  run<12, 2, 1, 4>(out, src, ns);
  run<10, 2, 2, 4>(out, src, ns);
  run<12, 2, 2, 4>(out, src, ns);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
