// Pair-evaluation rate limits on B200 (sm_100a): MUFU.RSQ64H throughput, and the
// k_eval inner loop (4 targets per thread, sources broadcast from shared memory)
// with three FP64 reciprocal-square-root schemes:
//   rsq64h : MUFU.RSQ64H seed + one 3rd-order correction (5 FP64 ops, the production path)
//   f32seed: MUFU.RSQ (fp32) seed on float(r2) + one 3rd-order correction in FP64
//   iseed  : integer "magic" seed + 3rd-order corrections (no MUFU)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_rates pair_rates.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ double rsq_approx(double x) {
  double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y;
}
__device__ __forceinline__ double refine3(double r2, double y0) {
  double t = r2 * y0, e = fma(-t, y0, 1.0), p = fma(e, 0.375, 0.5), h = y0 * e;
  return fma(h, p, y0);
}

// MUFU.RSQ64H alone: 8 independent chains, each step one MUFU + one DADD
__global__ void k_mufu64(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = rsq_approx(x[i]) + 2.0;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
__device__ __forceinline__ double rinv(double r2) {
  if (MODE == 0) return refine3(r2, rsq_approx(r2));
  if (MODE == 1) {
    float f = __double2float_rn(r2);
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f));
    return refine3(r2, (double)y);
  }
  // integer seed (max rel err ~3.4%), two 3rd-order corrections -> ~1e-13, a third -> full
  long long i = __double_as_longlong(r2);
  double y = __longlong_as_double(0x5fe6eb50c7b537a9LL - (i >> 1));
  y = refine3(r2, y);
  y = refine3(r2, y);
  return refine3(r2, y);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_pairs(double* out, const double4* __restrict__ src, int ns, int reps) {
  __shared__ double4 sb[1024];
  for (int j = threadIdx.x; j < ns; j += blockDim.x) sb[j] = src[j];
  __syncthreads();
  double x[4][3], acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    x[u][0] = 0.5 + 1e-4 * (threadIdx.x + 7 * u); x[u][1] = 0.25; x[u][2] = -0.125 * u; acc[u] = 0;
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < ns; ++j) {
      const double4 sv = sb[j];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double dx = x[u][0] - sv.x, dy = x[u][1] - sv.y, dz = x[u][2] - sv.z;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        acc[u] = fma(sv.w, rinv<MODE>(r2), acc[u]);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * (1 << 24)));
  const int ns = 1024, reps = 8;
  double4* src; CK(cudaMalloc(&src, sizeof(double4) * ns));
  double4* hs = new double4[ns];
  for (int j = 0; j < ns; ++j) hs[j] = make_double4(0.1 + j * 1e-3, 0.2 + 1e-5 * j, 0.3 + j * 1e-4, 1.0 - 1e-3 * j);
  CK(cudaMemcpy(src, hs, sizeof(double4) * ns, cudaMemcpyHostToDevice));
  printf("{\"sms\": %d", sms);
  for (int bps : {4, 8}) {
    const int blocks = sms * bps, threads = 256, iters = 4096;
    float ms = time_it([&] { k_mufu64<<<blocks, threads>>>(out, iters); });
    printf(", \"mufu_rsq64h_per_clk_per_sm_b%d\": %.3f", bps,
           (double)blocks * threads * iters * 8 / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
    ms = time_it([&] { k_pairs<0><<<blocks, threads>>>(out, src, ns, reps); });
    const double pairs = (double)blocks * threads * 4 * ns * reps;
    printf(", \"pairs_rsq64h_b%d\": %.4e", bps, pairs / (ms * 1e-3));
    ms = time_it([&] { k_pairs<1><<<blocks, threads>>>(out, src, ns, reps); });
    printf(", \"pairs_f32seed_b%d\": %.4e", bps, pairs / (ms * 1e-3));
    ms = time_it([&] { k_pairs<2><<<blocks, threads>>>(out, src, ns, reps); });
    printf(", \"pairs_iseed_b%d\": %.4e", bps, pairs / (ms * 1e-3));
  }
  printf(", \"clock_khz\": %d}\n", prop.clockRate);
  CK(cudaGetLastError());
  return 0;
}
