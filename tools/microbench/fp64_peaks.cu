// FP64 roofline denominators on B200 (sm_100a): DFMA, DMMA (mma.sync .f64 shapes),
// fp64 rsqrt paths, and red.global.add.f64 throughput into an L2-resident array.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
// Prints one JSON object.  Timing: CUDA events, best of 5 after 2 warm-ups.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// m8n8k4: A 1 reg, B 1 reg, C 2 regs
__global__ void k_dmma_m8n8k4(double* out, double a, double b) {
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = 0; c[j][1] = 0; }
  double av = a + threadIdx.x, bv = b;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma_m16n8k4(double* out, double a, double b) {
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) for (int t = 0; t < 4; ++t) c[j][t] = 0;
  double a0 = a + threadIdx.x, a1 = a0 + 1, bv = b;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma_m16n8k8(double* out, double a, double b) {
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) for (int t = 0; t < 4; ++t) c[j][t] = 0;
  double a0 = a + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = b, b1 = b + 1;
  for (int i = 0; i < ITERS / 2; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma_m16n8k16(double* out, double a, double b) {
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) for (int t = 0; t < 4; ++t) c[j][t] = 0;
  double av[8], bv[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) av[t] = a + threadIdx.x + t;
#pragma unroll
  for (int t = 0; t < 4; ++t) bv[t] = b + t;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(av[0]), "d"(av[1]), "d"(av[2]), "d"(av[3]), "d"(av[4]), "d"(av[5]), "d"(av[6]), "d"(av[7]),
                     "d"(bv[0]), "d"(bv[1]), "d"(bv[2]), "d"(bv[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// pair-interaction style loop: 4 independent chains of (diff, r2, rsqrt(lib), fma)
__global__ void k_pair_lib(double* out, const double4* __restrict__ src, int ns) {
  double x = threadIdx.x * 1e-3, y = 0.5, z = 0.25, acc = 0;
  for (int it = 0; it < 16; ++it)
    for (int j = 0; j < ns; ++j) {
      double4 s = src[j];
      double dx = x - s.x, dy = y - s.y, dz = z - s.z;
      double r2 = dx * dx + dy * dy + dz * dz;
      acc = fma(s.w, rsqrt(r2), acc);
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__device__ __forceinline__ double rsqrt_nr(double r2) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  double t = r2 * y0;
  double e = fma(-t, y0, 1.0);
  double p = fma(e, 0.375, 0.5);
  double h = y0 * e;
  return fma(h, p, y0);
}

__global__ void k_pair_nr(double* out, const double4* __restrict__ src, int ns) {
  double x = threadIdx.x * 1e-3, y = 0.5, z = 0.25, acc = 0;
  for (int it = 0; it < 16; ++it)
    for (int j = 0; j < ns; ++j) {
      double4 s = src[j];
      double dx = x - s.x, dy = y - s.y, dz = z - s.z;
      double r2 = dx * dx + dy * dy + dz * dz;
      acc = fma(s.w, rsqrt_nr(r2), acc);
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// scattered fp64 reductions into an array of `len` doubles (fits L2)
__global__ void k_red(double* arr, uint32_t len, int per_thread) {
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < per_thread; ++i) {
    h = h * 1664525u + 1013904223u;
    atomicAdd(arr + (h % len), 1.0);
  }
}
// coalesced-row fp64 reductions: a warp adds 32 consecutive doubles of a random row of 64
__global__ void k_red_rows(double* arr, uint32_t nrows, int per_warp) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  uint32_t h = w * 2654435761u;
  for (int i = 0; i < per_warp; ++i) {
    h = h * 1664525u + 1013904223u;
    uint32_t row = h % nrows;
    atomicAdd(arr + (size_t)row * 64 + lane, 1.0);
    atomicAdd(arr + (size_t)row * 64 + 32 + lane, 1.0);
  }
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
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * 64 * 1024 * 1024));
  int blocks = sms * 8, threads = 256;
  double nthreads = (double)blocks * threads;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", prop.name, sms, prop.clockRate);
  float ms = time_it([&] { k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-9); });
  printf(", \"dfma_tflops\": %.2f", nthreads * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_dmma_m8n8k4<<<blocks, threads>>>(out, 1e-3, 1e-3); });
  printf(", \"dmma_m8n8k4_tflops\": %.2f", nthreads / 32 * ITERS * 4 * (8 * 8 * 4 * 2) / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_dmma_m16n8k4<<<blocks, threads>>>(out, 1e-3, 1e-3); });
  printf(", \"dmma_m16n8k4_tflops\": %.2f", nthreads / 32 * ITERS * 4 * (16 * 8 * 4 * 2) / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_dmma_m16n8k8<<<blocks, threads>>>(out, 1e-3, 1e-3); });
  printf(", \"dmma_m16n8k8_tflops\": %.2f", nthreads / 32 * (ITERS / 2) * 4 * (16 * 8 * 8 * 2) / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_dmma_m16n8k16<<<blocks, threads>>>(out, 1e-3, 1e-3); });
  printf(", \"dmma_m16n8k16_tflops\": %.2f", nthreads / 32 * (ITERS / 4) * 4 * (16 * 8 * 16 * 2) / (ms * 1e-3) / 1e12);
  // pair loops
  int ns = 1024;
  double4* src; CK(cudaMalloc(&src, sizeof(double4) * ns));
  double4* hs = new double4[ns];
  for (int j = 0; j < ns; ++j) hs[j] = make_double4(0.1 + j * 1e-3, 0.2, 0.3 + j * 1e-4, 1.0);
  CK(cudaMemcpy(src, hs, sizeof(double4) * ns, cudaMemcpyHostToDevice));
  ms = time_it([&] { k_pair_lib<<<blocks, threads>>>(out, src, ns); });
  printf(", \"pairs_per_s_lib_rsqrt\": %.4e", nthreads * 16 * ns / (ms * 1e-3));
  ms = time_it([&] { k_pair_nr<<<blocks, threads>>>(out, src, ns); });
  printf(", \"pairs_per_s_nr_rsqrt\": %.4e", nthreads * 16 * ns / (ms * 1e-3));
  // atomics
  uint32_t len = 4u << 20;  // 32 MB of doubles: L2 resident
  CK(cudaMemset(out, 0, sizeof(double) * len));
  int per = 256;
  ms = time_it([&] { k_red<<<blocks, threads>>>(out, len, per); });
  printf(", \"red_f64_scattered_per_s\": %.4e", nthreads * per / (ms * 1e-3));
  ms = time_it([&] { k_red_rows<<<blocks, threads>>>(out, len / 64, per); });
  printf(", \"red_f64_rows_per_s\": %.4e", nthreads * per * 2 / (ms * 1e-3));
  // HBM copy for reference
  size_t nb = 1ull << 28;  // 256M doubles? too big; use 2 GB buffers
  double *a2, *b2; CK(cudaMalloc(&a2, nb * 8)); CK(cudaMalloc(&b2, nb * 8));
  ms = time_it([&] { cudaMemcpyAsync(b2, a2, nb * 8, cudaMemcpyDeviceToDevice); });
  printf(", \"d2d_copy_gbs\": %.1f", 2.0 * nb * 8 / (ms * 1e-3) / 1e9);
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
