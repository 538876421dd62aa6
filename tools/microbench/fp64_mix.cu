// Do DFMA (fp64 pipe) and DMMA (tensor pipe) share throughput on B200?
// Half the warps of every CTA run a DFMA loop, the other half a DMMA loop.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 4096;
__global__ void k_mix(double* out, double a, double b, int mode) {
  int warp = threadIdx.x >> 5;
  bool do_mma = mode == 1 || (mode == 2 && (warp & 1));
  double s = 0;
  if (do_mma) {
    double c[4][2] = {};
    double av = a + threadIdx.x, bv = b;
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(av), "d"(bv));
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  } else {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    for (int j = 0; j < 8; ++j) s += x[j];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256;
  const char* names[3] = {"dfma_only", "dmma_only", "half_half"};
  printf("{");
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); k_mix<<<blocks, threads>>>(out, 1.0000001, 1e-9, mode); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    double warps = (double)blocks * threads / 32;
    double fl_fma = warps * 32 * IT * 8 * 2, fl_mma = warps * IT * 4 * 512.0;
    double fl = mode == 0 ? fl_fma : mode == 1 ? fl_mma : 0.5 * (fl_fma + fl_mma);
    printf("%s\"%s_ms\": %.3f, \"%s_tflops\": %.2f", mode ? ", " : "", names[mode], best, names[mode], fl / (best * 1e-3) / 1e12);
  }
  printf("}\n");
}
