// Throughput of scattering 512-byte FP64 rows (64 doubles) into an L2-resident
// array: (a) per-lane RED.F64 (warp covers a row in 2 instructions),
// (b) TMA bulk reduction cp.reduce.async.bulk .add.f64 (UBLKRED) from shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_red_rows(double* arr, uint32_t nrows, int rows_per_warp) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  uint32_t h = w * 2654435761u + 12345u;
  for (int i = 0; i < rows_per_warp; ++i) {
    h = h * 1664525u + 1013904223u;
    double* r = arr + (size_t)(h % nrows) * 64;
    atomicAdd(r + lane, 1.0);
    atomicAdd(r + 32 + lane, 1.0);
  }
}

__global__ void k_bulk_rows(double* arr, uint32_t nrows, int rows_per_cta) {
  __shared__ __align__(128) double s[8][64];
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) (&s[0][0])[i] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 8) {
    uint32_t h = (blockIdx.x * 8 + threadIdx.x) * 2654435761u + 777u;
    unsigned sa = (unsigned)__cvta_generic_to_shared(&s[threadIdx.x][0]);
    for (int i = 0; i < rows_per_cta / 8; ++i) {
      h = h * 1664525u + 1013904223u;
      double* r = arr + (size_t)(h % nrows) * 64;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 512;" :: "l"(r), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  uint32_t nrows = 37449;
  double* arr;
  cudaMalloc(&arr, sizeof(double) * 64 * nrows);
  cudaMemset(arr, 0, sizeof(double) * 64 * nrows);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = 148 * 8, threads = 256, rpw = 64;
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); k_red_rows<<<blocks, threads>>>(arr, nrows, rpw); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
  }
  double rows = (double)blocks * threads / 32 * rpw;
  printf("{\"red_rows_per_s\": %.4e, \"red_doubles_per_s\": %.4e", rows / (best * 1e-3), rows * 64 / (best * 1e-3));
  best = 1e30f;
  int rpc = 512;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); k_bulk_rows<<<blocks, threads>>>(arr, nrows, rpc); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
  }
  rows = (double)blocks * rpc;
  printf(", \"ublkred_rows_per_s\": %.4e, \"ublkred_doubles_per_s\": %.4e, \"err\": \"%s\"}\n", rows / (best * 1e-3), rows * 64 / (best * 1e-3),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
