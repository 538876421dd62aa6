// Structure costs of the production k_near (csrc/near.cu, included as is) on synthetic work
// units: which part of the gap between the isolated mutual pair loop (mutual_rates.cu,
// 74% of the FP64 instruction rate at TB = 5, MQ = 8 with the butterfly, RED and chunk
// barrier) and the kernel on C4 (~68% FP64 pipe) comes
// from the unit structure (chunks per unit, chunk fill, the checked own-point and
// one-sided regions, target padding) rather than from the data.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_1211_2517_b200/csrc -o near_struct near_struct.cu \
//        -L../../paper_1211_2517_b200 -lkifmm_b200 -Xlinker -rpath=$PWD/../../paper_1211_2517_b200
#include <cstdio>
#include <random>
#include <vector>

#include "near.cu"

using namespace kifmm;

struct Shape {
  const char* name;
  int tgt;       // targets per unit (capacity 40)
  int nchunk;    // chunks per unit
  int own;       // checked own points at the start of the first chunk
  int mutual;    // mutual sources per chunk (after own)
  int onesided;  // one-sided sources per chunk (after mutual)
};

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  g_num_sms = prop.multiProcessorCount;
  const Shape shapes[] = {
      {"ideal: 40 tgt, 4 x 512 mutual", 40, 4, 0, 512, 0},
      {"40 tgt, 1 x 512 mutual", 40, 1, 0, 512, 0},
      {"40 tgt, 1 x 256 mutual", 40, 1, 0, 256, 0},
      {"40 tgt, 1 x 128 mutual", 40, 1, 0, 128, 0},
      {"40 tgt, 1 x 256 one-sided", 40, 1, 0, 0, 256},
      {"40 tgt, own 40 + 256 mutual", 40, 1, 40, 256, 0},
      {"40 tgt, own 40 + 224 mutual + 32 one-sided", 40, 1, 40, 224, 32},
      {"35 tgt, own 35 + 224 mutual + 32 one-sided", 35, 1, 35, 224, 32},
      {"35 tgt, 2 chunks: own 35 + 224 mut + 32 one", 35, 2, 35, 224, 32},
  };
  const int units = 148 * 4 * 48;
  const int npool = 1 << 22;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  // points: [0, units * 40) targets (unit u: its own block), then a pool of sources
  std::vector<double4> pts((size_t)units * 40 + npool);
  for (auto& p : pts) p = make_double4(U(rng), U(rng), U(rng), U(rng) - 0.5);
  double4* d_pts;
  double* d_out;
  int* d_counter;
  cudaMalloc(&d_pts, sizeof(double4) * pts.size());
  cudaMalloc(&d_out, sizeof(double) * pts.size());
  cudaMalloc(&d_counter, sizeof(int));
  cudaMemcpy(d_pts, pts.data(), sizeof(double4) * pts.size(), cudaMemcpyHostToDevice);
  int per_sm = 0;
  cudaFuncSetAttribute(k_near<5, 8, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_near<5, 8, false>, NR_NT, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double lane_peak = (double)g_num_sms * 64 * clk * 1e3;  // FP64 instruction-lanes / s
  std::printf("{\"ctas_per_sm\": %d, \"units\": %d}\n", per_sm, units);
  for (const Shape& s : shapes) {
    std::vector<int4> items(units), chunks;
    std::vector<int> src;
    double fp64 = 0.0, pairs = 0.0;
    for (int u = 0; u < units; ++u) {
      const int t0 = u * 40;
      const int c0 = (int)chunks.size();
      for (int c = 0; c < s.nchunk; ++c) {
        const int first = (int)src.size();
        int n = 0, nchk = 0;
        if (c == 0)
          for (int j = 0; j < s.own; ++j) src.push_back(t0 + j), ++n;
        nchk = n;
        const int ml = n;
        for (int j = 0; j < s.mutual; ++j) src.push_back(units * 40 + (int)(rng() % npool)), ++n;
        const int mh = n;
        for (int j = 0; j < s.onesided; ++j) src.push_back(units * 40 + (int)(rng() % npool)), ++n;
        chunks.push_back(make_int4(first, n | (nchk << 10) | (ml << 20), mh, 0));
        // FP64 instructions (per thread-lane) the pairs need: one-sided 12, mutual 13 per pair
        const double m = (double)s.tgt;
        fp64 += m * (12.0 * (n - (mh - ml)) + 13.0 * (mh - ml));
        pairs += m * n + m * (mh - ml);
      }
      items[u] = make_int4(t0, s.tgt, c0, c0 + s.nchunk);
    }
    int4 *d_items, *d_chunks;
    int* d_src;
    cudaMalloc(&d_items, sizeof(int4) * items.size());
    cudaMalloc(&d_chunks, sizeof(int4) * chunks.size());
    cudaMalloc(&d_src, sizeof(int) * src.size());
    cudaMemcpy(d_items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_chunks, chunks.data(), sizeof(int4) * chunks.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_src, src.data(), sizeof(int) * src.size(), cudaMemcpyHostToDevice);
    NearArgs a;
    a.items = d_items;
    a.nitems = units;
    a.chunks = d_chunks;
    a.src = d_src;
    a.pts = d_pts;
    a.out = d_out;
    a.nrm = nullptr;
    a.counter = d_counter;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaMemsetAsync(d_counter, 0, sizeof(int));
      cudaEventRecord(e0);
      k_near<5, 8, false><<<std::min(units, per_sm * g_num_sms), NR_NT>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    std::printf("{\"shape\": \"%s\", \"ms\": %.4f, \"pairs_per_s\": %.4g, \"fp64_alg_frac\": %.3f, \"status\": \"%s\"}\n",
                s.name, best, pairs / (best * 1e-3), fp64 / (best * 1e-3) / lane_peak,
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(d_items);
    cudaFree(d_chunks);
    cudaFree(d_src);
  }
  return 0;
}
