// Host-code sanitizer driver (host code under -fsanitize=address,undefined).
// Builds the library's HOST-ONLY parts (partition.cpp, precompute.cpp, tables_io.cpp) from source with
// AddressSanitizer + UBSan and exercises them:
//   * build_partition for nranks 1, 2, 3, 5, 8 and every rank on a tree + lists read
//     from a binary dump (written by tests/test_native_asan.py from the oracle),
//     checking that what rank s sends to r is what r expects from s;
//   * build_tables (p = 4, k = 24), the operator-table file round trip (tables_io.cpp) and
//     build_stage2 (C2 = 1).
// Usage: asan_host dump.bin [table_file]   (exit 0 = clean)
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../paper_1211_2517_b200/csrc/fmm_internal.h"

namespace kifmm {
static std::string g_err;
void set_error(const std::string& m) { g_err = m; }
const char* last_error() { return g_err.c_str(); }
}  // namespace kifmm

using namespace kifmm;

template <typename T>
static bool rd(FILE* f, std::vector<T>& v, size_t n) {
  v.resize(n);
  return n == 0 || std::fread(v.data(), sizeof(T), n, f) == n;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t hdr[5];  // nboxes, nU, nV, nW, nX
  if (std::fread(hdr, sizeof(int64_t), 5, f) != 5) return 2;
  const int nb = (int)hdr[0];
  std::vector<int> level, parent, pbeg, pend, U, V, W, X;
  std::vector<uint8_t> leaf;
  if (!rd(f, level, nb) || !rd(f, parent, nb) || !rd(f, pbeg, nb) || !rd(f, pend, nb) || !rd(f, leaf, nb) ||
      !rd(f, U, 2 * hdr[1]) || !rd(f, V, 3 * hdr[2]) || !rd(f, W, 3 * hdr[3]) || !rd(f, X, 3 * hdr[4]))
    return 2;
  std::fclose(f);
  PartitionInput in;
  in.nboxes = nb;
  in.level = level.data(); in.parent = parent.data(); in.pbeg = pbeg.data(); in.pend = pend.data();
  in.leaf = leaf.data();
  in.nU = hdr[1]; in.U = U.data(); in.ustride = 2;
  in.nV = hdr[2]; in.V = V.data(); in.vstride = 3;
  in.nW = hdr[3]; in.W = W.data(); in.wstride = 3;
  in.nX = hdr[4]; in.X = X.data(); in.xstride = 3;
  in.n = 56; in.k = 25;
  for (int R : {1, 2, 3, 5, 8}) {
    std::vector<DistPlan> D(R);
    for (int r = 0; r < R; ++r)
      if (build_partition(in, R, r, &D[r])) { std::fprintf(stderr, "partition failed\n"); return 1; }
    for (int r = 0; r < R && R > 1; ++r)
      for (int s = 0; s < R; ++s) {
        if (r == s) continue;
        const int qs = D[s].q_send_off[r + 1] - D[s].q_send_off[r], qr = D[r].q_recv_off[s + 1] - D[r].q_recv_off[s];
        const int ds = D[s].d_send_off[r + 1] - D[s].d_send_off[r], dr = D[r].d_recv_off[s + 1] - D[r].d_recv_off[s];
        if (qs != qr || ds != dr) { std::fprintf(stderr, "inconsistent lists R=%d r=%d s=%d\n", R, r, s); return 1; }
      }
  }
  HostTables H;
  if (build_tables(4, 24, 0.1, 1e-10, &H) || H.k != 25) { std::fprintf(stderr, "tables failed\n"); return 1; }
  // the operator-table file: write, read back bit for bit, refuse a corrupted copy
  if (argc > 2) {
    const std::string path = argv[2];
    if (save_tables(H, 24, path)) { std::fprintf(stderr, "save failed\n"); return 1; }
    HostTables L;
    int kr = 0;
    if (load_tables(path, &L, &kr) || kr != 24 || L.C != H.C || L.U != H.U || L.S != H.S || L.T != H.T ||
        L.M != H.M || L.L != H.L || L.sigma != H.sigma || L.surf != H.surf) {
      std::fprintf(stderr, "table file round trip failed\n");
      return 1;
    }
    FILE* f = std::fopen(path.c_str(), "r+b");
    std::fseek(f, 200, SEEK_SET);
    std::fputc(0x5a, f);
    std::fclose(f);
    if (load_tables(path, &L, &kr) != -1) { std::fprintf(stderr, "corrupt table file accepted\n"); return 1; }
  }
  if (build_stage2(H, 1.0) || (int)H.ranks.size() != 316) { std::fprintf(stderr, "stage2 failed\n"); return 1; }
  std::printf("asan host driver ok\n");
  return 0;
}
