// Operator-table file (the one persisted artifact; it caches the host
// precompute and carries parity between runs).  Versioned little-endian binary:
//   magic "KIFMMTB\0", u32 version (1), u32 byte-order mark 0x01020304,
//   i32 p, n, k (k_eff), k_req (the requested k), f64 d, rcond,
//   8 arrays as (u64 count, count x f64): sigma (n), surf (3n), U (n k), C (316 k k),
//   S (k n), T (n k), M (8 k k), L (8 k k),
//   u64 FNV-1a hash of every array byte (corruption check).
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fmm_internal.h"

namespace kifmm {

namespace {

constexpr char kMagic[8] = {'K', 'I', 'F', 'M', 'M', 'T', 'B', '\0'};
constexpr uint32_t kVersion = 1, kBom = 0x01020304u;

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

}  // namespace

// Written to a temporary file unique to this process and call, then renamed over `path`
// (rename is atomic): several ranks that compute the same tables at once each publish a
// complete file, and the last rename wins.
int save_tables(const HostTables& H, int k_req, const std::string& path) {
  static std::atomic<unsigned> serial{0};
  const std::string tmp = path + ".tmp." + std::to_string((long)getpid()) + "." + std::to_string(serial++);
  File fl;
  fl.f = std::fopen(tmp.c_str(), "wb");
  if (!fl.f) {
    set_error("operator file: cannot write " + tmp);
    return -1;
  }
  const int32_t hdr[4] = {H.p, H.n, H.k, k_req};
  const double dd[2] = {H.d, H.rcond};
  bool ok = std::fwrite(kMagic, 1, 8, fl.f) == 8 && std::fwrite(&kVersion, 4, 1, fl.f) == 1 &&
            std::fwrite(&kBom, 4, 1, fl.f) == 1 && std::fwrite(hdr, 4, 4, fl.f) == 4 && std::fwrite(dd, 8, 2, fl.f) == 2;
  uint64_t h = 1469598103934665603ull;
  const std::vector<double>* arrs[8] = {&H.sigma, &H.surf, &H.U, &H.C, &H.S, &H.T, &H.M, &H.L};
  for (const auto* a : arrs) {
    const uint64_t cnt = a->size();
    ok = ok && std::fwrite(&cnt, 8, 1, fl.f) == 1 && (cnt == 0 || std::fwrite(a->data(), 8, cnt, fl.f) == cnt);
    h = fnv1a(h, a->data(), cnt * 8);
  }
  ok = ok && std::fwrite(&h, 8, 1, fl.f) == 1;
  ok = std::fclose(fl.f) == 0 && ok;
  fl.f = nullptr;
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    set_error("operator file: writing " + path + " failed");
    return -1;
  }
  return 0;
}

// 0: loaded; 1: no such file; -1: unreadable / corrupt / wrong version (error set)
int load_tables(const std::string& path, HostTables* H, int* k_req) {
  File fl;
  fl.f = std::fopen(path.c_str(), "rb");
  if (!fl.f) return 1;
  char magic[8];
  uint32_t ver = 0, bom = 0;
  int32_t hdr[4];
  double dd[2];
  if (std::fread(magic, 1, 8, fl.f) != 8 || std::memcmp(magic, kMagic, 8) != 0 || std::fread(&ver, 4, 1, fl.f) != 1 ||
      std::fread(&bom, 4, 1, fl.f) != 1) {
    set_error("operator file: " + path + " is not a KIFMM table file");
    return -1;
  }
  if (ver != kVersion || bom != kBom) {
    set_error("operator file: " + path + " has version " + std::to_string(ver) + " / byte order " +
              std::to_string(bom) + " (expected " + std::to_string(kVersion) + ", little-endian)");
    return -1;
  }
  // the header must describe tables this library builds (2 <= p <= 8, n = 6(p-1)^2 + 2,
  // 1 <= k <= n): array sizes are derived from it, so a corrupt header is refused
  // before anything is allocated
  if (std::fread(hdr, 4, 4, fl.f) != 4 || std::fread(dd, 8, 2, fl.f) != 2 || hdr[0] < 2 || hdr[0] > 8 ||
      hdr[1] != 6 * (hdr[0] - 1) * (hdr[0] - 1) + 2 || hdr[2] < 1 || hdr[2] > hdr[1] || hdr[3] < 1 ||
      hdr[3] > hdr[1]) {
    set_error("operator file: " + path + " has a corrupt header");
    return -1;
  }
  HostTables T;
  T.p = hdr[0]; T.n = hdr[1]; T.k = hdr[2]; T.d = dd[0]; T.rcond = dd[1];
  const uint64_t n = T.n, k = T.k;
  const uint64_t expect[8] = {n, 3 * n, n * k, 316 * k * k, k * n, n * k, 8 * k * k, 8 * k * k};
  std::vector<double>* arrs[8] = {&T.sigma, &T.surf, &T.U, &T.C, &T.S, &T.T, &T.M, &T.L};
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < 8; ++i) {
    uint64_t cnt = 0;
    if (std::fread(&cnt, 8, 1, fl.f) != 1 || cnt != expect[i]) {
      set_error("operator file: " + path + ": array " + std::to_string(i) + " has the wrong size");
      return -1;
    }
    arrs[i]->resize(cnt);
    if (std::fread(arrs[i]->data(), 8, cnt, fl.f) != cnt) {
      set_error("operator file: " + path + " is truncated");
      return -1;
    }
    h = fnv1a(h, arrs[i]->data(), cnt * 8);
  }
  uint64_t hf = 0;
  if (std::fread(&hf, 8, 1, fl.f) != 1 || hf != h) {
    set_error("operator file: " + path + " fails its checksum");
    return -1;
  }
  *H = std::move(T);
  if (k_req) *k_req = hdr[3];
  return 0;
}

}  // namespace kifmm
