// Development tool (not product, not oracle): an L2 model of the RHS (x) gathers of the pJDS kernel
// on an HMEp-shaped matrix, to rank CTA tile execution orders offline before spending GPU time.
//
// Model: the permuted basis (x stored in sorted-row order, columns = invperm[col]); CTA tile = 1024
// consecutive sorted rows (R = 4 x 256 threads); tiles execute in the given order; each tile's
// distinct x sectors (L1 dedups within a CTA) go to a set-associative LRU cache of C bytes
// (128-byte lines, 32-byte sectors, 16 ways) that stands for the L2 share x keeps next to the
// evict-first val/col stream.  Output: x sector misses -> x DRAM bytes and alpha = x bytes /
// (nnz * 8) (Eq. 1 L333-346 RHS re-load factor), per order and capacity.
//
//   g++ -O3 -march=native -fopenmp -o tools/l2sim tools/l2sim.cpp -ldl
//   tools/l2sim <config M> <ordering> <capacity MB list> <order spec> ...
// order specs: storage | row | pw:<W> (phonon window W, then original row) | ew:<W> (phonon window,
// then e-block in a bandwidth-reducing order, then row) | file:<path> (int32 tile order)
#include <dlfcn.h>
#include <omp.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

typedef void* (*create_t)(int, int, int, int, uint64_t);
typedef int64_t (*n_t)(void*);
typedef int64_t (*rowlen_t)(void*, int64_t, int64_t, int32_t*);
typedef void (*fill_t)(void*, int64_t, int64_t, const int64_t*, int32_t*, void*, int);

struct Cache {
  int64_t nsets;
  static constexpr int W = 16;
  std::vector<int64_t> tag;   // [nsets*W] line id or -1
  std::vector<uint32_t> age;  // LRU stamp
  std::vector<uint8_t> mask;  // sector valid bits
  uint32_t clock = 0;
  int64_t misses = 0;
  explicit Cache(int64_t bytes) {
    nsets = std::max<int64_t>(1, bytes / (128 * W));
    tag.assign(nsets * W, -1);
    age.assign(nsets * W, 0);
    mask.assign(nsets * W, 0);
  }
  void access(int64_t sector) {
    const int64_t line = sector >> 2;
    const int sb = 1 << (sector & 3);
    // hashed set index (hardware L2 hashes addresses over slices)
    uint64_t h = (uint64_t)line * 0x9E3779B97F4A7C15ull;
    const int64_t set = (int64_t)((h >> 20) % (uint64_t)nsets);
    int64_t* t = &tag[set * W];
    uint32_t* a = &age[set * W];
    uint8_t* m = &mask[set * W];
    ++clock;
    int victim = 0;
    for (int w = 0; w < W; ++w) {
      if (t[w] == line) {
        if (!(m[w] & sb)) {
          ++misses;
          m[w] |= sb;
        }
        a[w] = clock;
        return;
      }
      if (a[w] < a[victim]) victim = w;
    }
    ++misses;
    t[victim] = line;
    m[victim] = (uint8_t)sb;
    a[victim] = clock;
  }
};

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: l2sim <M> <ordering 0|1> <capMB,capMB,...> <order spec> [order spec ...]\n");
    return 1;
  }
  const int M = atoi(argv[1]), ordering = atoi(argv[2]);
  std::vector<int64_t> caps;
  for (char* p = strtok(argv[3], ","); p; p = strtok(nullptr, ",")) caps.push_back(atoll(p) << 20);
  void* L = dlopen("inputs/libpjdsgen.so", RTLD_NOW);
  if (!L) { fprintf(stderr, "%s\n", dlerror()); return 1; }
  auto create = (create_t)dlsym(L, "pjdsgen_create");
  auto gn = (n_t)dlsym(L, "pjdsgen_n");
  auto rowlen = (rowlen_t)dlsym(L, "pjdsgen_rowlen");
  auto fill = (fill_t)dlsym(L, "pjdsgen_fill");
  void* g = create(0 /*HMEP*/, M, ordering, 0, 0x11125588ull);
  const int64_t n = gn(g);
  std::vector<int32_t> len(n);
  rowlen(g, 0, n, len.data());
  std::vector<int64_t> rp(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + len[i];
  const int64_t nnz = rp[n];
  std::vector<int32_t> col(nnz);
  {
    const int64_t CH = 1 << 20;
    std::vector<float> vs;
    for (int64_t r0 = 0; r0 < n; r0 += CH) {
      const int64_t r1 = std::min(n, r0 + CH);
      std::vector<int64_t> lrp(r1 - r0 + 1);
      for (int64_t i = r0; i <= r1; ++i) lrp[i - r0] = rp[i] - rp[r0];
      vs.resize(lrp.back());
      fill(g, r0, r1, lrp.data(), col.data() + rp[r0], vs.data(), 0);
    }
  }
  // stable descending sort by length: perm[new] = old
  int32_t maxlen = *std::max_element(len.begin(), len.end());
  std::vector<int64_t> cnt(maxlen + 2, 0);
  for (int64_t i = 0; i < n; ++i) cnt[maxlen - len[i] + 1]++;
  for (int k = 1; k <= maxlen + 1; ++k) cnt[k] += cnt[k - 1];
  std::vector<int32_t> perm(n), inv(n);
  for (int64_t i = 0; i < n; ++i) perm[cnt[maxlen - len[i]]++] = (int32_t)i;
  for (int64_t k = 0; k < n; ++k) inv[perm[k]] = (int32_t)k;
  const int64_t TR = getenv("L2SIM_TILE") ? atoll(getenv("L2SIM_TILE")) : 1024, ntiles = (n + TR - 1) / TR;
  const int64_t GROUP = getenv("L2SIM_GROUP") ? atoll(getenv("L2SIM_GROUP")) : 1;  // tiles per L1 dedup unit
  // P (rows per e-block) from the generator's structure: the HMEp phonon count C(M+5,5)
  int64_t P = 1;
  for (int k = 1; k <= 5; ++k) P = P * (M + k) / k;
  fprintf(stderr, "n=%ld nnz=%ld tiles=%ld P=%ld\n", (long)n, (long)nnz, (long)ntiles, (long)P);

  for (int a = 4; a < argc; ++a) {
    std::string spec = argv[a];
    std::vector<int64_t> key(ntiles);
    std::vector<int32_t> order(ntiles);
    std::iota(order.begin(), order.end(), 0);
    if (spec == "storage") {
      for (int64_t t = 0; t < ntiles; ++t) key[t] = t;
    } else if (spec == "row") {
      for (int64_t t = 0; t < ntiles; ++t) key[t] = perm[t * TR];
    } else if (spec.rfind("pw:", 0) == 0) {
      const int64_t W = atoll(spec.c_str() + 3);
      for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t r = perm[t * TR];
        key[t] = ((r % P) / W) * n + r;
      }
    } else if (spec.rfind("file:", 0) == 0) {
      FILE* f = fopen(spec.c_str() + 5, "rb");
      if (!f || (int64_t)fread(order.data(), 4, ntiles, f) != ntiles) { fprintf(stderr, "bad order file\n"); return 1; }
      fclose(f);
      for (int64_t t = 0; t < ntiles; ++t) key[order[t]] = t;
    } else {
      fprintf(stderr, "unknown spec %s\n", spec.c_str());
      continue;
    }
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    for (int64_t cap : caps) {
      Cache c(cap);
      std::vector<int64_t> secs;
      int64_t l1_sectors = 0;
      for (int64_t oi0 = 0; oi0 < ntiles; oi0 += GROUP) {
        secs.clear();
        for (int64_t oi = oi0; oi < std::min(ntiles, oi0 + GROUP); ++oi) {
          const int64_t t = order[oi];
          for (int64_t k = t * TR; k < std::min(n, (t + 1) * TR); ++k) {
            const int32_t r = perm[k];
            for (int64_t q = rp[r]; q < rp[r + 1]; ++q) secs.push_back(((int64_t)inv[col[q]] * 8) >> 5);
          }
        }
        std::sort(secs.begin(), secs.end());
        secs.erase(std::unique(secs.begin(), secs.end()), secs.end());
        l1_sectors += (int64_t)secs.size();
        for (int64_t s : secs) c.access(s);
      }
      const double xbytes = c.misses * 32.0;
      printf("{\"spec\": \"%s\", \"tile\": %ld, \"group\": %ld, \"cap_mb\": %ld, \"x_dram_gb\": %.4f, \"alpha\": %.4f, "
             "\"loads_per_x\": %.3f, \"l2_x_requests_gb\": %.3f}\n",
             spec.c_str(), (long)TR, (long)GROUP, (long)(cap >> 20), xbytes / 1e9, xbytes / (nnz * 8.0),
             xbytes / (n * 8.0), l1_sectors * 32.0 / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}
