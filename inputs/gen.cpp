// Seeded synthetic input generators for the pJDS hot path (test / bench infrastructure).
//
// This module holds NONE of the method's arithmetic: it only produces CRS matrices
// (row pointer, column index, value) and dense vectors whose shapes follow the paper's
// workload descriptions.  Both the oracle (oracle/) and the CUDA path
// (paper_1112_5588_b200/) consume its output; neither is imported here.
//
// Matrix families (recipes stated in DESIGN.md §"Input recipe"):
//   HMEP        Holstein-Hubbard ring, 6 sites, 3 up + 3 down electrons, 5 phonon modes with
//               total occupation <= M.  PAPER.md L94-101 (§1.3 "HMEp": N = 6.2e6, ~15 nnz/row,
//               contiguous off-diagonals of length 15,000).  A = T (x) I_P + I_400 (x) (I_P + Ph),
//               row = pos(e)*P + p, so every electronic hop is a contiguous off-diagonal
//               segment of length P.  ordering 0 = lexicographic e = 20u+d,
//               ordering 1 = nested 4x2 spin-grid.
//   HMEP_BANDED tiny HMEp-like banded matrix (C1): 16 blocks x 4^5 phonon lattice,
//               block hops at +-{1,2,5,7,11,13} blocks.
//   SAMG        7-point Poisson stencil on an nx*ny*nz grid, Morton-numbered, 0.1% of rows
//               with 1-15 extra couplings from the 5^3 neighbourhood.  PAPER.md L104-109,
//               L274-276 (N = 3.4e6, N_nzr ~ 7, longest row > 4x shortest).
//   DLR1        46,417 jittered points x 6 unknowns, dense 6x6 coupling blocks to the d_p-1
//               nearest points.  PAPER.md L111-119, L270-274 (N = 2.8e5, N_nzr ~ 144,
//               max/min ~ 2, 80% of rows >= 0.8 N^max).
//
// Values: uniform in [-1,1) from a counter-based splitmix64 hash of (seed,row,col), so any row
// range can be generated independently (per rank).  x: uniform in [-1,1) from (seed+1, i).
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <algorithm>
#include <numeric>
#include <new>
#include <omp.h>

namespace {

inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return splitmix64(splitmix64(seed ^ splitmix64(a)) ^ b);
}
inline double unit_pm1(uint64_t h) {  // [-1, 1), 53-bit resolution
  return (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}
inline double unit01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

enum Family { HMEP = 0, HMEP_BANDED = 1, SAMG = 2, DLR1 = 3, DLR2 = 4, UHBR = 5 };

struct Gen {
  int family = 0;
  int64_t n = 0;
  uint64_t seed = 0;
  // HMEP
  int M = 0, P = 0;
  std::vector<int32_t> e_of_pos, pos_of_e;          // 400 electronic states
  std::vector<int32_t> thop_ptr, thop;              // hop graph T in e-index space
  std::vector<int32_t> ph_ptr, ph;                  // phonon coupling graph
  // SAMG
  int nx = 0, ny = 0, nz = 0;
  std::vector<int32_t> pt_of_row, row_of_pt;        // Morton order
  // DLR1
  std::vector<int32_t> nb_ptr, nb;                  // per point: sorted neighbour point ids (incl. self)
  int bs = 6;                                       // unknowns per point
  virtual ~Gen() {}
};

// ---------------------------------------------------------------- HMEp
void combos63(std::vector<uint8_t>& masks) {  // itertools.combinations(range(6),3) order
  masks.clear();
  for (int a = 0; a < 6; ++a)
    for (int b = a + 1; b < 6; ++b)
      for (int c = b + 1; c < 6; ++c) masks.push_back((uint8_t)((1 << a) | (1 << b) | (1 << c)));
}
int64_t binom(int64_t n, int64_t k) {
  if (k < 0 || k > n) return 0;
  int64_t r = 1;
  for (int64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

void build_hmep(Gen& g, int M, int ordering) {
  g.M = M;
  std::vector<uint8_t> cm;
  combos63(cm);
  auto idx_of = [&](uint8_t m) { return (int)(std::find(cm.begin(), cm.end(), m) - cm.begin()); };
  std::vector<std::vector<int>> hops(20);
  for (int c = 0; c < 20; ++c) {
    uint8_t m = cm[c];
    for (int s = 0; s < 6; ++s) {
      if (!(m >> s & 1)) continue;
      for (int t : {(s + 5) % 6, (s + 1) % 6}) {
        if (m >> t & 1) continue;
        hops[c].push_back(idx_of((uint8_t)((m & ~(1 << s)) | (1 << t))));
      }
    }
  }
  g.thop_ptr.assign(401, 0);
  g.thop.clear();
  for (int e = 0; e < 400; ++e) {
    int u = e / 20, d = e % 20;
    for (int u2 : hops[u]) g.thop.push_back(u2 * 20 + d);
    for (int d2 : hops[d]) g.thop.push_back(u * 20 + d2);
    g.thop_ptr[e + 1] = (int32_t)g.thop.size();
  }
  // electronic block order
  g.e_of_pos.resize(400);
  g.pos_of_e.resize(400);
  std::iota(g.e_of_pos.begin(), g.e_of_pos.end(), 0);
  if (ordering == 1) {  // nested 4x2 spin-grid
    static const int up_groups[4][5] = {{8, 15, 17, 18, 19}, {3, 5, 6, 7, 11}, {1, 2, 4, 10, 16}, {0, 9, 12, 13, 14}};
    static const int dn_group1[10] = {0, 1, 2, 3, 5, 6, 8, 9, 12, 15};
    int gu[20], gd[20];
    for (int gi = 0; gi < 4; ++gi)
      for (int k = 0; k < 5; ++k) gu[up_groups[gi][k]] = gi;
    for (int i = 0; i < 20; ++i) gd[i] = 0;
    for (int k = 0; k < 10; ++k) gd[dn_group1[k]] = 1;
    std::stable_sort(g.e_of_pos.begin(), g.e_of_pos.end(), [&](int a, int b) {
      int ca = 2 * gu[a / 20] + gd[a % 20], cb = 2 * gu[b / 20] + gd[b % 20];
      return ca < cb;  // ties keep (u,d) lexicographic order
    });
  }
  for (int p = 0; p < 400; ++p) g.pos_of_e[g.e_of_pos[p]] = p;
  // phonon states: 5-tuples with sum <= M, lexicographic (nested loops n1..n5)
  const int K = 5;
  int64_t P = binom(M + K, K);
  g.P = (int)P;
  std::vector<int> cnt((M + 1) * (K + 1));  // cnt[k][s] = C(s+k, k)
  for (int k = 0; k <= K; ++k)
    for (int s = 0; s <= M; ++s) cnt[k * (M + 1) + s] = (int)binom(s + k, k);
  auto rank = [&](const int* nv) {
    int64_t r = 0;
    int s = 0;
    for (int i = 0; i < K; ++i) {
      for (int v = 0; v < nv[i]; ++v) r += cnt[(K - 1 - i) * (M + 1) + (M - s - v)];
      s += nv[i];
    }
    return (int)r;
  };
  std::vector<int> states;
  states.reserve(P * K);
  int nv[K];
  for (nv[0] = 0; nv[0] <= M; ++nv[0])
    for (nv[1] = 0; nv[0] + nv[1] <= M; ++nv[1])
      for (nv[2] = 0; nv[0] + nv[1] + nv[2] <= M; ++nv[2])
        for (nv[3] = 0; nv[0] + nv[1] + nv[2] + nv[3] <= M; ++nv[3])
          for (nv[4] = 0; nv[0] + nv[1] + nv[2] + nv[3] + nv[4] <= M; ++nv[4])
            for (int i = 0; i < K; ++i) states.push_back(nv[i]);
  g.ph_ptr.assign(P + 1, 0);
  g.ph.clear();
  for (int64_t p = 0; p < P; ++p) {
    int t[K];
    int tot = 0;
    for (int i = 0; i < K; ++i) { t[i] = states[p * K + i]; tot += t[i]; }
    for (int i = 0; i < K; ++i) {
      if (tot < M) { t[i]++; g.ph.push_back(rank(t)); t[i]--; }
      if (t[i] > 0) { t[i]--; g.ph.push_back(rank(t)); t[i]++; }
    }
    g.ph_ptr[p + 1] = (int32_t)g.ph.size();
  }
  g.n = (int64_t)400 * P;
}

int hmep_row(const Gen& g, int64_t r, int32_t* cols) {
  int64_t P = g.P;
  int pos = (int)(r / P);
  int64_t p = r % P;
  int e = g.e_of_pos[pos];
  int k = 0;
  cols[k++] = (int32_t)r;
  for (int h = g.thop_ptr[e]; h < g.thop_ptr[e + 1]; ++h) cols[k++] = (int32_t)(g.pos_of_e[g.thop[h]] * P + p);
  for (int h = g.ph_ptr[p]; h < g.ph_ptr[p + 1]; ++h) cols[k++] = (int32_t)(pos * P + g.ph[h]);
  std::sort(cols, cols + k);
  return k;
}

// ---------------------------------------------------------------- HMEp banded (C1)
int hmep_banded_row(const Gen&, int64_t r, int32_t* cols) {
  const int PB = 1024, NB = 16;
  int b = (int)(r / PB), p = (int)(r % PB);
  static const int offs[6] = {1, 2, 5, 7, 11, 13};
  int k = 0;
  cols[k++] = (int32_t)r;
  for (int d = 0, w = 1; d < 5; ++d, w *= 4) {
    int dig = (p / w) % 4;
    if (dig < 3) cols[k++] = (int32_t)(b * PB + p + w);
    if (dig > 0) cols[k++] = (int32_t)(b * PB + p - w);
  }
  for (int o : offs) {
    if (b + o < NB) cols[k++] = (int32_t)((b + o) * PB + p);
    if (b - o >= 0) cols[k++] = (int32_t)((b - o) * PB + p);
  }
  std::sort(cols, cols + k);
  return k;
}

// ---------------------------------------------------------------- sAMG-shaped (C2)
inline uint64_t spread3(uint64_t v) {  // 10-bit -> every third bit
  uint64_t x = v & 0x3ff;
  x = (x | (x << 16)) & 0x30000ff;
  x = (x | (x << 8)) & 0x300f00f;
  x = (x | (x << 4)) & 0x30c30c3;
  x = (x | (x << 2)) & 0x9249249;
  return x;
}
void build_samg(Gen& g, int nx, int ny, int nz) {
  g.nx = nx; g.ny = ny; g.nz = nz;
  int64_t n = (int64_t)nx * ny * nz;
  g.n = n;
  std::vector<uint64_t> key(n);
#pragma omp parallel for
  for (int64_t pt = 0; pt < n; ++pt) {
    int64_t x = pt % nx, y = (pt / nx) % ny, z = pt / ((int64_t)nx * ny);
    key[pt] = (spread3(x) | (spread3(y) << 1) | (spread3(z) << 2)) << 32 | (uint64_t)pt;
  }
  std::sort(key.begin(), key.end());
  g.pt_of_row.resize(n);
  g.row_of_pt.resize(n);
  for (int64_t r = 0; r < n; ++r) {
    int32_t pt = (int32_t)(key[r] & 0xffffffffu);
    g.pt_of_row[r] = pt;
    g.row_of_pt[pt] = (int32_t)r;
  }
}
int samg_row(const Gen& g, int64_t r, int32_t* cols) {
  int64_t nx = g.nx, ny = g.ny, nz = g.nz;
  int64_t pt = g.pt_of_row[r];
  int64_t x = pt % nx, y = (pt / nx) % ny, z = pt / (nx * ny);
  auto id = [&](int64_t a, int64_t b, int64_t c) { return g.row_of_pt[a + nx * (b + ny * c)]; };
  int k = 0;
  cols[k++] = (int32_t)r;
  if (x > 0) cols[k++] = id(x - 1, y, z);
  if (x < nx - 1) cols[k++] = id(x + 1, y, z);
  if (y > 0) cols[k++] = id(x, y - 1, z);
  if (y < ny - 1) cols[k++] = id(x, y + 1, z);
  if (z > 0) cols[k++] = id(x, y, z - 1);
  if (z < nz - 1) cols[k++] = id(x, y, z + 1);
  // extra couplings: 0.1% of rows (hash-selected) get 1..15 extra entries from the 5^3
  // neighbourhood; the grid-centre point always gets 15, fixing N^max = 22.
  int extra = 0;
  bool centre = (x == nx / 2 && y == ny / 2 && z == nz / 2);
  if (centre) extra = 15;
  else if (unit01(hash3(g.seed, (uint64_t)pt, 0xE77A)) < 0.001)
    extra = 1 + (int)(hash3(g.seed, (uint64_t)pt, 0xC0) % 15);
  if (extra) {
    int base = k;
    uint64_t best[125];
    int nc = 0;
    for (int dz = -2; dz <= 2; ++dz)
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          int64_t a = x + dx, b = y + dy, c = z + dz;
          if (a < 0 || b < 0 || c < 0 || a >= nx || b >= ny || c >= nz) continue;
          int manh = std::abs(dx) + std::abs(dy) + std::abs(dz);
          if (manh <= 1) continue;  // stencil entries already present
          int32_t col = id(a, b, c);
          uint64_t h = hash3(g.seed ^ 0x5A5A, (uint64_t)pt, (uint64_t)col);
          best[nc++] = (h & ~0xffffffffull) | (uint32_t)col;
        }
    std::sort(best, best + nc);
    if (extra > nc) extra = nc;
    for (int i = 0; i < extra; ++i) cols[base + i] = (int32_t)(best[i] & 0xffffffffu);
    k = base + extra;
  }
  std::sort(cols, cols + k);
  return k;
}

// ---------------------------------------------------------------- DLR1-shaped (C4)
// Block k-NN family: G^3 jittered grid points minus NDROP hash-chosen ones, Morton-ordered, B
// unknowns per point (dense B x B coupling blocks) to the d_p - 1 nearest points within a +-W cell
// window.  kind 0 = DLR1 pmf, 1 = DLR2 (d_p: 60 % uniform 28..60, 40 % uniform 61..121 -> N_nzr ~
// 315, N^max 605, ELLPACK reduction ~ 48 % as Table 1), 2 = UHBR (d_p uniform 18..31, N_nzr ~ 123).
void build_blockknn(Gen& g, int G, int NDROP, int B, int kind, int W) {
  const int NP = G * G * G;
  std::vector<uint64_t> hk(NP);
  for (int i = 0; i < NP; ++i) hk[i] = (hash3(g.seed, (uint64_t)i, 0xD409) & ~0xffffull) | 0;
  std::vector<int> order(NP);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return hk[a] != hk[b] ? hk[a] < hk[b] : a < b; });
  std::vector<char> dropped(NP, 0);
  for (int i = 0; i < NDROP; ++i) dropped[order[i]] = 1;
  // Morton order of the surviving grid points
  std::vector<uint64_t> key;
  for (int pt = 0; pt < NP; ++pt) {
    if (dropped[pt]) continue;
    int x = pt % G, y = (pt / G) % G, z = pt / (G * G);
    key.push_back((spread3(x) | (spread3(y) << 1) | (spread3(z) << 2)) << 32 | (uint64_t)pt);
  }
  std::sort(key.begin(), key.end());
  int npts = (int)key.size();
  std::vector<int> id_of_grid(NP, -1), grid_of_id(npts);
  for (int i = 0; i < npts; ++i) {
    int pt = (int)(key[i] & 0xffffffffu);
    id_of_grid[pt] = i;
    grid_of_id[i] = pt;
  }
  // jittered positions
  std::vector<double> pos(3 * (size_t)npts);
  for (int i = 0; i < npts; ++i) {
    int pt = grid_of_id[i];
    int x = pt % G, y = (pt / G) % G, z = pt / (G * G);
    pos[3 * i + 0] = x + 0.35 * unit_pm1(hash3(g.seed, (uint64_t)pt, 0x11));
    pos[3 * i + 1] = y + 0.35 * unit_pm1(hash3(g.seed, (uint64_t)pt, 0x22));
    pos[3 * i + 2] = z + 0.35 * unit_pm1(hash3(g.seed, (uint64_t)pt, 0x33));
  }
  // coupling count d_p: P(d)=0.2/9 for 15..23, 0.8*{.46,.20,.12,.10,.07,.05} for 24..29
  static const double pmf_hi[6] = {.46, .20, .12, .10, .07, .05};
  std::vector<int> dp(npts);
  for (int i = 0; i < npts; ++i) {
    double u = unit01(hash3(g.seed, (uint64_t)grid_of_id[i], 0xDDDD));
    int d;
    if (kind == 1) d = u < 0.6 ? 28 + std::min(32, (int)(u / 0.6 * 33)) : 61 + std::min(60, (int)((u - 0.6) / 0.4 * 61));
    else if (kind == 2) d = 18 + std::min(13, (int)(u * 14));
    else if (u < 0.2) d = 15 + std::min(8, (int)(u / (0.2 / 9)));
    else {
      double acc = 0.2;
      d = 29;
      for (int k = 0; k < 6; ++k) {
        acc += 0.8 * pmf_hi[k];
        if (u < acc) { d = 24 + k; break; }
      }
    }
    dp[i] = d;
  }
  g.nb_ptr.assign(npts + 1, 0);
  g.nb.clear();
  std::vector<std::vector<int>> lists(npts);
#pragma omp parallel for schedule(dynamic, 256)
  for (int i = 0; i < npts; ++i) {
    int pt = grid_of_id[i];
    int x = pt % G, y = (pt / G) % G, z = pt / (G * G);
    std::vector<std::pair<double, int>> cand;
    for (int dz = -W; dz <= W; ++dz)
      for (int dy = -W; dy <= W; ++dy)
        for (int dx = -W; dx <= W; ++dx) {
          int a = x + dx, b = y + dy, c = z + dz;
          if (a < 0 || b < 0 || c < 0 || a >= G || b >= G || c >= G) continue;
          int j = id_of_grid[a + G * (b + G * c)];
          if (j < 0 || j == i) continue;
          double ddx = pos[3 * j] - pos[3 * i], ddy = pos[3 * j + 1] - pos[3 * i + 1], ddz = pos[3 * j + 2] - pos[3 * i + 2];
          cand.push_back({ddx * ddx + ddy * ddy + ddz * ddz, j});
        }
    std::sort(cand.begin(), cand.end());
    std::vector<int> l;
    l.push_back(i);
    for (int k = 0; k < dp[i] - 1 && k < (int)cand.size(); ++k) l.push_back(cand[k].second);
    std::sort(l.begin(), l.end());
    lists[i] = std::move(l);
  }
  for (int i = 0; i < npts; ++i) {
    for (int j : lists[i]) g.nb.push_back(j);
    g.nb_ptr[i + 1] = (int32_t)g.nb.size();
  }
  g.bs = B;
  g.n = (int64_t)npts * B;
}
int dlr1_row(const Gen& g, int64_t r, int32_t* cols) {
  const int B = g.bs;
  int i = (int)(r / B);
  int k = 0;
  for (int h = g.nb_ptr[i]; h < g.nb_ptr[i + 1]; ++h)
    for (int c = 0; c < B; ++c) cols[k++] = (int32_t)(g.nb[h] * B + c);
  return k;  // already ascending
}

int row_cols(const Gen& g, int64_t r, int32_t* cols) {
  switch (g.family) {
    case HMEP: return hmep_row(g, r, cols);
    case HMEP_BANDED: return hmep_banded_row(g, r, cols);
    case SAMG: return samg_row(g, r, cols);
    case DLR1:
    case DLR2:
    case UHBR: return dlr1_row(g, r, cols);
  }
  return 0;
}
const int kMaxRow = 1024;

}  // namespace

extern "C" {

// family: 0 HMEP (p0 = M, p1 = ordering), 1 HMEP_BANDED, 2 SAMG (p0,p1,p2 = nx,ny,nz), 3 DLR1,
// 4 DLR2, 5 UHBR.
// Returns nullptr on bad arguments.
void* pjdsgen_create(int family, int p0, int p1, int p2, uint64_t seed) {
  Gen* g = new (std::nothrow) Gen();
  if (!g) return nullptr;
  g->family = family;
  g->seed = seed;
  switch (family) {
    case HMEP:
      if (p0 < 1 || p0 > 40 || (p1 != 0 && p1 != 1)) { delete g; return nullptr; }
      build_hmep(*g, p0, p1);
      break;
    case HMEP_BANDED: g->n = 16 * 1024; break;
    case SAMG:
      if (p0 < 2 || p1 < 2 || p2 < 2 || p0 > 1024 || p1 > 1024 || p2 > 1024) { delete g; return nullptr; }
      build_samg(*g, p0, p1, p2);
      break;
    case DLR1: build_blockknn(*g, 36, 239, 6, 0, 3); break;          // 46,417 points x 6
    case DLR2: build_blockknn(*g, 48, 2196, 5, 1, 4); break;         // 108,396 points x 5
    case UHBR: build_blockknn(*g, 97, 12673, 5, 2, 3); break;        // 900,000 points x 5
    default: delete g; return nullptr;
  }
  return g;
}
void pjdsgen_destroy(void* h) { delete (Gen*)h; }
int64_t pjdsgen_n(void* h) { return ((Gen*)h)->n; }

// Row lengths for rows [r0, r1) -> len[r1-r0]. Returns total entries.
int64_t pjdsgen_rowlen(void* h, int64_t r0, int64_t r1, int32_t* len) {
  const Gen& g = *(Gen*)h;
  int64_t tot = 0;
#pragma omp parallel for reduction(+ : tot) schedule(static, 4096)
  for (int64_t r = r0; r < r1; ++r) {
    int32_t cols[kMaxRow];
    int k = row_cols(g, r, cols);
    len[r - r0] = k;
    tot += k;
  }
  return tot;
}

// Fill rows [r0, r1) given rowptr (length r1-r0+1, rowptr[0] = 0): ascending global column ids
// and values.  dtype 0 = float32 (rounded from the double value), 1 = float64; +2 = symmetric
// values a(r,c) = a(c,r) (hash of the unordered pair; every family's pattern is structurally
// symmetric except DLR1's k-NN blocks).
void pjdsgen_fill(void* h, int64_t r0, int64_t r1, const int64_t* rowptr, int32_t* col, void* val, int dtype) {
  const bool sym = dtype & 2;
  dtype &= 1;
  const Gen& g = *(Gen*)h;
#pragma omp parallel for schedule(static, 4096)
  for (int64_t r = r0; r < r1; ++r) {
    int32_t cols[kMaxRow];
    int k = row_cols(g, r, cols);
    int64_t o = rowptr[r - r0];
    for (int i = 0; i < k; ++i) {
      col[o + i] = cols[i];
      const uint64_t a = sym ? (uint64_t)std::min<int64_t>(r, cols[i]) : (uint64_t)r;
      const uint64_t b = sym ? (uint64_t)std::max<int64_t>(r, cols[i]) : (uint64_t)cols[i];
      double v = unit_pm1(hash3(g.seed, a, b));
      if (dtype == 1) ((double*)val)[o + i] = v;
      else ((float*)val)[o + i] = (float)v;
    }
  }
}

// Dense vector entries [i0, i1): uniform [-1,1) from (seed, i).
void pjdsgen_vector(uint64_t seed, int64_t i0, int64_t i1, void* out, int dtype) {
#pragma omp parallel for schedule(static, 65536)
  for (int64_t i = i0; i < i1; ++i) {
    double v = unit_pm1(hash3(seed, (uint64_t)i, 0x5EC7));
    if (dtype == 1) ((double*)out)[i - i0] = v;
    else ((float*)out)[i - i0] = (float)v;
  }
}

// Value of entry (row, col) as generated (lets tests re-derive single entries).
double pjdsgen_value(uint64_t seed, int64_t row, int64_t col) {
  return unit_pm1(hash3(seed, (uint64_t)row, (uint64_t)col));
}

}  // extern "C"
