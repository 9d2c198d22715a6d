// Device kernels for sm_100a: pJDS spMVM (Listing 2), ELLPACK-R spMVM
// (Listing 1), halo pack ("local gather", Fig. 4 caption L401-402), and the stream
// bandwidth probe that supplies the roofline denominator.
//
// The path is HBM-bandwidth bound (code balance 6+4a+4/N_nzr B/flop DP, Eq. 1
// with write-only y): no tensor cores.  What matters on B200 is bytes in flight per SM and the
// L2 residency of x:
//   * val/col are streamed once: ld.global.nc.L1::no_allocate with an L2 evict_first policy;
//   * x is gathered through the read-only path (ld.global.nc, L1 allocate) with an L2
//     evict_last policy so it survives the val/col stream (RHS reuse alpha, L340-351);
//   * the j-loop is unrolled by U with all U val/col loads issued before the dependent x gathers,
//     and every thread owns R consecutive sorted rows (vector loads, R independent chains) so a
//     warp keeps U*R*(s_v+4)*32 bytes in flight;
//   * col_start[] is staged in shared memory ("assumed to always come from cache", L349).
// Each row is ONE fused-multiply-add chain over its stored entries in CRS order starting from
// +0.0 (padding adds exact +0): bitwise reproducible against oracle/ O3 for every R, U.
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <algorithm>
#include <climits>
#include <type_traits>
#include <vector>
#include "internal.h"

namespace pjds {

static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t k) { g_launches += k; }

namespace {

// ---- load helpers --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// L2 eviction policy by kind: 0 evict_normal, 1 evict_first, 2 evict_last, 3 evict_unchanged
__device__ __forceinline__ uint64_t make_policy(int kind) {
  uint64_t p;
  if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 3) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// streaming (read once): no L1 allocation, L2 evict-first
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ld_stream2(const float* p, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ld_stream2(const int* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
// RHS gather (reused): read-only path, L1 allocate, L2 evict-last
__device__ __forceinline__ double ld_rhs(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_rhs(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// window gathers use the plain (coherent) global load, L1-allocating: the windows include peer
// memory mapped over NVLink, for which the plain load is the conservative choice
__device__ __forceinline__ double ld_win(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_win(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// RHS gather of the fused remote-gather dist kernel (PJDS_TRANSPORT_DIRECT): column code
// (owner << shift) | position addresses owner's x window (own memory, or a peer's through its
// CUDA-IPC mapping -- an NVLink load between GPUs); otherwise a plain x[c] gather
constexpr int kMaxWin = 64;
template <bool WIN, typename T>
__device__ __forceinline__ T gather_x(const T* x, const T* const* win, int shift, int c, uint64_t pol) {
  if constexpr (WIN) return ld_win(win[(unsigned)c >> shift] + (c & ((1 << shift) - 1)), pol);
  else return ld_rhs(x + c, pol);
}
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// R-wide vector of T / int for the R consecutive sorted rows a thread owns (one jagged column)
template <typename T, int R> struct Vec;
template <typename T> struct Vec<T, 1> {
  T v[1];
  __device__ __forceinline__ void load(const T* p, uint64_t pol) { v[0] = ld_stream(p, pol); }
};
template <typename T> struct Vec<T, 2> {
  T v[2];
  __device__ __forceinline__ void load(const T* p, uint64_t pol) {
    auto t = ld_stream2(p, pol);
    v[0] = t.x; v[1] = t.y;
  }
};
template <> struct Vec<double, 4> {  // 256-bit LDG (sm_100): L2 evict-first is encoded in the op
  double v[4];
  __device__ __forceinline__ void load(const double* p, uint64_t) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  }
};
template <> struct Vec<float, 4> {
  float v[4];
  __device__ __forceinline__ void load(const float* p, uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
  }
};
template <> struct Vec<int, 4> {
  int v[4];
  __device__ __forceinline__ void load(const int* p, uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(p), "l"(pol));
  }
};

// R-wide vector store of a thread's R consecutive results with an L2 policy (y-store experiment)
template <typename T, int R>
__device__ __forceinline__ void st_rows(T* p, const T (&a)[R], uint64_t pol) {
  if constexpr (sizeof(T) == 8 && R == 4)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "d"((double)a[0]), "d"((double)a[1]), "d"((double)a[2]), "d"((double)a[3]), "l"(pol) : "memory");
  else if constexpr (sizeof(T) == 8 && R == 2)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;"
                 :: "l"(p), "d"((double)a[0]), "d"((double)a[1]), "l"(pol) : "memory");
  else if constexpr (sizeof(T) == 4 && R == 4)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"((float)a[0]), "f"((float)a[1]), "f"((float)a[2]), "f"((float)a[3]), "l"(pol) : "memory");
  else if constexpr (sizeof(T) == 4 && R == 2)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;"
                 :: "l"(p), "f"((float)a[0]), "f"((float)a[1]), "l"(pol) : "memory");
  else
#pragma unroll
    for (int r = 0; r < R; ++r) p[r] = a[r];
}

// one scattered y element with an L2 policy (row-only basis: y[perm[k]]; dist nonlocal part: y += )
__device__ __forceinline__ void st_one(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_one(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_one(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_one(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// IL (lane-interleaved rows): the R rows of a thread are 32 apart (row warp_k0 + lane + 32 r), so
// one gather instruction covers 32 consecutive rows; val/col then take R scalar loads per slot.
template <bool IL, typename T, int R>
__device__ __forceinline__ void load_rows(Vec<T, R>& v, const T* p, uint64_t pol) {
  if constexpr (IL) {
#pragma unroll
    for (int r = 0; r < R; ++r) v.v[r] = ld_stream(p + 32 * r, pol);
  } else {
    v.load(p, pol);
  }
}

#ifndef PJDS_CTA_THREADS
#define PJDS_CTA_THREADS 256
#endif
constexpr int kThreads = PJDS_CTA_THREADS;  // CTA size (build-time; a CTA tile is kThreads x R sorted rows)
static_assert(kThreads % 32 == 0 && kThreads <= 256, "CTA size: a multiple of 32, at most 256");
constexpr int kSmemCS = 1024;  // col_start entries staged in shared memory
// Register budget: plain __launch_bounds__(256) (48 registers for the R=4 DP kernel).  Measured:
// __launch_bounds__(256, 6) (<= 40 regs) is 3-15 % slower in DP, and __launch_bounds__(256, 1)
// lets ptxas take 84 registers, halving occupancy (C2 DP 58 -> 147 us).

// Store modes: y[perm[k]] = acc (row-only basis), y[k] = acc (permuted basis, PJDS_PERM_SYMMETRIC),
// y[perm[k]] += acc (dist nonlocal part: the result is written twice).
// STORE_DIRECT_DOT additionally writes per-CTA partial sums of y[k]*x[k] (permuted basis, so x[k]
// is the input entry of row k): the Lanczos alpha = (A v).v fused into the product's epilogue.
enum { STORE_PERM = 0, STORE_DIRECT = 1, STORE_PERM_ACC = 2, STORE_DIRECT_DOT = 3 };

// ---- programmatic dependent launch (sm_90+; B200 launch overlap of back-to-back products) -----
// A product launched with cudaLaunchAttributeProgrammaticStreamSerialization may start while the
// previous grid on the stream drains: its CTAs run the matrix-only prologue (tile/warp lookup,
// col_start staging, and -- first-wave CTAs only -- an L2 prefetch of the first jagged columns of
// their val/col tiles) and then block in griddepcontrol.wait until the previous grid has completed
// and its writes are visible.  x, y and dot_part are touched only after the wait, so any producer /
// consumer order of an iterative scheme is kept.  Launched without the attribute both instructions
// are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}
// lane j < ncols of the warp prefetches the warp's rows [warp_k0, warp_k0 + 32R) of jagged column j
// (val and col; column j holds sorted rows [0, col_start[j+1] - col_start[j]) of a global sort).
// Ranges are 16-byte aligned multiples of 16 bytes: col_start entries are multiples of b_r (>= 32)
// and warp_k0 a multiple of 32R.
template <typename T, typename Off, int R>
__device__ __forceinline__ void pdl_prefetch_warp(const T* val, const int* col, const Off* s_cs,
                                                  const int64_t* col_start, int64_t warp_k0, int ncols, uint64_t pol) {
  const int j = threadIdx.x & 31;
  if (j >= ncols) return;
  const int64_t c0 = j < kSmemCS ? (int64_t)s_cs[j] : col_start[j];
  const int64_t c1 = j + 1 < kSmemCS ? (int64_t)s_cs[j + 1] : col_start[j + 1];
  int64_t m = c1 - c0 - warp_k0;  // rows of the warp present in column j
  if (m <= 0) return;
  if (m > 32 * R) m = 32 * R;
  prefetch_l2_bulk(val + c0 + warp_k0, (uint32_t)(m * sizeof(T)), pol);
  prefetch_l2_bulk(col + c0 + warp_k0, (uint32_t)(m * sizeof(int)), pol);
}

// ---- pJDS kernel -----------------------------------------------------------------------------

// The R row chains of one thread (rows k0 + r*RS, all of length `len`, one jagged column per
// step): the j-loop of Listing 2 (L231-237) shared by the static and the dynamic-schedule kernel.
template <typename T, typename Off, int R, int U, bool PIPE, bool IL, bool WIN>
__device__ __forceinline__ void row_chains(T (&acc)[R], const T* __restrict__ val, const int* __restrict__ col,
                                           const Off* s_cs, const int64_t* __restrict__ col_start, int64_t k0,
                                           int len, const T* __restrict__ x, const T* const* s_win, int win_shift,
                                           uint64_t pol_s, uint64_t pol_x) {
  auto cs = [&](int j) -> Off { return j < kSmemCS ? s_cs[j] : (Off)col_start[j]; };
  int j = 0;
  if (PIPE && U <= len) {
    // software pipeline: the val/col loads of chunk j+U are issued before the FMAs of chunk j, so
    // the stream of the next chunk overlaps the dependent x gathers of the current one
    Vec<T, R> va[U];
    Vec<int, R> ca[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const Off o = cs(u) + (Off)k0;
      load_rows<IL>(va[u], val + o, pol_s);
      load_rows<IL>(ca[u], col + o, pol_s);
    }
    for (;;) {
      T xv[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) xv[u][r] = gather_x<WIN>(x, s_win, win_shift, ca[u].v[r], pol_x);
      const int jn = j + U;
      const bool more = jn + U <= len;
      Vec<T, R> vb[U];
      Vec<int, R> cb[U];
      if (more) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Off o = cs(jn + u) + (Off)k0;
          load_rows<IL>(vb[u], val + o, pol_s);
          load_rows<IL>(cb[u], col + o, pol_s);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma_rn(va[u].v[r], xv[u][r], acc[r]);
      j = jn;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        va[u] = vb[u];
        ca[u] = cb[u];
      }
    }
  }
  for (; j + U <= len; j += U) {  // full chunks: no predicates, all U loads issued back to back
    Vec<T, R> v[U];
    Vec<int, R> c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const Off o = cs(j + u) + (Off)k0;
      load_rows<IL>(v[u], val + o, pol_s);
      load_rows<IL>(c[u], col + o, pol_s);
    }
    T xv[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) xv[u][r] = gather_x<WIN>(x, s_win, win_shift, c[u].v[r], pol_x);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fma_rn(v[u].v[r], xv[u][r], acc[r]);
  }
  if (j < len) {  // ragged tail of the j-loop: predicated, same chain order
    Vec<T, R> v[U];
    Vec<int, R> c[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < len) {
        const Off o = cs(j + u) + (Off)k0;
        load_rows<IL>(v[u], val + o, pol_s);
        load_rows<IL>(c[u], col + o, pol_s);
      }
    T xv[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < len)
#pragma unroll
        for (int r = 0; r < R; ++r) xv[u][r] = gather_x<WIN>(x, s_win, win_shift, c[u].v[r], pol_x);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < len)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma_rn(v[u].v[r], xv[u][r], acc[r]);
  }
}

// Thread t owns the R consecutive sorted rows k0 = R*t .. R*t+R-1 (R divides b_r, so they share
// one pJDS block and its length).  A warp covers 32R rows = one or several consecutive blocks;
// lanes of a block loop to that block's length (PAPER.md L219-222 / Listing 2, reading 6).
// PIPE: software-pipelined main loop (next chunk's val/col loads in flight during the current
// chunk's x gathers) -- for long rows, whose chunks otherwise cost two dependent round trips each.
// Per row: acc = +0; for j < block_len: acc = fma(val[col_start[j]+k], x[col[...]], acc).
// WIN: fused remote-gather dist kernel (x = the owners' windows, see gather_x).
// dev experiments only (-DPJDS_IL_MINB=n): minimum resident CTAs for the lane-interleaved kernels;
// the default build gives every kernel plain __launch_bounds__(kThreads) (ptxas: 48 / 56 registers)
#ifdef PJDS_IL_MINB
#define PJDS_KERNEL_BOUNDS __launch_bounds__(kThreads, IL ? PJDS_IL_MINB : 4)
#else
#define PJDS_KERNEL_BOUNDS __launch_bounds__(kThreads)
#endif
template <typename T, typename Off, int R, int U, int MODE, bool PIPE, bool IL = false, bool WIN = false>
__global__ void PJDS_KERNEL_BOUNDS
pjds_spmv_kernel(const T* __restrict__ val, const int* __restrict__ col, const int64_t* __restrict__ col_start,
                 const int* __restrict__ block_len, const int* __restrict__ perm, const T* __restrict__ x,
                 T* __restrict__ y, int64_t n, int64_t n_pad, int br, int pol, const int* __restrict__ tile_order,
                 double* __restrict__ dot_part, int64_t sigma, const int64_t* __restrict__ wcs_off,
                 const T* const* __restrict__ win, int win_shift, const int* __restrict__ warp_order,
                 int64_t n_wtiles, int pf_cols, int pf_ctas, int trig_late) {
  // programmatic dependent launch (see pdl_trigger): the next grid on the stream may be scheduled
  // once every CTA of this one has started, i.e. into the SM slots this grid's last wave frees --
  // or, trig_late (one-wave grids), once every CTA has finished its row chains
  if (!trig_late) pdl_trigger();
  __shared__ Off s_cs[kSmemCS];
  __shared__ const T* s_win[WIN ? kMaxWin : 1];
  if constexpr (WIN)
    for (int i = threadIdx.x; i < kMaxWin; i += kThreads) s_win[i] = win[i];
  constexpr int RS = IL ? 32 : 1;  // distance between a thread's rows
  int64_t k0, cta_k0;
  int cta_len;
  if (warp_order) {
    // warp-granular order (tile order mode 3): each warp takes the warp tile (32 R consecutive
    // sorted rows) the table assigns to its slot, so one CTA runs warp tiles of several length
    // classes from one region of the original matrix; staged col_start covers the widest (block 0)
    const int64_t slot = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const int64_t wt = slot < n_wtiles ? (int64_t)warp_order[slot] : (n_pad / (32 * R) + 1);
    k0 = wt * 32 * R + (int64_t)(threadIdx.x & 31) * (IL ? 1 : R);
    cta_k0 = 0;
    cta_len = block_len[0];
  } else {
    // execution order of the CTA tiles (storage order, or by original row; results are identical)
    const int64_t tile = tile_order ? (int64_t)tile_order[blockIdx.x] : (int64_t)blockIdx.x;
    const int64_t t = tile * kThreads + threadIdx.x;
    k0 = IL ? ((t & ~int64_t(31)) * R + (t & 31)) : t * R;
    cta_k0 = tile * kThreads * R;
    cta_len = block_len[cta_k0 / br];  // first block of the CTA is its longest
  }
  // sort window of this CTA (CTAs never straddle windows: sigma is a multiple of the tile size);
  // its col_start table already includes the window's storage offset (kernel view)
  col_start += wcs_off[cta_k0 / sigma];
  const int lim = min(cta_len + 1, kSmemCS);
  for (int j = threadIdx.x; j < lim; j += kThreads) s_cs[j] = (Off)col_start[j];
  __syncthreads();
  const bool active = k0 < n_pad;
  if (!active && MODE != STORE_DIRECT_DOT) return;
  T acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = T(0);
  const int64_t warp_k0 = IL ? (k0 - (threadIdx.x & 31)) : (k0 - (int64_t)(threadIdx.x & 31) * R);
  const int wlen = active ? block_len[warp_k0 / br] : 0;
  // everything above reads only the matrix; x (and y, dot_part) only after the previous grid is done
  if (pf_cols > 0 && (int)blockIdx.x < pf_ctas && active)
    pdl_prefetch_warp<T, Off, R>(val, col, s_cs, col_start, warp_k0, min(wlen, pf_cols), make_policy(pol & 0xff));
  pdl_wait();
  if (active) {
  const int len = (br >= 32 * R) ? wlen : block_len[k0 / br];
  const uint64_t pol_s = make_policy(pol & 0xff);
  const uint64_t pol_x = make_policy((pol >> 8) & 0xff);
  row_chains<T, Off, R, U, PIPE, IL, WIN>(acc, val, col, s_cs, col_start, k0, len, x, s_win, win_shift, pol_s, pol_x);
  if (trig_late) pdl_trigger();
  const int y_kind = (pol >> 16) & 0xff;
  const int p_kind = (pol >> 24) & 0x7f;  // scattered stores through perm: 0 plain, 1 + L2 policy kind
  if ((MODE == STORE_DIRECT || MODE == STORE_DIRECT_DOT) && !IL && R > 1 && y_kind && k0 + R <= n) {
    // (the Lanczos product's y is read by the next pass: no evict-first there)
    st_rows<T, R>(y + k0, acc, make_policy(MODE == STORE_DIRECT_DOT ? 0 : y_kind - 1));
  } else
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t k = k0 + r * RS;
    if (k < n) {
      if (MODE == STORE_DIRECT || MODE == STORE_DIRECT_DOT) {
        y[k] = acc[r];
      } else {
        const int p = perm[k];
        if (p_kind) {
          const uint64_t pp = make_policy(p_kind - 1);
          st_one(y + p, MODE == STORE_PERM_ACC ? ld_one(y + p, pp) + acc[r] : acc[r], pp);
        } else if (MODE == STORE_PERM_ACC) {
          y[p] = y[p] + acc[r];
        } else {
          y[p] = acc[r];
        }
      }
    }
  }
  }  // active
  if (MODE == STORE_DIRECT_DOT) {
    // one partial per warp (no CTA barrier: a warp's lanes leave as soon as their warp is done)
    double d = 0.0;
    if (active)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (k0 + r * RS < n) d = fma((double)acc[r], (double)x[k0 + r * RS], d);
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) dot_part[blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)] = d;
  }
}

// Dynamic warp-tile schedule (opt-in experiment, pjds_set_schedule(1); measured slower, see g_sched).  A static grid of CTA
// tiles leaves SMs idle in the last partial wave, and with one wave (DLR1: 544 CTAs) the SMs that
// drew the longest rows finish last.  Here a persistent grid of (SMs x resident CTAs) warps takes
// warp tiles of 32R sorted rows from a global counter in storage order -- longest rows first, so
// the schedule is greedy longest-processing-time -- and runs the same row chains (results are
// bitwise those of the static kernel).  The last CTA to finish resets the counter, so launches on
// one stream need no memset (graph-capture safe; a handle must not run on two streams at once).
template <typename T, typename Off, int R, int U, int MODE, bool PIPE, bool WIN>
__global__ void __launch_bounds__(kThreads)
pjds_spmv_dyn_kernel(const T* __restrict__ val, const int* __restrict__ col, const int64_t* __restrict__ col_start,
                     const int* __restrict__ block_len, const int* __restrict__ perm, const T* __restrict__ x,
                     T* __restrict__ y, int64_t n, int64_t n_pad, int br, int pol, const int* __restrict__ tile_order,
                     const T* const* __restrict__ win, int win_shift, int64_t n_slots,
                     unsigned long long* __restrict__ sched, int width) {
  __shared__ Off s_cs[kSmemCS];
  __shared__ const T* s_win[WIN ? kMaxWin : 1];
  if constexpr (WIN)
    for (int i = threadIdx.x; i < kMaxWin; i += kThreads) s_win[i] = win[i];
  const int lim = min(width + 1, kSmemCS);  // the whole table: every warp tile may come here
  for (int j = threadIdx.x; j < lim; j += kThreads) s_cs[j] = (Off)col_start[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t pol_s = make_policy(pol & 0xff);
  const uint64_t pol_x = make_policy((pol >> 8) & 0xff);
  constexpr int kWarpsPerTile = kThreads / 32;
#pragma unroll 1
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(&sched[0], 1ull);
    w = __shfl_sync(0xffffffffu, w, 0);
    if ((int64_t)w >= n_slots) break;
    // warp tile -> rows, following the CTA tile order (kWarpsPerTile warp tiles per CTA tile)
    const int64_t wt = tile_order ? (int64_t)tile_order[w / kWarpsPerTile] * kWarpsPerTile + (int64_t)(w % kWarpsPerTile)
                                  : (int64_t)w;
    const int64_t warp_k0 = wt * 32 * R;
    const int64_t k0 = warp_k0 + (int64_t)lane * R;
    if (k0 >= n_pad) continue;
    const int wlen = block_len[warp_k0 / br];
    const int len = (br >= 32 * R) ? wlen : block_len[k0 / br];
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    row_chains<T, Off, R, U, PIPE, false, WIN>(acc, val, col, s_cs, col_start, k0, len, x, s_win, win_shift, pol_s,
                                               pol_x);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t k = k0 + r;
      if (k < n) {
        if (MODE == STORE_DIRECT) {
          y[k] = acc[r];
        } else {
          const int p = perm[k];
          if (MODE == STORE_PERM_ACC) y[p] = y[p] + acc[r];
          else y[p] = acc[r];
        }
      }
    }
  }
  __syncthreads();  // every warp of this CTA is past its last counter read
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&sched[1], 1ull) == (unsigned long long)gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// Long-row ("split-j") variant: S warps share one group of 32 rows so that long
// rows (DLR1/DLR2/UHBR, N_nzr 123-315) do not leave each thread a long serial chain of dependent
// gathers.  Warp w of a CTA works on row group w / S as sub s = w % S: lane l owns row
// cta_k0 + 32*(w / S) + l and runs the FMA chain over its slots j = s, s+S, s+2S, ... < block_len
// from +0 (every load instruction still reads 32 consecutive slots of one jagged column); the S
// partial sums meet in shared memory and sub 0 adds them in the fixed tree ((p0+p1)+(p2+p3))+...
// Not the single-chain order of reading 14: checked bitwise against oracle_spmv_split_chain and
// against the O2 bound.
template <typename T, typename Off, int S, int U, int MODE>
__global__ void __launch_bounds__(kThreads, 4)
pjds_spmv_split_kernel(const T* __restrict__ val, const int* __restrict__ col, const int64_t* __restrict__ col_start,
                       const int* __restrict__ block_len, const int* __restrict__ perm, const T* __restrict__ x,
                       T* __restrict__ y, int64_t n, int64_t n_pad, int br, int pol, double* __restrict__ dot_part,
                       int64_t sigma, const int64_t* __restrict__ wcs_off) {
  constexpr int kWarps = kThreads / 32;
  constexpr int RPC = 32 * kWarps / S;  // rows per CTA
  __shared__ Off s_cs[kSmemCS];
  __shared__ T s_part[kWarps][32];
  const int64_t cta_k0 = (int64_t)blockIdx.x * RPC;
  const int cta_len = block_len[cta_k0 / br];
  col_start += wcs_off[cta_k0 / sigma];
  const int lim = min(cta_len + 1, kSmemCS);
  for (int j = threadIdx.x; j < lim; j += kThreads) s_cs[j] = (Off)col_start[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sub = w % S;
  const int64_t k = cta_k0 + 32 * (w / S) + lane;
  const bool active = k < n_pad;
  T acc = T(0);
  if (active) {
    const int len = block_len[k / br];  // 32 rows of a group share one block (b_r % 32 == 0)
    const uint64_t pol_s = make_policy(pol & 0xff);
    const uint64_t pol_x = make_policy((pol >> 8) & 0xff);
    auto cs = [&](int j) -> Off { return j < kSmemCS ? s_cs[j] : (Off)col_start[j]; };
    int j = sub;
    for (; j + S * (U - 1) < len; j += S * U) {
      T v[U];
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const Off o = cs(j + S * u) + (Off)k;
        v[u] = ld_stream(val + o, pol_s);
        c[u] = ld_stream(col + o, pol_s);
      }
      T xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = ld_rhs(x + c[u], pol_x);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma_rn(v[u], xv[u], acc);
    }
    for (; j < len; j += S) {
      const Off o = cs(j) + (Off)k;
      acc = fma_rn(ld_stream(val + o, pol_s), ld_rhs(x + ld_stream(col + o, pol_s), pol_x), acc);
    }
  }
  s_part[w][lane] = acc;
  __syncthreads();
  const bool owner = active && sub == 0 && k < n;
  if (sub == 0) {
    // pairwise tree over the group's S partials (warps w .. w+S-1), written out so that no
    // partial needs a local-memory array
    auto P = [&](int q) -> T { return s_part[w + q][lane]; };
    if constexpr (S == 2) acc = P(0) + P(1);
    else if constexpr (S == 4) acc = (P(0) + P(1)) + (P(2) + P(3));
    else acc = ((P(0) + P(1)) + (P(2) + P(3))) + ((P(4) + P(5)) + (P(6) + P(7)));
    if (owner) {
      if (MODE == STORE_DIRECT || MODE == STORE_DIRECT_DOT) {
        y[k] = acc;
      } else {
        const int pr = perm[k];
        if (MODE == STORE_PERM_ACC) y[pr] = y[pr] + acc;
        else y[pr] = acc;
      }
    }
  }
  if (MODE == STORE_DIRECT_DOT) {
    __shared__ double s_red[kWarps];
    double d = owner ? (double)acc * (double)x[k] : 0.0;
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) s_red[w] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tsum = 0.0;
      for (int q = 0; q < kWarps; ++q) tsum += s_red[q];
      dot_part[blockIdx.x] = tsum;
    }
  }
}

static int g_pol = 1 | (2 << 8) | (2 << 16);  // val/col evict_first, x evict_last, y vector store evict_first
static int g_tile_order = 2;  // 0 storage order, 1 by first row's original index, 2 auto (see launch_pjds_t),
                              // 3 warp tiles by their first row's original index

// Tiles (CTAs of rows_per_tile consecutive sorted rows) ordered by the original index of their first
// row: all length classes of one region of the original matrix run together, so the RHS entries
// they share are reused from L2 (the sort destroys this locality).
int tile_order_for(const pjds_mat* A, int R, const int** out) {
  *out = A->d_order[R == 4 ? 2 : (R == 2 ? 1 : 0)];
  if (!*out) return set_error(PJDS_ERR_CUDA, "tile order table missing (handle not uploaded)");
  return PJDS_OK;
}

int set_tile_order_impl(int mode) {
  if (mode < 0 || mode > 3)
    return set_error(PJDS_ERR_INVALID_ARG, "tile order: 0 storage, 1 original-row, 2 auto, 3 warp-granular original-row");
  g_tile_order = mode;
  return PJDS_OK;
}
// 0 static CTA grid (default), 1 dynamic warp tiles.  Measured (profiles/r01_kbench_schedule.jsonl):
// dynamic is slower on every config -- C4 DP 80 -> 146 us, W4 DP 310 -> 540, C2 DP 58 -> 60,
// C5 DP 2045 -> 2184 -- because warp tiles handed out in arrival order scatter adjacent row tiles
// over different SMs, and the block-structured matrices (DLR1/DLR2: 6 or 5 consecutive rows share
// their x entries) lose the L1 reuse that a CTA of 8 adjacent warp tiles gets on one SM.
static int g_sched = 0;

int set_schedule_impl(int mode) {
  if (mode < 0 || mode > 1) return set_error(PJDS_ERR_INVALID_ARG, "schedule: 0 static, 1 dynamic warp tiles");
  g_sched = mode;
  return PJDS_OK;
}

static int num_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
  }
  return v;
}

// Launch the dynamic warp-tile kernel when the schedule asks for it.  *launched = false leaves the
// static launch to the caller.
template <typename T, typename Off, int R, int U, int M, bool PF, bool W>
int launch_dyn(const pjds_mat* A, T* y, const T* x, cudaStream_t s, const int* order, int64_t grid_static,
               bool* launched) {
  *launched = false;
  if (g_sched == 0) return PJDS_OK;
  static int occ = 0;
  auto kern = pjds_spmv_dyn_kernel<T, Off, R, U, M, PF, W>;
  if (!occ) {
    PJDS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
    occ = std::max(occ, 1);
  }
  const int64_t cap = (int64_t)num_sms() * occ;
  (void)grid_static;
  const auto& h = A->h;
  // warp-tile slots: every CTA tile of the order contributes kThreads/32 slots (the partial last
  // CTA tile can sit anywhere in the order; its slots past the matrix are skipped in the kernel)
  const int64_t wpt = kThreads / 32;
  const int64_t n_wtiles = (h.n_pad + 32 * R - 1) / (32 * R);
  const int64_t n_slots = (n_wtiles + wpt - 1) / wpt * wpt;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cap, n_slots / wpt));
  kern<<<(unsigned)grid, kThreads, 0, s>>>((const T*)A->d_val, A->d_col, A->d_col_start, A->d_block_len, A->d_perm, x,
                                           y, h.n, h.n_pad, h.br, g_pol, order, (const T* const*)A->d_win,
                                           A->win_shift, n_slots, A->d_sched, h.width);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  *launched = true;
  return PJDS_OK;
}

template <typename T, typename Off, int R, int U, int M>
int launch_dyn_any(const pjds_mat* A, T* y, const T* x, cudaStream_t s, const int* order, int64_t grid_static,
                   bool pipe, bool* launched) {
  *launched = false;
  if (A->d_win) {  // window matrices: y = A x only, 32-bit offsets (else the static path reports it)
    if constexpr (std::is_same<Off, int32_t>::value && M != STORE_PERM_ACC)
      return launch_dyn<T, Off, R, U, M, false, true>(A, y, x, s, order, grid_static, launched);
    return PJDS_OK;
  }
  if (pipe) return launch_dyn<T, Off, R, U, M, true, false>(A, y, x, s, order, grid_static, launched);
  return launch_dyn<T, Off, R, U, M, false, false>(A, y, x, s, order, grid_static, launched);
}

// Programmatic dependent launch of the static pJDS kernel (pjds_set_launch_overlap): 0 off, 1 on,
// 2 auto (default: grids of more than one wave; prefetch 2 columns, the best of 0/2/4/8/64 measured);
// g_pdl_pf = jagged columns of its val/col tile a first-wave warp prefetches into L2 while the
// previous grid drains (0 = none).
static int g_pdl = 2, g_pdl_pf = 2;

// first-wave CTA count of a kernel (SMs x resident CTAs), cached per kernel
template <typename K>
static int first_wave_ctas(K kern) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find((const void*)kern);
  if (it != cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0) != cudaSuccess || occ < 1) occ = 1;
  return cache[(const void*)kern] = num_sms() * occ;
}
// mode 2 (auto): early trigger on grids of more than one wave, late trigger (after the row chains)
// on one-wave grids.  A one-wave grid launched as an early-triggered dependent places its CTAs into
// whichever slots the previous grid frees first, unevenly over the SMs, where a plain launch spreads
// them evenly: measured C4 (DLR1, 544 CTAs on 740 slots) DP 80.7 -> 83.6 us, SP 63.0 -> 66.8; with
// the late trigger 81.6 -> 79.2 and 63.2 -> 61.0; the multi-wave C2 gains 4.5-9 % either way
// (profiles/r02_kbench_launch_overlap.jsonl, r02_kbench_launch_overlap_late.jsonl).
// 0 plain launch, 1 dependent launch with the trigger at kernel start, 2 trigger after the chains
template <typename K>
static int pdl_for(K kern, int64_t grid) {
  if (g_pdl == 0) return 0;
  if (g_pdl == 1) return 1;
  if (g_pdl == 3) return 2;
  return grid > first_wave_ctas(kern) ? 1 : 2;
}

// launch with or without cudaLaunchAttributeProgrammaticStreamSerialization
template <typename... P, typename... A>
static int launch_ex(void (*kern)(P...), int64_t grid, cudaStream_t s, bool pdl, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  PJDS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
  return PJDS_OK;
}

// the static pJDS kernel: launch_ex + its trailing (pf_cols, pf_ctas) parameters
template <typename... P, typename... A>
static int launch_pjds_kernel(void (*kern)(P...), int64_t grid, cudaStream_t s, bool pdl_ok, int pf_base, A&&... args) {
  const int pdl = pdl_ok ? pdl_for(kern, grid) : 0;
  const int pf_cols = pdl == 1 ? pf_base : 0;
  return launch_ex(kern, grid, s, pdl != 0, std::forward<A>(args)..., pf_cols,
                   pf_cols > 0 ? first_wave_ctas(kern) : 0, pdl == 2 ? 1 : 0);
}

static bool g_pipe = false;  // software-pipelined main loop (variant knob unroll + 16)
static bool g_il = false;    // lane-interleaved rows (variant knob unroll + 32; needs b_r % (32 R) == 0)

template <typename T, typename Off, int R, int U>
int launch_pjds_t(const pjds_mat* A, T* y, const T* x, cudaStream_t s, int mode, double* dot_part, int64_t* nparts,
                  bool pipe, bool il_req = false) {
  const auto& h = A->h;
  const int64_t threads = h.n_pad / R;
  const int64_t grid = (threads + kThreads - 1) / kThreads;
  if (nparts) *nparts = grid * (kThreads / 32);  // STORE_DIRECT_DOT: one partial per warp
  if (grid == 0) return PJDS_OK;
  const int* order = nullptr;
  // auto: original-row order when y is scattered through perm (keeps the stores of a region
  // together) or when x does not fit comfortably in L2 (measured: C5 DP permuted +6 %, rows-only
  // +44 %; C2/C4, whose x fits L2, lose ~1 % with it, so they keep storage order)
  const bool by_row = g_tile_order == 1 ||
                      (g_tile_order == 2 && h.n_windows <= 1 &&  // windowed sorts already run in row order
                       (mode == STORE_PERM || mode == STORE_PERM_ACC || A->ncols * (int64_t)sizeof(T) > (int64_t(64) << 20)));
  if (by_row) PJDS_TRY(tile_order_for(A, R, &order));
  // warp-granular order (mode 3; auto: the row-only / accumulate stores when no length class
  // dominates -- measured C5 DP rows-only 2384 -> 2256 us, C3 253 -> 238, C4 84 -> 81; the sAMG C2,
  // 96 % of rows in one class, loses 16 % with it, and the permuted basis loses 1-3 %)
  const bool il = il_req && R > 1 && h.br % (32 * R) == 0;
  const bool by_warp = (g_tile_order == 3 || (g_tile_order == 2 && A->mixed_classes &&
                                              (mode == STORE_PERM || mode == STORE_PERM_ACC))) &&
                       h.n_windows <= 1 && !A->d_win;
  const int* worder = by_warp ? A->d_worder[R == 4 ? 2 : (R == 2 ? 1 : 0)] : nullptr;
  const int64_t n_wtiles = (h.n_pad + 32 * R - 1) / (32 * R);
  // grids of a few waves: dynamic warp tiles (same row chains, bitwise the same y)
  if (A->d_sched && h.n_windows <= 1 && !(il_req && R > 1) && mode != STORE_DIRECT_DOT && !by_warp) {
    bool done = false;
int st;
    if (mode == STORE_DIRECT) st = launch_dyn_any<T, Off, R, U, STORE_DIRECT>(A, y, x, s, order, grid, pipe, &done);
    else if (mode == STORE_PERM_ACC) st = launch_dyn_any<T, Off, R, U, STORE_PERM_ACC>(A, y, x, s, order, grid, pipe, &done);
    else st = launch_dyn_any<T, Off, R, U, STORE_PERM>(A, y, x, s, order, grid, pipe, &done);
    if (st != PJDS_OK) return st;
    if (done) return PJDS_OK;
  }
  // per-handle y-store override (dist A_loc: its y is read again by the nonlocal pass), then the
  // vector y store needs y aligned to R elements (caller pointers need only T alignment)
  int pol = g_pol;
  if (A->y_store >= 0) pol = (pol & 0xff00ffff) | ((A->y_store & 0xff) << 16);
  if ((uintptr_t)y % (R * sizeof(T))) pol &= 0xff00ffff;
  // programmatic dependent launch for y = A x / y += A x (not the Lanczos dot product, whose
  // launches are captured into a graph with its reduce passes)
  const bool pdl_ok = mode != STORE_DIRECT_DOT;
  const int pf_base = h.n_windows <= 1 ? g_pdl_pf : 0;
#define PJDS_LAUNCH_W(M, PF, IL, W)                                                                      \
  PJDS_TRY(launch_pjds_kernel(pjds_spmv_kernel<T, Off, R, U, M, PF, IL, W>, grid, s, pdl_ok, pf_base,     \
      (const T*)A->d_val, (const int*)A->d_col, (const int64_t*)A->d_col_start, (const int*)A->d_block_len, \
      (const int*)A->d_perm, x, y, h.n, h.n_pad, (int)h.br, pol, order, dot_part, h.sigma,                  \
      (const int64_t*)A->d_wcs_off, (const T* const*)A->d_win, (int)A->win_shift, worder, n_wtiles))
#define PJDS_LAUNCH_PF(M, PF, IL) PJDS_LAUNCH_W(M, PF, IL, false)
  if (A->d_win) {  // fused remote-gather dist matrix: plain (or lane-interleaved) main loop, direct or perm store
    if constexpr (std::is_same<Off, int32_t>::value) {
      if (mode == STORE_DIRECT && il) PJDS_LAUNCH_W(STORE_DIRECT, false, true, true);
      else if (mode == STORE_DIRECT) PJDS_LAUNCH_W(STORE_DIRECT, false, false, true);
      else if (mode == STORE_PERM) PJDS_LAUNCH_W(STORE_PERM, false, false, true);
      else return set_error(PJDS_ERR_UNSUPPORTED, "window matrices support y = A x only");
      count_launch();
      PJDS_CUDA_TRY(cudaGetLastError());
      return PJDS_OK;
    } else {
      return set_error(PJDS_ERR_UNSUPPORTED, "window matrices need 32-bit jagged offsets");
    }
  }
#define PJDS_LAUNCH(M)                    \
  if (pipe) PJDS_LAUNCH_PF(M, true, false); \
  else if (il) PJDS_LAUNCH_PF(M, false, true); \
  else PJDS_LAUNCH_PF(M, false, false)
  if (mode == STORE_DIRECT) {
    PJDS_LAUNCH(STORE_DIRECT);
  } else if (mode == STORE_DIRECT_DOT) {
    PJDS_LAUNCH(STORE_DIRECT_DOT);
  } else if (mode == STORE_PERM_ACC) {
    PJDS_LAUNCH(STORE_PERM_ACC);
  } else {
    PJDS_LAUNCH(STORE_PERM);
  }
#undef PJDS_LAUNCH
#undef PJDS_LAUNCH_PF
#undef PJDS_LAUNCH_W
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

template <typename T, typename Off, int S, int U>
int launch_pjds_split_t(const pjds_mat* A, T* y, const T* x, cudaStream_t s, int mode, double* dot_part,
                        int64_t* nparts) {
  const auto& h = A->h;
  const int64_t grid = (h.n_pad * S + kThreads - 1) / kThreads;
  if (nparts) *nparts = grid;
  if (grid == 0) return PJDS_OK;
#define PJDS_LAUNCH_SPLIT(M)                                                                            \
  pjds_spmv_split_kernel<T, Off, S, U, M><<<(unsigned)grid, kThreads, 0, s>>>(                           \
      (const T*)A->d_val, A->d_col, A->d_col_start, A->d_block_len, A->d_perm, x, y, h.n, h.n_pad, h.br, g_pol, \
      dot_part, h.sigma, A->d_wcs_off)
  if (mode == STORE_DIRECT) PJDS_LAUNCH_SPLIT(STORE_DIRECT);
  else if (mode == STORE_DIRECT_DOT) PJDS_LAUNCH_SPLIT(STORE_DIRECT_DOT);
  else if (mode == STORE_PERM_ACC) PJDS_LAUNCH_SPLIT(STORE_PERM_ACC);
  else PJDS_LAUNCH_SPLIT(STORE_PERM);
#undef PJDS_LAUNCH_SPLIT
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

// kernel variant (rows per thread R, j-unroll U); 0 = automatic choice
static int g_var_r = 0, g_var_u = 0;
static int g_split = 0;  // > 0: long-row variant with S = g_split threads per row (knob rows_per_thread = 16 + S)
static bool g_force_off64 = false;  // test hook: exercise the 64-bit offset kernels on small inputs

template <typename T, typename Off>
int launch_pjds_off(const pjds_mat* A, void* y, const void* x, cudaStream_t s, int mode, double* dp, int64_t* np) {
  int R = g_var_r, U = g_var_u;
  bool pipe = g_pipe && !A->d_win;
  if (g_split && !A->d_win) {
    T* yy = (T*)y;
    const T* xx = (const T*)x;
    if (g_split == 2) return U >= 8 ? launch_pjds_split_t<T, Off, 2, 8>(A, yy, xx, s, mode, dp, np)
                                    : launch_pjds_split_t<T, Off, 2, 4>(A, yy, xx, s, mode, dp, np);
    if (g_split == 4) return U >= 8 ? launch_pjds_split_t<T, Off, 4, 8>(A, yy, xx, s, mode, dp, np)
                                    : launch_pjds_split_t<T, Off, 4, 4>(A, yy, xx, s, mode, dp, np);
    return launch_pjds_split_t<T, Off, 8, 4>(A, yy, xx, s, mode, dp, np);
  }
  bool il = g_il;
  if (R == 0) {
    // enough warps to cover the SMs several times: R = 4 (256-bit DP loads) for large matrices,
    // R = 2 / 1 when n_pad / R would leave the GPU short of warps (long-row matrices like DLR1)
    const int64_t np = A->h.n_pad;
    if (np / 4 >= (int64_t(1) << 19)) { R = 4; U = 2; }
    else if (np / 2 >= (int64_t(1) << 17)) { R = 2; U = 4; }
    else { R = 1; U = 8; }
    // long rows in SP (half the bytes per load): overlapping the next chunk's stream with the
    // current gathers pays (measured C4 SP +5 %, W4 SP +10 %; DP on C4 loses, so DP stays plain)
    pipe = sizeof(T) == 4 && R == 2;
    // DP, permuted basis, R = 4 with 128-row blocks: lane-interleaved rows (one gather instruction
    // covers 32 consecutive sorted rows).  With the index arrays compressed the kernel is no longer
    // at the DRAM ceiling and the 4x fewer L1 gather wavefronts pay: C5 DP 1943-1952 -> 1922 us,
    // C3 DP 190-192 -> 182.6, C2 DP 57.0 -> 53.6; SP loses on C3/C5 (115 -> 120, 1188 -> 1275)
    // (profiles/r02_kbench_variants_compress.jsonl)
    // SP: only when one length class holds >= 90 % of the rows (consecutive sorted rows are then
    // nearly consecutive original rows; sAMG C2 SP 35.1 -> 33.0 us), not on the mixed-class HMEp
    // The same rule for the row-only / y += stores, whose warp-granular order now takes interleaved
    // rows inside each warp tile, while x fits the 64 MB the tile-order rule uses: C3 DP 223 -> 215
    // us, C2 DP 65.2 -> 63.7, C2 SP 39.3 -> 37.6; on C5 (x 456 MB) neutral warm and 3.4 % slower cold
    // (2003 -> 2071 us under ncu), so plain there (profiles/r02_kbench_rows_il_worder.jsonl)
    const bool perm_store = mode == STORE_PERM || mode == STORE_PERM_ACC;
    il = il || ((sizeof(T) == 8 || !A->mixed_classes) && R == 4 && A->h.br % 128 == 0 && A->h.n_windows <= 1 &&
                (!perm_store || A->ncols * (int64_t)sizeof(T) <= (int64_t(64) << 20)));
  }
  while (A->h.br % R) R >>= 1;  // R must divide b_r
  T* yy = (T*)y;
  const T* xx = (const T*)x;
  if (R == 4)
    return U >= 4 ? launch_pjds_t<T, Off, 4, 4>(A, yy, xx, s, mode, dp, np, pipe, il)
                  : launch_pjds_t<T, Off, 4, 2>(A, yy, xx, s, mode, dp, np, pipe, il);
  if (R == 2)
    return U >= 8 ? launch_pjds_t<T, Off, 2, 8>(A, yy, xx, s, mode, dp, np, pipe, il)
                  : launch_pjds_t<T, Off, 2, 4>(A, yy, xx, s, mode, dp, np, pipe, il);
  return launch_pjds_t<T, Off, 1, 8>(A, yy, xx, s, mode, dp, np, pipe, il);
}

template <typename T>
int launch_pjds_dt(const pjds_mat* A, void* y, const void* x, cudaStream_t s, int mode, double* dp = nullptr,
                   int64_t* np = nullptr) {
  const bool off32 = !g_force_off64 && A->h.stored + A->h.n_pad < (int64_t(1) << 31);
  if (off32) return launch_pjds_off<T, int32_t>(A, y, x, s, mode, dp, np);
  return launch_pjds_off<T, int64_t>(A, y, x, s, mode, dp, np);
}

// ---- ELLPACK-R kernel ------------------------------------------------------------------------
// Consecutive rows to consecutive threads, R consecutive rows per thread with
// vector loads of val[j*N_pad + i .. +R-1]; each row stops at its own rowmax[i] ("threads only
// execute non-zero contributions", L187-191); lanes of a warp diverge at the tail, so the warp
// stays resident until its longest row is done (the "hardware reservation" of Fig. 2b).
template <typename T, int R, int U>
__global__ void __launch_bounds__(kThreads)
ellr_spmv_kernel(const T* __restrict__ val, const int* __restrict__ col, const int* __restrict__ rowmax,
                 const T* __restrict__ x, T* __restrict__ y, int64_t n, int64_t n_pad, int trig_late) {
  if (!trig_late) pdl_trigger();  // programmatic dependent launch, as in the pJDS kernel (no prefetch)
  const int64_t i0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * R;
  if (i0 >= n_pad) return;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_x = policy_evict_last();
  Vec<int, R> lens;
  lens.load(rowmax + i0, pol_s);
  pdl_wait();
  int tmax = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) tmax = max(tmax, lens.v[r]);
  // one predicated loop to the warp's longest row keeps the lanes converged; measured faster than
  // an unpredicated per-thread main loop + tail (which diverges inside mixed-length warps)
  const int wmax = __reduce_max_sync(__activemask(), tmax);
  T acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = T(0);
  for (int j = 0; j < wmax; j += U) {
    Vec<T, R> v[U];
    Vec<int, R> c[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < tmax) {
        const int64_t off = (int64_t)(j + u) * n_pad + i0;
        v[u].load(val + off, pol_s);
        c[u].load(col + off, pol_s);
      }
    T xv[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (j + u < lens.v[r]) xv[u][r] = ld_rhs(x + c[u].v[r], pol_x);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (j + u < lens.v[r]) acc[r] = fma_rn(v[u].v[r], xv[u][r], acc[r]);
  }
  if (trig_late) pdl_trigger();
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (i0 + r < n) y[i0 + r] = acc[r];
}

// basis change: to permuted dst[k] = src[perm[k]]; back dst[perm[k]] = src[k]
template <typename T>
__global__ void permute_kernel(const int* __restrict__ perm, int64_t n, const T* __restrict__ src, T* __restrict__ dst,
                               int back) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    if (back) dst[perm[k]] = src[k];
    else dst[k] = src[perm[k]];
  }
}

template <typename T>
__global__ void pack_kernel(const int* __restrict__ idx, int64_t count, const T* __restrict__ x, T* __restrict__ buf) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = x[idx[i]];
}

// ---- bandwidth probe -------------------------------------------------------------------------
__global__ void copy_kernel(const int4* __restrict__ a, int4* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void read_kernel(const int4* __restrict__ a, int64_t n, int* __restrict__ out) {
  int acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = a[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;  // practically never; keeps the loads alive
}

}  // namespace

// Tiles (CTAs of 256 R consecutive sorted rows) ordered by the original index of their first row,
// one table per rows-per-thread variant R in {1, 2, 4}; built once at upload.
// Tile execution orders for R = 1, 2, 4: tiles sorted (stably) by the key of their first row's
// original index — the index itself by default, or a caller key per original row
// (pjds_set_tile_keys).  Only the order of independent CTAs changes, never a result.
int build_tile_orders(pjds_mat* A, const int64_t* row_key) {
  const auto& h = A->h;
  const int Rs[3] = {1, 2, 4};
  for (int slot = 0; slot < 3; ++slot) {
    const int64_t rows = (int64_t)kThreads * Rs[slot];
    const int64_t tiles = std::max<int64_t>((h.n_pad + rows - 1) / rows, 1);
    std::vector<int64_t> key(tiles);
    for (int64_t t = 0; t < tiles; ++t) {
      const int64_t k = t * rows;
      key[t] = k < h.n ? (row_key ? row_key[h.perm[k]] : (int64_t)h.perm[k]) : INT64_MAX;
    }
    std::vector<int32_t> ord(tiles);
    for (int64_t t = 0; t < tiles; ++t) ord[t] = (int32_t)t;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    if (!A->d_order[slot]) PJDS_CUDA_TRY(cudaMalloc(&A->d_order[slot], tiles * 4));
    PJDS_CUDA_TRY(cudaMemcpy(A->d_order[slot], ord.data(), tiles * 4, cudaMemcpyHostToDevice));
    // the same key at warp-tile granularity (32 R rows)
    const int64_t wrows = 32 * Rs[slot];
    const int64_t wt = std::max<int64_t>((h.n_pad + wrows - 1) / wrows, 1);
    std::vector<int64_t> wkey(wt);
    for (int64_t t = 0; t < wt; ++t) {
      const int64_t k = t * wrows;
      wkey[t] = k < h.n ? (row_key ? row_key[h.perm[k]] : (int64_t)h.perm[k]) : INT64_MAX;
    }
    std::vector<int32_t> word(wt);
    for (int64_t t = 0; t < wt; ++t) word[t] = (int32_t)t;
    std::stable_sort(word.begin(), word.end(), [&](int32_t a, int32_t b) { return wkey[a] < wkey[b]; });
    if (!A->d_worder[slot]) PJDS_CUDA_TRY(cudaMalloc(&A->d_worder[slot], wt * 4));
    PJDS_CUDA_TRY(cudaMemcpy(A->d_worder[slot], word.data(), wt * 4, cudaMemcpyHostToDevice));
  }
  return PJDS_OK;
}

int launch_pjds_spmv(const pjds_mat* A, void* y, const void* x, cudaStream_t s, bool accumulate) {
  const int mode = accumulate ? STORE_PERM_ACC : (A->direct_store ? STORE_DIRECT : STORE_PERM);
  if (A->h.dtype == PJDS_F64) return launch_pjds_dt<double>(A, y, x, s, mode);
  return launch_pjds_dt<float>(A, y, x, s, mode);
}

int launch_pjds_spmv_dot(const pjds_mat* A, void* y, const void* x, cudaStream_t s, double* part, int64_t* nparts) {
  if (!A->direct_store) return set_error(PJDS_ERR_INVALID_ARG, "fused dot needs the permuted basis");
  if (A->h.dtype == PJDS_F64) return launch_pjds_dt<double>(A, y, x, s, STORE_DIRECT_DOT, part, nparts);
  return launch_pjds_dt<float>(A, y, x, s, STORE_DIRECT_DOT, part, nparts);
}

int set_tile_order(int mode) { return set_tile_order_impl(mode); }
int set_schedule(int mode) { return set_schedule_impl(mode); }
int set_launch_overlap(int mode, int prefetch_cols) {
  if (mode < 0 || mode > 3)
    return set_error(PJDS_ERR_INVALID_ARG,
                     "launch overlap: mode 0 off, 1 dependent launch (early trigger), 2 auto, 3 dependent launch (late trigger)");
  if (prefetch_cols < 0 || prefetch_cols > 64) return set_error(PJDS_ERR_INVALID_ARG, "launch overlap: prefetch_cols in [0, 64]");
  g_pdl = mode;
  g_pdl_pf = prefetch_cols;
  return PJDS_OK;
}

int set_cache_policy(int stream_kind, int x_kind) {
  // bits 8-15 of stream_kind: y store of the permuted-basis kernel (0 plain scalar stores,
  // 1 + kind: one R-wide vector store with that L2 policy; default 2 = vector, evict_first);
  // bits 16-23: the scattered stores through perm (row-only basis, dist nonlocal +=): 0 plain
  // (default), 1 + kind: L1::no_allocate store (and load for +=) with that L2 policy
  const int y_kind = (stream_kind >> 8) & 0xff;
  const int p_kind = (stream_kind >> 16) & 0xff;
  stream_kind &= 0xff;
  if (stream_kind > 3 || x_kind < 0 || x_kind > 3 || y_kind > 4 || p_kind > 4)
    return set_error(PJDS_ERR_INVALID_ARG, "cache policy kinds: 0 normal, 1 evict_first, 2 evict_last, 3 unchanged");
  g_pol = stream_kind | (x_kind << 8) | (y_kind << 16) | (p_kind << 24);
  return PJDS_OK;
}

int set_kernel_variant(int r, int u) {
  // r >= 16: long-row split-j kernel with S = r - 16 threads per row (2, 4 or 8; unroll 4 or 8)
  if (r >= 16) {
    const int S = r - 16;
    if (!((S == 2 || S == 4) && (u == 4 || u == 8)) && !(S == 8 && u == 4))
      return set_error(PJDS_ERR_INVALID_ARG, "split variant: threads per row 2 or 4 with unroll 4 or 8, or 8 with 4");
    g_split = S;
    g_var_r = 0;
    g_var_u = u;
    g_pipe = false;
    g_il = false;
    g_force_off64 = false;
    return PJDS_OK;
  }
  // u >= 32: lane-interleaved rows (u - 32); u >= 16 encodes "software-pipelined main loop" (u - 16)
  const bool il = u >= 32;
  if (u >= 32) u -= 32;
  const bool pf = u >= 16;
  if (u >= 16) u -= 16;
  const bool off64 = r >= 8;  // rows_per_thread + 8: force 64-bit jagged offsets
  if (r >= 8) r -= 8;
  if (!((r == 0 && u == 0) || ((r == 1 || r == 2 || r == 4) && (u == 2 || u == 4 || u == 8))))
    return set_error(PJDS_ERR_INVALID_ARG, "variant: rows_per_thread in {1,2,4}, unroll in {2,4,8} (or 0,0)");
  g_split = 0;
  g_var_r = r;
  g_var_u = u;
  g_pipe = pf;
  g_il = il;
  g_force_off64 = off64;
  return PJDS_OK;
}

template <typename T, int R, int U>
int launch_ellr_t(const ellr_mat* A, void* y, const void* x, cudaStream_t s) {
  const auto& h = A->h;
  const int64_t grid = (h.n_pad / R + kThreads - 1) / kThreads;
  if (grid == 0) return PJDS_OK;
  const int pdl = pdl_for(ellr_spmv_kernel<T, R, U>, grid);
  PJDS_TRY(launch_ex(ellr_spmv_kernel<T, R, U>, grid, s, pdl != 0, (const T*)A->d_val, (const int*)A->d_col,
                     (const int*)A->d_rowmax, (const T*)x, (T*)y, h.n, h.n_pad, pdl == 2 ? 1 : 0));
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

template <typename T>
int launch_ellr_dt(const ellr_mat* A, void* y, const void* x, cudaStream_t s) {
  int R = g_var_r;
  if (R == 0) {
    // ELLPACK-R's own sweep (profiles/r01_kbench_ellr_variants.jsonl): R=4,U=2 is fastest on
    // C2/C3/C5 in SP and DP and on the DLR1-shaped C4 in DP (114.9 vs 127.3 us at R=2, 178.8 at
    // R=1); C4 SP keeps R=2 (68.2 vs 76.1 us at R=4)
    const int64_t np = A->h.n_pad;
    const int64_t r4_rows = sizeof(T) == 8 ? (int64_t(1) << 16) : (int64_t(1) << 19);
    R = np / 4 >= r4_rows ? 4 : (np / 2 >= (int64_t(1) << 17) ? 2 : 1);
  }
  if (R == 4) return launch_ellr_t<T, 4, 2>(A, y, x, s);
  if (R == 2) return launch_ellr_t<T, 2, 4>(A, y, x, s);
  return launch_ellr_t<T, 1, 8>(A, y, x, s);
}

int launch_ellr_spmv(const ellr_mat* A, void* y, const void* x, cudaStream_t s) {
  if (A->h.dtype == PJDS_F64) return launch_ellr_dt<double>(A, y, x, s);
  return launch_ellr_dt<float>(A, y, x, s);
}

int launch_permute(const int32_t* perm, int64_t n, const void* src, void* dst, int dtype, int back, cudaStream_t s) {
  if (n <= 0) return PJDS_OK;
  const int64_t grid = std::min<int64_t>((n + 255) / 256, 148 * 32);
  if (dtype == PJDS_F64)
    permute_kernel<double><<<(unsigned)grid, 256, 0, s>>>(perm, n, (const double*)src, (double*)dst, back);
  else
    permute_kernel<float><<<(unsigned)grid, 256, 0, s>>>(perm, n, (const float*)src, (float*)dst, back);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int launch_pack(const int32_t* idx, int64_t count, const void* x, void* buf, int dtype, cudaStream_t s) {
  if (count <= 0) return PJDS_OK;
  const int64_t grid = std::min<int64_t>((count + 255) / 256, 148 * 16);
  if (dtype == PJDS_F64)
    pack_kernel<double><<<(unsigned)grid, 256, 0, s>>>(idx, count, (const double*)x, (double*)buf);
  else
    pack_kernel<float><<<(unsigned)grid, 256, 0, s>>>(idx, count, (const float*)x, (float*)buf);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int launch_copy16(const void* src, void* dst, size_t bytes, cudaStream_t s) {
  const int64_t n = (int64_t)(bytes / 16);
  if (!n) return PJDS_OK;
  const int64_t grid = std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(148) * 16);
  copy_kernel<<<(unsigned)grid, kThreads, 0, s>>>((const int4*)src, (int4*)dst, n);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int bw_probe(int64_t bytes, int reps, double* copy_gbs, double* read_gbs) {
  if (bytes < (1 << 20) || reps < 1) return set_error(PJDS_ERR_INVALID_ARG, "bw_probe: bytes >= 1 MiB, reps >= 1");
  int64_t n = bytes / 16;
  int4 *a = nullptr, *b = nullptr;
  int* o = nullptr;
  PJDS_CUDA_TRY(cudaMalloc(&a, n * 16));
  if (cudaMalloc(&b, n * 16) != cudaSuccess || cudaMalloc(&o, 16) != cudaSuccess) {
    cudaFree(a); cudaFree(b);
    return set_error(PJDS_ERR_OOM, "bw_probe: cudaMalloc failed");
  }
  cudaMemset(a, 1, n * 16);
  cudaMemset(b, 0, n * 16);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_c = 1e30f, best_r = 1e30f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<grid, 256>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best_c = std::min(best_c, ms);
    cudaEventRecord(e0);
    read_kernel<<<grid, 256>>>(b, n, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best_r = std::min(best_r, ms);
  }
  count_launch(2 * (reps + 1));
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(a); cudaFree(b); cudaFree(o);
  if (err != cudaSuccess) return set_error(PJDS_ERR_CUDA, std::string("bw_probe: ") + cudaGetErrorString(err));
  *copy_gbs = 2.0 * n * 16 / (best_c * 1e-3) / 1e9;
  *read_gbs = 1.0 * n * 16 / (best_r * 1e-3) / 1e9;
  return PJDS_OK;
}

}  // namespace pjds

extern "C" int64_t pjds_launch_count(void) { return pjds::g_launches.load(); }
