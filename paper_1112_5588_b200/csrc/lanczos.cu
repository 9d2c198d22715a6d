// Lanczos driver in the permuted basis: the eigensolver usage the paper's
// HMEp matrix comes from (PAPER.md L94-101 Holstein-Hubbard; L521-525 "production-grade
// eigensolver") run entirely on permuted vectors, with the basis change only before the first and
// after the last step.
//
// Recurrence (symmetric A, v_0 = v0 / ||v0||, beta_{-1} = 0):
//   w = A v_j ; alpha_j = w . v_j ; w -= alpha_j v_j + beta_{j-1} v_{j-1} ; beta_j = ||w|| ;
//   v_{j+1} = w / beta_j.
// Stored vectors are unnormalised u_j with v_j = c_j u_j (c_j = 1 / ||u_j||), so no separate
// scaling pass is needed:
//   K1  y = A u_j, with per-CTA partial sums of y . u_j fused into the pJDS kernel's epilogue
//       (STORE_DIRECT_DOT: in the permuted basis u_j[k] is the input entry of row k)
//   R1  alpha_j = c_j^2 * sum                      (148 CTAs + last-CTA sum, fixed order: deterministic)
//   K3  u_{j+1} = c_j y - alpha_j c_j u_j - beta_{j-1} c_{j-1} u_{j-1}  (in place of u_{j-1}),
//       partial sums of u_{j+1} . u_{j+1}
//   R2  beta_j = sqrt(sum), c_{j+1} = 1 / beta_j  (fused into K3: its last CTA to finish)
// All m iterations are captured once into a CUDA graph and launched on the caller's stream.
// Dot products accumulate in double for both SP and DP vectors.
#include <algorithm>
#include <cmath>
#include <vector>
#include "internal.h"

namespace pjds {
namespace {

constexpr int kRedThreads = 256;
constexpr int kRedCTAs = 148 * 8;  // vector passes: 8 CTAs per SM, 4 elements in flight per thread
constexpr int kAlphaCTAs = 148;    // R1: one CTA per SM, then one CTA sums their 148 results

__device__ __forceinline__ double block_sum(double v, double* sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // valid in thread 0
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) dot_partials(const T* __restrict__ a, const T* __restrict__ b, int64_t n,
                                                            double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma((double)a[i], (double)b[i], s);
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// scal layout: c[j] at scal[j] (j = 0..m), alpha[j] at scal[(m+1) + j], beta[j] at scal[(m+1)+m + j]
// One CTA sums the np partials in a fixed order (deterministic).  Eight independent loads per
// thread per round: a plain strided loop waits one L2 round trip per element (C5: 55.7 K
// partials of the product's CTAs took 28 us; measured with tools/lanczos_bench.py)
// CG: L2-coherent loads (__ldcg) for partials written by other CTAs of the running grid.
template <bool CG = false>
__device__ __forceinline__ double sum_partials(const double* part, int np, double* sm) {
  constexpr int kIn = 8;
  double s[kIn];
#pragma unroll
  for (int q = 0; q < kIn; ++q) s[q] = 0.0;
  const int bd = blockDim.x;
  int i = threadIdx.x;
  for (; i + (kIn - 1) * bd < np; i += kIn * bd) {
    double v[kIn];
#pragma unroll
    for (int q = 0; q < kIn; ++q) v[q] = CG ? __ldcg(part + i + q * bd) : part[i + q * bd];
#pragma unroll
    for (int q = 0; q < kIn; ++q) s[q] += v[q];
  }
  for (; i < np; i += bd) s[0] += CG ? __ldcg(part + i) : part[i];  // < kIn ragged rounds
  const double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  return block_sum(t, sm);  // valid in thread 0
}

// R1 over many CTAs: CTA b sums its contiguous chunk of the product's partials, the last CTA to
// finish sums the per-CTA results (fixed order: deterministic) and writes alpha_j
__global__ void __launch_bounds__(kRedThreads) reduce_alpha(const double* __restrict__ part, int np, double* part2,
                                                             unsigned* ctr, double* scal, int m, int j) {
  __shared__ double sm[32];
  __shared__ bool last;
  const int chunk = (np + gridDim.x - 1) / gridDim.x;
  const int lo = min(np, (int)blockIdx.x * chunk), hi = min(np, lo + chunk);
  const double s = sum_partials(part + lo, hi - lo, sm);
  if (threadIdx.x == 0) {
    part2[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double t = sum_partials<true>(part2, gridDim.x, sm);
  if (threadIdx.x == 0) {
    const double c = scal[j];
    scal[(m + 1) + j] = t * c * c;
    *ctr = 0u;
  }
}

// u_next (aliases u_prev) = c_j y - alpha_j c_j u_j - beta_{j-1} c_{j-1} u_prev ; partial |u_next|^2
template <typename T>
__global__ void __launch_bounds__(kRedThreads) lanczos_update(const T* __restrict__ y, const T* __restrict__ u,
                                                              T* u_prev_next, int64_t n, double* scal,
                                                              int m, int j, double* part, unsigned* ctr) {
  __shared__ double sm[32];
  const double cj = scal[j];
  const double aj = scal[(m + 1) + j];
  const double cp = j > 0 ? scal[j - 1] : 0.0;
  const double bp = j > 0 ? scal[(m + 1) + m + (j - 1)] : 0.0;
  const double ka = cj, kb = -aj * cj, kc = -bp * cp;
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // 4 independent elements in flight per thread
    T yv[4], uv[4], pv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      yv[q] = y[i + q * stride];
      uv[q] = u[i + q * stride];
      pv[q] = j > 0 ? u_prev_next[i + q * stride] : T(0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const T vt = (T)(ka * (double)yv[q] + kb * (double)uv[q] + kc * (double)pv[q]);
      u_prev_next[i + q * stride] = vt;
      s = fma((double)vt, (double)vt, s);
    }
  }
  for (; i < n; i += stride) {
    const double up = j > 0 ? (double)u_prev_next[i] : 0.0;
    const T vt = (T)(ka * (double)y[i] + kb * (double)u[i] + kc * up);
    u_prev_next[i] = vt;
    s = fma((double)vt, (double)vt, s);
  }
  s = block_sum(s, sm);
  // R2 fused: the last CTA to finish sums the partials (fixed order) and writes beta_j, c_{j+1}
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double t = sum_partials<true>(part, gridDim.x, sm);
  if (threadIdx.x == 0) {
    const double b = sqrt(t);
    scal[(m + 1) + m + j] = b;
    scal[j + 1] = b > 0.0 ? 1.0 / b : 0.0;
    *ctr = 0u;  // ready for the next step's launch
  }
}

__global__ void init_c0(const double* __restrict__ part, int np, double* scal) {
  __shared__ double sm[32];
  const double s = sum_partials(part, np, sm);
  if (threadIdx.x == 0) scal[0] = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
}

template <typename T>
int lanczos_t(pjds_mat* A, const void* v0, int m, double* alpha, double* beta, int* steps, cudaStream_t user) {
  const int64_t n = A->h.n;
  const size_t vb = (size_t)n * sizeof(T);
  T *u0 = nullptr, *u1 = nullptr, *y = nullptr;
  double *part = nullptr, *scal = nullptr;
  unsigned* ctr = nullptr;
  cudaStream_t s = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int st = PJDS_OK;
  auto cleanup = [&]() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (s) cudaStreamDestroy(s);
    cudaFree(u0); cudaFree(u1); cudaFree(y); cudaFree(part); cudaFree(scal); cudaFree(ctr);
  };
#define LZ_TRY(expr)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      st = set_error(e_ == cudaErrorMemoryAllocation ? PJDS_ERR_OOM : PJDS_ERR_CUDA,   \
                     std::string("lanczos: ") + #expr + ": " + cudaGetErrorString(e_)); \
      cleanup();                                                                       \
      return st;                                                                       \
    }                                                                                  \
  } while (0)
  LZ_TRY(cudaMalloc(&u0, vb ? vb : 16));
  LZ_TRY(cudaMalloc(&u1, vb ? vb : 16));
  LZ_TRY(cudaMalloc(&y, vb ? vb : 16));
  // product partials: one per warp (<= n_pad / 32 + 8) or one per CTA of the split kernel (<= n_pad / 32)
  const int64_t np_max = std::max<int64_t>(kRedCTAs, A->h.n_pad / 32 + 64);
  LZ_TRY(cudaMalloc(&part, (np_max + kAlphaCTAs) * sizeof(double)));  // + R1's second level
  LZ_TRY(cudaMalloc(&scal, (size_t)(3 * m + 1) * sizeof(double)));
  LZ_TRY(cudaMalloc(&ctr, 2 * sizeof(unsigned)));  // [0] update (R2), [1] reduce_alpha (R1)
  LZ_TRY(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned), user));
  LZ_TRY(cudaMemsetAsync(scal, 0, (size_t)(3 * m + 1) * sizeof(double), user));
  LZ_TRY(cudaMemcpyAsync(u0, v0, vb, cudaMemcpyDeviceToDevice, user));
  // prepare lazily-built kernel state (tile order) outside the capture
  if ((st = launch_pjds_spmv(A, y, u0, user, false)) != PJDS_OK) { cleanup(); return st; }
  LZ_TRY(cudaStreamSynchronize(user));
  LZ_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  LZ_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  dot_partials<T><<<kRedCTAs, kRedThreads, 0, s>>>(u0, u0, n, part);
  init_c0<<<1, 1024, 0, s>>>(part, kRedCTAs, scal);
  T* uj = u0;
  T* up = u1;
  for (int j = 0; j < m; ++j) {
    int64_t np = 0;
    if ((st = launch_pjds_spmv_dot(A, y, uj, s, part, &np)) != PJDS_OK) {
      cudaStreamEndCapture(s, &graph);
      cleanup();
      return st;
    }
    reduce_alpha<<<kAlphaCTAs, kRedThreads, 0, s>>>(part, (int)np, part + np_max, ctr + 1, scal, m, j);
    lanczos_update<T><<<kRedCTAs, kRedThreads, 0, s>>>(y, uj, up, n, scal, m, j, part, ctr);
    std::swap(uj, up);
  }
  count_launch(2 + 3 * (int64_t)m - m);
  LZ_TRY(cudaStreamEndCapture(s, &graph));
  LZ_TRY(cudaGraphInstantiate(&exec, graph, 0));
  LZ_TRY(cudaGraphLaunch(exec, user));
  std::vector<double> h(3 * m + 1);
  LZ_TRY(cudaMemcpyAsync(h.data(), scal, h.size() * sizeof(double), cudaMemcpyDeviceToHost, user));
  LZ_TRY(cudaStreamSynchronize(user));
#undef LZ_TRY
  if (!(h[0] > 0.0)) {  // scal[0] = 1/||v0||, 0 when v0 = 0 (or non-finite)
    cleanup();
    return set_error(PJDS_ERR_INVALID_ARG, "pjds_lanczos: v0 has zero (or non-finite) norm");
  }
  int done = m;
  for (int j = 0; j < m; ++j) {
    alpha[j] = h[(m + 1) + j];
    beta[j] = h[(m + 1) + m + j];
    if (!(beta[j] > 0.0) && done == m) done = j + 1;  // breakdown: invariant subspace found
  }
  if (steps) *steps = done;
  cleanup();
  return PJDS_OK;
}

}  // namespace

// Eigenvalues of the symmetric tridiagonal matrix (diag alpha[0..m), off-diag beta[0..m-1)) by
// Sturm-sequence bisection (Gerschgorin interval, ascending output).
int tridiag_eigenvalues(int m, const double* a, const double* b, double* ev) {
  if (m <= 0) return PJDS_OK;
  double lo = a[0], hi = a[0];
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i < m - 1 ? std::fabs(b[i]) : 0.0);
    lo = std::fmin(lo, a[i] - r);
    hi = std::fmax(hi, a[i] + r);
  }
  const double span = std::fmax(hi - lo, 1e-300);
  // number of eigenvalues < x
  auto count = [&](double x) {
    int c = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      const double bb = i > 0 ? b[i - 1] * b[i - 1] : 0.0;
      q = a[i] - x - (i > 0 ? bb / q : 0.0);
      if (q == 0.0) q = -1e-300 * span;
      if (q < 0.0) ++c;
    }
    return c;
  };
  for (int k = 0; k < m; ++k) {
    double l = lo, h = hi;
    for (int it = 0; it < 200 && h - l > 4e-16 * std::fmax(std::fabs(l), std::fabs(h)) + 1e-300; ++it) {
      const double mid = 0.5 * (l + h);
      if (count(mid) > k) h = mid;
      else l = mid;
    }
    ev[k] = 0.5 * (l + h);
  }
  return PJDS_OK;
}

int lanczos(pjds_mat* A, const void* v0, int m, double* alpha, double* beta, int* steps, cudaStream_t s) {
  if (A->h.dtype == PJDS_F64) return lanczos_t<double>(A, v0, m, alpha, beta, steps, s);
  return lanczos_t<float>(A, v0, m, alpha, beta, steps, s);
}

}  // namespace pjds

extern "C" {

int pjds_lanczos(pjds_t A, const void* v0, int32_t m, double* alpha, double* beta, int32_t* steps_done, void* stream) {
  if (!A || !v0 || !alpha || !beta || m < 1) return pjds::set_error(PJDS_ERR_INVALID_ARG, "pjds_lanczos: bad argument");
  if (!A->on_device) return pjds::set_error(PJDS_ERR_INVALID_ARG, "pjds_lanczos: handle is host-only");
  if (!(A->flags & PJDS_PERM_SYMMETRIC))
    return pjds::set_error(PJDS_ERR_INVALID_ARG, "pjds_lanczos: needs a PJDS_PERM_SYMMETRIC (permuted-basis) handle");
  pjds::DeviceGuard dg(A->device);
  return pjds::lanczos(A, v0, m, alpha, beta, steps_done, (cudaStream_t)stream);
}

int pjds_tridiag_eigenvalues(int32_t m, const double* alpha, const double* beta, double* evals) {
  if (m < 0 || (m > 0 && (!alpha || !evals || (m > 1 && !beta))))
    return pjds::set_error(PJDS_ERR_INVALID_ARG, "pjds_tridiag_eigenvalues: bad argument");
  return pjds::tridiag_eigenvalues(m, alpha, beta, evals);
}

}  // extern "C"
