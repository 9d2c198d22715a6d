// P2P transport of the distributed spMVM: the "local gather" of PAPER.md
// Fig. 4 (L401-402) and the halo transfer fused into ONE kernel that stores each send entry
// straight into the receiving rank's halo buffer through a CUDA-IPC mapping of the peer's memory
// (NVLink P2P stores between GPUs of one node; plain device stores between processes that share a
// GPU).  No NCCL on the per-call path, no send buffer, no SMs spent in a collective library.
//
// Per rank, one IPC-exported region: [halo buffer 0][halo buffer 1][ready[R] u64][done[R] u64][err].
// Call s (1, 2, ...) uses halo buffer s % 2:
//   comm stream   : wait done[q] >= s-2 for every receiver q (q finished reading buffer s%2 of call
//                   s-2), pack_put (x[send ids] -> q's halo, buffer s%2), signal ready[r] = s at q
//   compute stream: A_loc || ... ; wait own pack (event) ; wait ready[p] >= s for every sender p ;
//                   A_nl on halo buffer s%2 ; signal done[r] = s at every sender p
// Signals are system-scope release stores after __threadfence_system(); waits are acquire loads
// with a bounded spin (the err word records a timeout instead of hanging the GPU).
// The DIRECT transport (dist.cpp) reuses the flags with p2p_signal_wait_kernel: "my x window holds
// call s" out + the owners' "ready" in before its kernel, "done reading" out + the readers' "done"
// in after it.
#include <algorithm>
#include <cstring>
#include "internal.h"

namespace pjds {
namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one thread per awaited flag; gives up after ~10 s of spinning and records it in *err
__global__ void p2p_wait_kernel(const uint64_t* flags, const int* peers, int np, uint64_t target, unsigned* err) {
  const int i = threadIdx.x;
  if (i >= np) return;
  const uint64_t* f = flags + peers[i];
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < target) {
    if (clock64() - t0 > 20000000000LL) {
      atomicExch(err, 1u);
      return;
    }
    __nanosleep(200);
  }
}

__global__ void p2p_signal_kernel(uint64_t* const* targets, int nt, uint64_t value) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int i = 0; i < nt; ++i) st_release_sys(targets[i], value);
}

// signal, then wait, in one launch (DIRECT transport: "ready" out / owners' "ready" in, and
// "done" out / readers' "done" in)
__global__ void p2p_signal_wait_kernel(uint64_t* const* targets, int nt, uint64_t value, const uint64_t* flags,
                                       const int* peers, int np, uint64_t target, unsigned* err) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < nt; ++i) st_release_sys(targets[i], value);
  }
  __syncthreads();
  const int i = threadIdx.x;
  if (i >= np) return;
  const uint64_t* f = flags + peers[i];
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < target) {
    if (clock64() - t0 > 20000000000LL) {
      atomicExch(err, 1u);
      return;
    }
    __nanosleep(200);
  }
}

// blockIdx.y = send peer; entries [seg[p], seg[p+1]) of idx go to dst[p][0 .. count)
template <typename T>
__global__ void p2p_pack_put_kernel(const T* __restrict__ x, const int* __restrict__ idx,
                                    const int64_t* __restrict__ seg, T* const* __restrict__ dst) {
  const int p = blockIdx.y;
  const int64_t a = seg[p], b = seg[p + 1];
  T* d = dst[p];
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
    d[i - a] = x[idx[i]];
}

}  // namespace

int p2p_launch_wait(const uint64_t* flags, const int* peers, int np, uint64_t target, unsigned* err, cudaStream_t s) {
  if (np <= 0) return PJDS_OK;
  p2p_wait_kernel<<<1, 64, 0, s>>>(flags, peers, np, target, err);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int p2p_launch_signal(uint64_t* const* targets, int nt, uint64_t value, cudaStream_t s) {
  if (nt <= 0) return PJDS_OK;
  p2p_signal_kernel<<<1, 32, 0, s>>>(targets, nt, value);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int p2p_launch_signal_wait(uint64_t* const* targets, int nt, uint64_t value, const uint64_t* flags, const int* peers,
                           int np, uint64_t target, unsigned* err, cudaStream_t s) {
  if (nt <= 0 && np <= 0) return PJDS_OK;
  p2p_signal_wait_kernel<<<1, 64, 0, s>>>(targets, nt, value, flags, peers, np, target, err);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

int p2p_launch_pack_put(const void* x, const int* idx, const int64_t* seg, void* const* dst, int npeers,
                        int64_t max_count, int dtype, cudaStream_t s) {
  if (npeers <= 0 || max_count <= 0) return PJDS_OK;
  const unsigned gx = (unsigned)std::min<int64_t>((max_count + 255) / 256, 148 * 4);
  dim3 grid(gx, npeers);
  if (dtype == PJDS_F64)
    p2p_pack_put_kernel<double><<<grid, 256, 0, s>>>((const double*)x, idx, seg, (double* const*)dst);
  else
    p2p_pack_put_kernel<float><<<grid, 256, 0, s>>>((const float*)x, idx, seg, (float* const*)dst);
  count_launch();
  PJDS_CUDA_TRY(cudaGetLastError());
  return PJDS_OK;
}

}  // namespace pjds
