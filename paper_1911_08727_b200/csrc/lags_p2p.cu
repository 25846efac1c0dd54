// Peer-memory exchange of the fixed-size bucket messages over NVLink / NVSwitch (one process per
// GPU, CUDA IPC mappings): the all-gather step of R: training.py:245-248 without a collective
// library.  Every rank owns one receive area in its HBM, mapped into every peer:
//
//   [ flags: P * G u32 ] [ pad to 256 B ] [ parity 0: P messages ] [ parity 1: P messages ]
//
// lags_p2p_push: G CTAs per destination copy the local message into slot `rank` of the
// destination's parity (epoch & 1) area with 16-byte stores (remote ones travel over NVLink),
// then each CTA publishes `epoch` in its own flag of the destination with a system-scope
// release.  lags_p2p_wait: one warp acquires all P * G local flags (>= epoch) before the decode
// that follows it on the stream reads the area, then advances the device-resident epoch counter
// (the push reads it: no host argument changes per step, so the step can be graph-captured).  Double buffering by parity is enough: a rank
// pushes step t+1 only after it received every rank's step-t message, and each rank pushed step t
// only after its own decode of step t-1 (stream order), so parity (t+1) & 1 is free everywhere.
// The wait is bounded (globaltimer): a missing peer sets LAGS_STATUS_P2P_TIMEOUT instead of
// hanging the GPU.
#include <cuda_runtime.h>

#include <string>

#include "lags_b200.h"
#include "lags_common.cuh"
#include "lags_internal.h"

namespace lags {

constexpr int P2P_NT = 512;

__global__ void __launch_bounds__(P2P_NT) p2p_push_kernel(const uint4* __restrict__ src, int64_t n16,
                                                           int64_t msg_bytes, uint64_t flags_bytes,
                                                           const uint64_t* __restrict__ bases, int P, int rank,
                                                           int G, const uint32_t* epoch_dev) {
  griddep_wait();  // the compress that wrote the message (and the last wait, the epoch) completed
  const uint32_t epoch = *reinterpret_cast<const volatile uint32_t*>(epoch_dev) + 1u;
  // the wait kernel may start polling now: it reads only the flags (acquire) and the epoch, which
  // it advances after every flag -- this push's own included, published after the read above
  griddep_launch_dependents();
  const int p = static_cast<int>(blockIdx.x) / G, gq = static_cast<int>(blockIdx.x) % G;
  char* base = reinterpret_cast<char*>(bases[p]);
  uint4* dst = reinterpret_cast<uint4*>(base + flags_bytes + static_cast<int64_t>(epoch & 1u) * P * msg_bytes +
                                        static_cast<int64_t>(rank) * msg_bytes);
  const int64_t lo = n16 * gq / G, hi = n16 * (gq + 1) / G;
  for (int64_t i = lo + threadIdx.x; i < hi; i += P2P_NT) dst[i] = __ldg(src + i);
  __syncthreads();
  if (threadIdx.x == 0) {
    // st.release.sys = fence.acq_rel.sys + relaxed store: cumulative over what this thread has
    // observed, which after the barrier includes every store of the CTA (a separate
    // __threadfence_system() here measured 2 us slower per exchange and orders nothing more;
    // -DLAGS_P2P_SC_FENCE restores it)
#ifdef LAGS_P2P_SC_FENCE
    __threadfence_system();
#endif
    uint32_t* flag = reinterpret_cast<uint32_t*>(base) + rank * G + gq;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
  }
}

__global__ void p2p_wait_kernel(const uint32_t* flags, int nflags, uint32_t* epoch_dev, int32_t* status,
                                uint64_t timeout_ns) {
  const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(epoch_dev) + 1u;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = threadIdx.x; i < nflags; i += blockDim.x) {
    for (;;) {
      uint32_t f;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + i) : "memory");
      if (static_cast<int32_t>(f - epoch) >= 0) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicOr(reinterpret_cast<unsigned int*>(status), LAGS_STATUS_P2P_TIMEOUT);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
  if (threadIdx.x == 0) *epoch_dev = epoch;  // this exchange is complete: the next push uses epoch + 1
}

}  // namespace lags

using namespace lags;

extern "C" {

int lags_ipc_malloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle || bytes == 0) return host_fail(LAGS_ERR_INVALID_ARG, "lags_ipc_malloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), p);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return host_fail(LAGS_ERR_CUDA, std::string("lags_ipc_malloc: ") + cudaGetErrorString(e));
  }
  *ptr = p;
  return LAGS_OK;
}

int lags_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return host_fail(LAGS_ERR_INVALID_ARG, "lags_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return host_fail(LAGS_ERR_CUDA, std::string("lags_ipc_open: ") + cudaGetErrorString(e));
  return LAGS_OK;
}

int lags_ipc_close(void* ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? LAGS_OK : host_fail(LAGS_ERR_CUDA, std::string("lags_ipc_close: ") + cudaGetErrorString(e));
}

int lags_ipc_free(void* ptr) {
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? LAGS_OK : host_fail(LAGS_ERR_CUDA, std::string("lags_ipc_free: ") + cudaGetErrorString(e));
}

int lags_p2p_push(const void* msg, int64_t msg_bytes, const uint64_t* bases, int P, int rank, int ctas_per_peer,
                  uint64_t flags_bytes, const uint32_t* epoch, lags_stream_t stream) {
  if (!msg || !bases || !epoch || P < 1 || rank < 0 || rank >= P || ctas_per_peer < 1 || msg_bytes <= 0 || (msg_bytes & 15) ||
      (flags_bytes & 255) || flags_bytes < static_cast<uint64_t>(P) * ctas_per_peer * 4u ||
      (reinterpret_cast<uintptr_t>(msg) & 15))
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_p2p_push: bad arguments (16-byte aligned message and sizes)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(P * ctas_per_peer));
  cfg.blockDim = dim3(P2P_NT);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, p2p_push_kernel, static_cast<const uint4*>(msg), msg_bytes / 16,
                                           msg_bytes, flags_bytes, bases, P, rank, ctas_per_peer, epoch);
  if (e != cudaSuccess) return host_fail(LAGS_ERR_CUDA, std::string("lags_p2p_push: ") + cudaGetErrorString(e));
  host_count_launches(1);
  return LAGS_OK;
}

int lags_p2p_wait(const uint32_t* flags, int nflags, uint32_t* epoch, int32_t* status, uint64_t timeout_ns,
                  lags_stream_t stream) {
  if (!flags || !epoch || !status || nflags < 1) return host_fail(LAGS_ERR_INVALID_ARG, "lags_p2p_wait: bad arguments");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // scheduled as the push drains
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, p2p_wait_kernel, flags, nflags, epoch, status, timeout_ns);
  if (e != cudaSuccess) return host_fail(LAGS_ERR_CUDA, std::string("lags_p2p_wait: ") + cudaGetErrorString(e));
  host_count_launches(1);
  return LAGS_OK;
}

}  // extern "C"
