// LAGS-SGD hot path for B200 (sm_100a): accumulate -> select -> compact -> decode/update.
//
// Kernels (see DESIGN.md for rooflines):
//   K1 accum_kernel      acc = r + alpha*g (two roundings), finiteness of g, r <- acc
//                        R: training.py:250 and :174 (fused)
//   K2 select_kernel     per-layer exact top-k (radix select on |acc| keys, lowest-index ties)
//                        + ordered compaction into (int32 idx, value) + zero selected residuals
//                        R: sparsify.py:84-90, training.py:251-252
//   K5 decode kernels    rank-ordered fp64 accumulation of the gathered sparse sets and the
//                        SGD (optionally momentum) update  R: training.py:248,253-254
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <string>

#include "lags_common.cuh"
#include "lags_select.cuh"

namespace lags {

// ------------------------------------------------------------------------------------------
// K1: fused accumulate over the flat bucket
// ------------------------------------------------------------------------------------------

// TIn: storage type of g and r.  TAcc: arithmetic type of acc.  When TIn != TAcc the
// accumulated values go to `acc_out` (fp64 workspace) and r is rewritten by K2's epilogue.
template <typename TIn, typename TAcc>
__global__ void __launch_bounds__(256) accum_scalar_kernel(const TIn* __restrict__ g, TIn* __restrict__ r,
                                                           TAcc* __restrict__ acc_out, TAcc alpha, int64_t n,
                                                           uint32_t* status) {
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const TIn gi = g[i];
    bad |= nonfinite(gi);
    const TAcc a = accum(static_cast<TAcc>(r[i]), static_cast<TAcc>(gi), alpha);
    acc_out[i] = a;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// fp32 fast path: 16-byte vectors, g streamed (evict-first), r read+written in place.
__global__ void __launch_bounds__(256) accum_f32x4_kernel(const float4* __restrict__ g, float4* __restrict__ r,
                                                          float alpha, int64_t n4, uint32_t* status) {
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 gv = __ldcs(g + i);
    float4 rv = r[i];
    bad |= nonfinite(gv.x) | nonfinite(gv.y) | nonfinite(gv.z) | nonfinite(gv.w);
    rv.x = accum(rv.x, gv.x, alpha);
    rv.y = accum(rv.y, gv.y, alpha);
    rv.z = accum(rv.z, gv.z, alpha);
    rv.w = accum(rv.w, gv.w, alpha);
    r[i] = rv;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// Stand-alone finiteness check (R: training.py:174), used only to order error reports exactly
// like the reference when a later worker also has a layout error.
template <typename T>
__global__ void __launch_bounds__(256) finite_kernel(const T* __restrict__ x, int64_t n, uint32_t* status) {
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= nonfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// ------------------------------------------------------------------------------------------
// K2: one CTA per layer -- exact select + ordered compaction (+ residual zeroing)
// ------------------------------------------------------------------------------------------

template <typename T>
__global__ void __launch_bounds__(SEL_NT) select_kernel(const lags_layer_t* __restrict__ layers,
                                                        lags_layer_t single, T* acc, int32_t* idx_out,
                                                        T* val_out, int32_t* count_out, int zero_selected) {
  __shared__ SelectSmem<T> sm;
  const lags_layer_t L = layers ? layers[blockIdx.x] : single;
  T* data = acc + L.offset;
  const auto th = radix_select<T>(data, L.dim, static_cast<uint32_t>(L.k), sm);
  const uint32_t cnt =
      ordered_compact<T>(data, L.dim, th, idx_out + L.slot, val_out + L.slot, zero_selected != 0, sm);
  if (threadIdx.x == 0) count_out[layers ? blockIdx.x : 0] = static_cast<int32_t>(cnt);
}

// Mixed mode epilogue: r (fp32) <- fl32(acc) where acc (fp64) already has +0.0 at selected slots.
__global__ void __launch_bounds__(256) store_residual_kernel(const double* __restrict__ acc, float* __restrict__ r,
                                                             int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    r[i] = static_cast<float>(acc[i]);
}

// ------------------------------------------------------------------------------------------
// decompress (R: sparsify.py:63-68)
// ------------------------------------------------------------------------------------------

template <typename T>
__global__ void decompress_kernel(const int32_t* __restrict__ idx, const T* __restrict__ val,
                                  const int32_t* __restrict__ count, T* out) {
  const int32_t c = *count;
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) out[idx[j]] = val[j];
}

// ------------------------------------------------------------------------------------------
// K5: decode + update.  Phase A scatters every rank's pairs into a per-rank dense plane and
// marks the owner bitmask; phase B lets the lowest rank holding index i sum the planes in
// rank order (fp64, R: training.py:248,253) and apply v = v - total / P (R: :254).
// Grid: (layer, rank); each block walks that layer's slots of that rank.
// ------------------------------------------------------------------------------------------

template <typename TVal>
__global__ void __launch_bounds__(256) decode_scatter_kernel(const lags_layer_t* __restrict__ layers,
                                                             const char* msg_idx, const char* msg_val,
                                                             const char* msg_cnt, int64_t stride,
                                                             TVal* planes, int64_t n, uint32_t* mask) {
  const lags_layer_t L = layers[blockIdx.x];
  const int p = blockIdx.y;
  const int32_t* idx = reinterpret_cast<const int32_t*>(msg_idx + p * stride) + L.slot;
  const TVal* val = reinterpret_cast<const TVal*>(msg_val + p * stride) + L.slot;
  const int32_t cnt = reinterpret_cast<const int32_t*>(msg_cnt + p * stride)[blockIdx.x];
  TVal* plane = planes + static_cast<int64_t>(p) * n + L.offset;
  uint32_t* m = mask + L.offset;
  for (int32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
    const int32_t i = idx[j];
    plane[i] = val[j];
    atomicOr(m + i, 1u << p);
  }
}

template <typename TV, typename TVal>
__global__ void __launch_bounds__(256) decode_update_kernel(const lags_layer_t* __restrict__ layers,
                                                            const char* msg_idx, const char* msg_cnt,
                                                            int64_t stride, const TVal* planes, int64_t n,
                                                            uint32_t* mask, int P, TV* v) {
  const lags_layer_t L = layers[blockIdx.x];
  const int p = blockIdx.y;
  const int32_t* idx = reinterpret_cast<const int32_t*>(msg_idx + p * stride) + L.slot;
  const int32_t cnt = reinterpret_cast<const int32_t*>(msg_cnt + p * stride)[blockIdx.x];
  for (int32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
    const int64_t i = L.offset + idx[j];
    const uint32_t bits = mask[i];
    if (bits == 0 || (__ffs(bits) - 1) != p) continue;  // not the owner (or already applied)
    double total = 0.0;
    for (uint32_t b = bits; b; b &= b - 1) {
      const int q = __ffs(b) - 1;
      total = __dadd_rn(total, static_cast<double>(planes[static_cast<int64_t>(q) * n + i]));
    }
    v[i] = static_cast<TV>(__dsub_rn(static_cast<double>(v[i]), __ddiv_rn(total, static_cast<double>(P))));
    mask[i] = 0u;
  }
}

// Momentum variant (mu > 0, parity unpinned): dense over the bucket.
template <typename TV, typename TVal>
__global__ void __launch_bounds__(256) decode_momentum_kernel(const TVal* planes, int64_t n, uint32_t* mask,
                                                              int P, TV* v, TV* mom, double mu) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t bits = mask[i];
    double total = 0.0;
    if (bits) {
      for (uint32_t b = bits; b; b &= b - 1) {
        const int q = __ffs(b) - 1;
        total = __dadd_rn(total, static_cast<double>(planes[static_cast<int64_t>(q) * n + i]));
      }
      mask[i] = 0u;
    }
    const double mnew = __dadd_rn(__dmul_rn(mu, static_cast<double>(mom[i])), __ddiv_rn(total, static_cast<double>(P)));
    mom[i] = static_cast<TV>(mnew);
    v[i] = static_cast<TV>(__dsub_rn(static_cast<double>(v[i]), mnew));
  }
}

}  // namespace lags

// ==========================================================================================
// C ABI
// ==========================================================================================

using namespace lags;

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

std::atomic<unsigned long long> g_launches{0};

int cuda_check(const char* where, int launches = 1) {
  g_launches.fetch_add(static_cast<unsigned long long>(launches), std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return LAGS_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int stream_grid(int64_t work_items, int threads, int per_sm) {
  int64_t blocks = (work_items + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

bool valid_dtype(int32_t dtype) { return dtype == LAGS_F32 || dtype == LAGS_F64 || dtype == LAGS_F32_ACC64; }
size_t acc_size(int32_t dtype) { return dtype == LAGS_F32 ? 4 : 8; }

template <typename TIn, typename TAcc>
int launch_accum(const void* g, void* r, void* acc, double alpha, int64_t n, uint32_t* status, cudaStream_t s) {
  const TAcc a = static_cast<TAcc>(alpha);  // numpy casts a Python float to the array dtype (NEP 50)
  accum_scalar_kernel<TIn, TAcc><<<stream_grid(n, 256, 8), 256, 0, s>>>(
      static_cast<const TIn*>(g), static_cast<TIn*>(r), static_cast<TAcc*>(acc), a, n, status);
  return cuda_check("accum_scalar_kernel");
}

int launch_accum_f32(const float* g, float* r, double alpha, int64_t n, uint32_t* status, cudaStream_t s) {
  const float a = static_cast<float>(alpha);
  const uintptr_t ug = reinterpret_cast<uintptr_t>(g), ur = reinterpret_cast<uintptr_t>(r);
  if (n >= 1024 && (ug % 16) == (ur % 16) && (ug % 4) == 0) {
    const int64_t head = static_cast<int64_t>(((16 - ur % 16) % 16) / 4);
    const int64_t n4 = (n - head) / 4;
    const int64_t tail0 = head + n4 * 4;
    if (head) {
      accum_scalar_kernel<float, float><<<1, 256, 0, s>>>(g, r, r, a, head, status);
    }
    accum_f32x4_kernel<<<stream_grid(n4, 256, 8), 256, 0, s>>>(reinterpret_cast<const float4*>(g + head),
                                                                reinterpret_cast<float4*>(r + head), a, n4,
                                                                status);
    if (tail0 < n) {
      accum_scalar_kernel<float, float><<<1, 256, 0, s>>>(g + tail0, r + tail0, r + tail0, a, n - tail0, status);
    }
    return cuda_check("accum_f32x4_kernel", 1 + (head ? 1 : 0) + (tail0 < n ? 1 : 0));
  }
  accum_scalar_kernel<float, float><<<stream_grid(n, 256, 8), 256, 0, s>>>(g, r, r, a, n, status);
  return cuda_check("accum_scalar_kernel");
}

}  // namespace

extern "C" {

int lags_abi_version(void) { return 1; }

unsigned long long lags_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* lags_last_error(void) { return g_last_error.c_str(); }

size_t lags_compress_workspace_bytes(int32_t dtype, int32_t nlayers, int64_t n_total, int64_t total_k) {
  (void)nlayers;
  (void)total_k;
  size_t b = 256;
  if (dtype == LAGS_F32_ACC64) b += align_up(static_cast<size_t>(n_total) * 8, 256);
  return b;
}

int lags_compress(int32_t dtype, const lags_layer_t* layers, int32_t nlayers, int64_t n_total, int64_t total_k,
                  const void* g, void* r, double alpha, int32_t* idx_out, void* val_out, int32_t* count_out,
                  uint32_t* status, lags_layer_state_t* state, void* workspace, size_t workspace_bytes,
                  lags_stream_t stream) {
  (void)state;
  if (!valid_dtype(dtype)) return fail(LAGS_ERR_INVALID_ARG, "lags_compress: unknown dtype");
  if (!layers || nlayers <= 0 || n_total <= 0 || !g || !r || !idx_out || !val_out || !count_out || !status)
    return fail(LAGS_ERR_INVALID_ARG, "lags_compress: null pointer or empty bucket");
  if (total_k <= 0) return fail(LAGS_ERR_INVALID_ARG, "lags_compress: total_k must be positive");
  if (workspace_bytes < lags_compress_workspace_bytes(dtype, nlayers, n_total, total_k))
    return fail(LAGS_ERR_WORKSPACE, "lags_compress: workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if (dtype == LAGS_F32) {
    rc = launch_accum_f32(static_cast<const float*>(g), static_cast<float*>(r), alpha, n_total, status, s);
    if (rc) return rc;
    select_kernel<float><<<nlayers, SEL_NT, 0, s>>>(layers, lags_layer_t{}, static_cast<float*>(r), idx_out,
                                                    static_cast<float*>(val_out), count_out, 1);
    return cuda_check("select_kernel<float>");
  }
  if (dtype == LAGS_F64) {
    rc = launch_accum<double, double>(g, r, r, alpha, n_total, status, s);
    if (rc) return rc;
    select_kernel<double><<<nlayers, SEL_NT, 0, s>>>(layers, lags_layer_t{}, static_cast<double*>(r), idx_out,
                                                     static_cast<double*>(val_out), count_out, 1);
    return cuda_check("select_kernel<double>");
  }
  // LAGS_F32_ACC64: fp64 acc in the workspace, fp32 residual written back after selection.
  double* acc = reinterpret_cast<double*>(align_up(reinterpret_cast<uintptr_t>(workspace), 256));
  rc = launch_accum<float, double>(g, r, acc, alpha, n_total, status, s);
  if (rc) return rc;
  select_kernel<double><<<nlayers, SEL_NT, 0, s>>>(layers, lags_layer_t{}, acc, idx_out,
                                                   static_cast<double*>(val_out), count_out, 1);
  rc = cuda_check("select_kernel<double>");
  if (rc) return rc;
  store_residual_kernel<<<stream_grid(n_total, 256, 8), 256, 0, s>>>(acc, static_cast<float*>(r), n_total);
  return cuda_check("store_residual_kernel");
}

int lags_check_finite(int32_t dtype, const void* x, int64_t n, uint32_t* status, lags_stream_t stream) {
  if (!x || !status || n < 0) return fail(LAGS_ERR_INVALID_ARG, "lags_check_finite: bad argument");
  if (n == 0) return LAGS_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == LAGS_F64)
    finite_kernel<double><<<stream_grid(n, 256, 8), 256, 0, s>>>(static_cast<const double*>(x), n, status);
  else
    finite_kernel<float><<<stream_grid(n, 256, 8), 256, 0, s>>>(static_cast<const float*>(x), n, status);
  return cuda_check("finite_kernel");
}

size_t lags_top_k_workspace_bytes(int32_t dtype, int64_t dim) {
  return 256 + align_up(static_cast<size_t>(dim) * (dtype == LAGS_F64 ? 8 : 4), 256);
}

int lags_top_k(int32_t dtype, const void* x, int64_t dim, int32_t k, int32_t* idx_out, void* val_out,
               int32_t* count_out, void* workspace, size_t workspace_bytes, lags_stream_t stream) {
  if (dtype != LAGS_F32 && dtype != LAGS_F64) return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: dtype must be F32 or F64");
  if (!x || !idx_out || !val_out || !count_out || !workspace) return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: null pointer");
  if (dim <= 0) return fail(LAGS_ERR_INVALID_ARG, "input must be a non-empty 1-D array");
  if (k < 1 || k > dim) return fail(LAGS_ERR_K_OUT_OF_RANGE, "k=" + std::to_string(k) + " outside 1.." + std::to_string(dim));
  if (dim > 0x7fffffffLL) return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: dim exceeds int32 index range");
  if (workspace_bytes < lags_top_k_workspace_bytes(dtype, dim)) return fail(LAGS_ERR_WORKSPACE, "lags_top_k: workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == LAGS_F64 ? 8 : 4;
  void* copy = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 256));
  if (cudaMemcpyAsync(copy, x, static_cast<size_t>(dim) * es, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return cuda_check("lags_top_k copy", 0);
  lags_layer_t one{0, dim, k, 0};
  if (dtype == LAGS_F32)
    select_kernel<float><<<1, SEL_NT, 0, s>>>(nullptr, one, static_cast<float*>(copy), idx_out,
                                              static_cast<float*>(val_out), count_out, 0);
  else
    select_kernel<double><<<1, SEL_NT, 0, s>>>(nullptr, one, static_cast<double*>(copy), idx_out,
                                               static_cast<double*>(val_out), count_out, 0);
  return cuda_check("select_kernel(top_k)");
}

int lags_decompress(int32_t dtype, const int32_t* idx, const void* val, const int32_t* count, int64_t dim, void* out,
                    lags_stream_t stream) {
  if (dtype != LAGS_F32 && dtype != LAGS_F64) return fail(LAGS_ERR_INVALID_ARG, "lags_decompress: dtype must be F32 or F64");
  if (!idx || !val || !count || !out || dim <= 0) return fail(LAGS_ERR_INVALID_ARG, "lags_decompress: bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == LAGS_F64 ? 8 : 4;
  if (cudaMemsetAsync(out, 0, static_cast<size_t>(dim) * es, s) != cudaSuccess) return cuda_check("lags_decompress memset", 0);
  if (dtype == LAGS_F32)
    decompress_kernel<float><<<64, 256, 0, s>>>(idx, static_cast<const float*>(val), count, static_cast<float*>(out));
  else
    decompress_kernel<double><<<64, 256, 0, s>>>(idx, static_cast<const double*>(val), count, static_cast<double*>(out));
  return cuda_check("decompress_kernel");
}

size_t lags_decode_workspace_bytes(int32_t dtype, int64_t n_total, int32_t P) {
  if (!valid_dtype(dtype) || n_total <= 0 || P <= 0) return 0;
  return align_up(static_cast<size_t>(n_total) * 4, 256) +
         align_up(static_cast<size_t>(n_total) * static_cast<size_t>(P) * acc_size(dtype), 256);
}

int lags_decode_update(int32_t dtype, const lags_layer_t* layers, int32_t nlayers, int64_t n_total, int64_t total_k,
                       const int32_t* idx0, const void* val0, const int32_t* cnt0, int64_t rank_stride_bytes, int32_t P,
                       void* v, void* momentum, double mu, void* workspace, size_t workspace_bytes,
                       lags_stream_t stream) {
  (void)total_k;
  if (!valid_dtype(dtype)) return fail(LAGS_ERR_INVALID_ARG, "lags_decode_update: unknown dtype");
  if (!layers || nlayers <= 0 || n_total <= 0 || !idx0 || !val0 || !cnt0 || !v || !workspace)
    return fail(LAGS_ERR_INVALID_ARG, "lags_decode_update: null pointer or empty bucket");
  if (P < 1 || P > 32) return fail(LAGS_ERR_INVALID_ARG, "lags_decode_update: P must be in 1..32");
  if (mu != 0.0 && !momentum) return fail(LAGS_ERR_INVALID_ARG, "lags_decode_update: mu > 0 needs a momentum buffer");
  if (workspace_bytes < lags_decode_workspace_bytes(dtype, n_total, P))
    return fail(LAGS_ERR_WORKSPACE, "lags_decode_update: workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* mask = static_cast<uint32_t*>(workspace);
  char* planes = static_cast<char*>(workspace) + align_up(static_cast<size_t>(n_total) * 4, 256);
  const char* mi = reinterpret_cast<const char*>(idx0);
  const char* mv = static_cast<const char*>(val0);
  const char* mc = reinterpret_cast<const char*>(cnt0);
  dim3 grid(nlayers, P);
  if (dtype == LAGS_F32) {
    decode_scatter_kernel<float><<<grid, 256, 0, s>>>(layers, mi, mv, mc, rank_stride_bytes,
                                                      reinterpret_cast<float*>(planes), n_total, mask);
    if (mu == 0.0)
      decode_update_kernel<float, float><<<grid, 256, 0, s>>>(layers, mi, mc, rank_stride_bytes,
                                                              reinterpret_cast<const float*>(planes), n_total,
                                                              mask, P, static_cast<float*>(v));
    else
      decode_momentum_kernel<float, float><<<stream_grid(n_total, 256, 8), 256, 0, s>>>(
          reinterpret_cast<const float*>(planes), n_total, mask, P, static_cast<float*>(v),
          static_cast<float*>(momentum), mu);
  } else if (dtype == LAGS_F64) {
    decode_scatter_kernel<double><<<grid, 256, 0, s>>>(layers, mi, mv, mc, rank_stride_bytes,
                                                       reinterpret_cast<double*>(planes), n_total, mask);
    if (mu == 0.0)
      decode_update_kernel<double, double><<<grid, 256, 0, s>>>(layers, mi, mc, rank_stride_bytes,
                                                                reinterpret_cast<const double*>(planes), n_total,
                                                                mask, P, static_cast<double*>(v));
    else
      decode_momentum_kernel<double, double><<<stream_grid(n_total, 256, 8), 256, 0, s>>>(
          reinterpret_cast<const double*>(planes), n_total, mask, P, static_cast<double*>(v),
          static_cast<double*>(momentum), mu);
  } else {
    decode_scatter_kernel<double><<<grid, 256, 0, s>>>(layers, mi, mv, mc, rank_stride_bytes,
                                                       reinterpret_cast<double*>(planes), n_total, mask);
    if (mu == 0.0)
      decode_update_kernel<float, double><<<grid, 256, 0, s>>>(layers, mi, mc, rank_stride_bytes,
                                                               reinterpret_cast<const double*>(planes), n_total,
                                                               mask, P, static_cast<float*>(v));
    else
      decode_momentum_kernel<float, double><<<stream_grid(n_total, 256, 8), 256, 0, s>>>(
          reinterpret_cast<const double*>(planes), n_total, mask, P, static_cast<float*>(v),
          static_cast<float*>(momentum), mu);
  }
  return cuda_check("decode kernels", 2);
}

}  // extern "C"
