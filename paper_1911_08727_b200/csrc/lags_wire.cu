// Sparse wire format on the device (R: sparsify.py:260-310):
//   chunk   = u32 layer_id, u32 dim, u32 count, count x (u32 index, f64 value)   little-endian, packed
//   message = u32 chunk count, then the chunks back to back
// Byte-moving work: an encoder turns a chunk table (a bucket's compress output, or uploaded
// SparseChunks) into wire bytes; a decoder parses wire bytes back into a chunk table, with the
// reference's validation (truncation, trailing bytes, index range / order of each chunk, the
// first error in chunk order wins).  Entries are 12 bytes at 4-byte alignment, so every access
// is a 32-bit word: the f64 value is written / read as two words.
#include <cuda_runtime.h>

#include <string>

#include "lags_common.cuh"
#include "lags_internal.h"

namespace lags {

constexpr int WIRE_NT = 512;
constexpr int WIRE_MAX_CHUNKS = 4096;  // decode: chunk table staged in shared memory

// Exclusive prefix of wire offsets over nchunks chunk sizes (12 + 12 * count), in shared memory.
// Returns the message length (header included when with_header).  All threads.
__device__ int64_t wire_offsets(int nchunks, const int32_t* counts, bool with_header, int64_t* off) {
  __shared__ int64_t part[WIRE_NT / 32 + 1];
  __shared__ int64_t carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = with_header ? 4 : 0;
  __syncthreads();
  for (int base = 0; base < nchunks; base += WIRE_NT) {
    const int c = base + threadIdx.x;
    const int64_t sz = c < nchunks ? 12 + 12 * static_cast<int64_t>(max(counts[c], 0)) : 0;
    int64_t x = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) part[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t s = 0;
      for (int w = 0; w < WIRE_NT / 32; ++w) {
        const int64_t t = part[w];
        part[w] = s;
        s += t;
      }
      part[WIRE_NT / 32] = s;
    }
    __syncthreads();
    if (c < nchunks) off[c] = carry_s + part[warp] + x - sz;
    __syncthreads();
    if (threadIdx.x == 0) carry_s += part[WIRE_NT / 32];
    __syncthreads();
  }
  return carry_s;
}

__device__ __forceinline__ void put_u32(char* w, int64_t at, uint32_t x) {
  *reinterpret_cast<uint32_t*>(w + at) = x;
}
__device__ __forceinline__ uint32_t get_u32(const char* w, int64_t at) {
  return __ldcg(reinterpret_cast<const uint32_t*>(w + at));
}

// Encoder: every CTA derives the chunk offsets, then writes the headers and entries of chunks
// blockIdx.x, blockIdx.x + gridDim.x, ...  Nothing is written when the message exceeds capacity.
template <typename TVal>
__global__ void __launch_bounds__(WIRE_NT) wire_encode_kernel(int with_header, int nchunks,
                                                              const uint32_t* __restrict__ layer_ids,
                                                              const uint32_t* __restrict__ dims,
                                                              const int32_t* __restrict__ counts,
                                                              const int64_t* __restrict__ first,
                                                              const int32_t* __restrict__ idx,
                                                              const TVal* __restrict__ val, char* wire,
                                                              int64_t capacity, int64_t* wire_len,
                                                              uint64_t* error) {
  extern __shared__ int64_t off[];
  griddep_wait();
  const int64_t total = wire_offsets(nchunks, counts, with_header != 0, off);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *wire_len = total;
    *error = total > capacity ? (static_cast<uint64_t>(nchunks) << 8) | LAGS_WIRE_ERR_CAPACITY : ~0ull;
    if (with_header && total <= capacity) put_u32(wire, 0, static_cast<uint32_t>(nchunks));
  }
  if (total > capacity) return;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t at = off[c];
    const int32_t n = max(counts[c], 0);
    if (threadIdx.x == 0) {
      put_u32(wire, at, layer_ids[c]);
      put_u32(wire, at + 4, dims[c]);
      put_u32(wire, at + 8, static_cast<uint32_t>(n));
    }
    const int64_t f = first[c];
    for (int q = threadIdx.x; q < n; q += WIRE_NT) {
      const double x = static_cast<double>(val[f + q]);
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
      const int64_t e = at + 12 + 12 * static_cast<int64_t>(q);
      put_u32(wire, e, static_cast<uint32_t>(idx[f + q]));
      put_u32(wire, e + 4, static_cast<uint32_t>(bits));
      put_u32(wire, e + 8, static_cast<uint32_t>(bits >> 32));
    }
  }
}

// Decoder: one CTA.  Thread 0 walks the chunk headers (each position depends on the previous
// count); then all threads copy the entries and validate every chunk's indices.
template <typename TVal>
__global__ void __launch_bounds__(WIRE_NT) wire_decode_kernel(
    int with_header, const char* __restrict__ wire, int64_t wire_len, int64_t offset, int max_chunks,
    const int64_t* __restrict__ first, const int32_t* __restrict__ caps, int64_t entry_capacity, uint32_t* layer_ids,
    uint32_t* dims, int32_t* counts, int32_t* idx, TVal* val, int32_t* nchunks_out, int64_t* end_out, uint64_t* error) {
  extern __shared__ int64_t sh[];
  int64_t* woff = sh;                       // [max_chunks] wire offset of each chunk
  int64_t* dst = sh + max_chunks;           // [max_chunks] first output slot
  __shared__ int n_s;
  __shared__ unsigned long long err_s;
  griddep_wait();
  if (threadIdx.x == 0) {
    unsigned long long err = ~0ull;
    int64_t p = offset;
    int n = 0;
    int64_t packed = 0;
    auto fail = [&](int chunk, uint32_t code) {
      err = (static_cast<unsigned long long>(static_cast<uint32_t>(chunk)) << 8) | code;
    };
    uint32_t want = 1;
    if (with_header) {
      if (p + 4 > wire_len) {
        fail(0, LAGS_WIRE_ERR_TRUNCATED_MESSAGE);
        want = 0;
      } else {
        want = get_u32(wire, p);
        p += 4;
      }
    }
    for (uint32_t c = 0; c < want && err == ~0ull; ++c) {
      if (p + 12 > wire_len) {
        fail(static_cast<int>(c), LAGS_WIRE_ERR_TRUNCATED_HEADER);
        break;
      }
      const uint32_t cnt = get_u32(wire, p + 8);
      const int64_t need = 12 * static_cast<int64_t>(cnt);
      if (p + 12 + need > wire_len) {
        fail(static_cast<int>(c), LAGS_WIRE_ERR_TRUNCATED_PAYLOAD);
        break;
      }
      const int64_t d0 = first ? first[c] : packed;
      const int64_t room = caps ? caps[c] : entry_capacity - packed;
      if (static_cast<int>(c) >= max_chunks || cnt > 0x7fffffffu || static_cast<int64_t>(cnt) > room) {
        fail(static_cast<int>(c), LAGS_WIRE_ERR_CAPACITY);
        break;
      }
      layer_ids[c] = get_u32(wire, p);
      dims[c] = get_u32(wire, p + 4);
      counts[c] = static_cast<int32_t>(cnt);
      woff[c] = p;
      dst[c] = d0;
      packed += cnt;
      p += 12 + need;
      n = static_cast<int>(c) + 1;
    }
    if (err == ~0ull && with_header && p != wire_len) fail(n, LAGS_WIRE_ERR_TRAILING);
    n_s = n;
    err_s = err;
    *nchunks_out = n;
    *end_out = p;
  }
  __syncthreads();
  const int n = n_s;
  // copy + validation (R: sparsify.py:41-52 via decode_chunk's SparseChunk): last index < dim,
  // then strictly increasing; the first failing chunk (in order) is reported
  for (int c = 0; c < n; ++c) {
    const int64_t at = woff[c] + 12;
    const int32_t cnt = counts[c];
    const uint32_t dim = dims[c];
    const int64_t d0 = dst[c];
    bool order_bad = false;
    for (int q = threadIdx.x; q < cnt; q += WIRE_NT) {
      const int64_t e = at + 12 * static_cast<int64_t>(q);
      const uint32_t ix = get_u32(wire, e);
      const unsigned long long bits =
          static_cast<unsigned long long>(get_u32(wire, e + 4)) | (static_cast<unsigned long long>(get_u32(wire, e + 8)) << 32);
      idx[d0 + q] = static_cast<int32_t>(ix);
      val[d0 + q] = static_cast<TVal>(__longlong_as_double(static_cast<long long>(bits)));
      if (q > 0 && get_u32(wire, e - 12) >= ix) order_bad = true;
      if (q == cnt - 1 && (ix >= dim || ix > 0x7fffffffu))
        atomicMin(&err_s, (static_cast<unsigned long long>(c) << 8) | LAGS_WIRE_ERR_INDEX_RANGE);
    }
    if (order_bad) atomicMin(&err_s, (static_cast<unsigned long long>(c) << 8) | LAGS_WIRE_ERR_INDEX_ORDER);
  }
  __syncthreads();
  if (threadIdx.x == 0) *error = err_s;
}

}  // namespace lags

using namespace lags;

extern "C" {

int lags_wire_encode(uint32_t mode, int32_t nchunks, const uint32_t* layer_ids, const uint32_t* dims,
                     const int32_t* counts, const int64_t* first, const int32_t* idx, const void* val,
                     int32_t val_dtype, void* wire, int64_t wire_capacity, int64_t* wire_len, uint64_t* error,
                     lags_stream_t stream) {
  if (nchunks < 0 || (nchunks > 0 && (!layer_ids || !dims || !counts || !first || !idx || !val)) || !wire ||
      !wire_len || !error)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_encode: null pointer or negative chunk count");
  if (mode != LAGS_WIRE_MESSAGE && !(mode == LAGS_WIRE_CHUNK && nchunks == 1))
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_encode: chunk mode encodes exactly one chunk");
  if (val_dtype != LAGS_F32 && val_dtype != LAGS_F64)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_encode: values must be LAGS_F32 or LAGS_F64");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = nchunks < 1 ? 1 : (nchunks < 148 ? nchunks : 148);
  const size_t smem = sizeof(int64_t) * static_cast<size_t>(nchunks > 0 ? nchunks : 1);
  if (smem > 200 * 1024) return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_encode: too many chunks");
  const int hdr = mode == LAGS_WIRE_MESSAGE ? 1 : 0;
  cudaError_t e;
  if (val_dtype == LAGS_F32) {
    cudaFuncSetAttribute(wire_encode_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    wire_encode_kernel<float><<<grid, WIRE_NT, smem, s>>>(hdr, nchunks, layer_ids, dims, counts, first, idx,
                                                         static_cast<const float*>(val), static_cast<char*>(wire),
                                                         wire_capacity, wire_len, error);
  } else {
    cudaFuncSetAttribute(wire_encode_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    wire_encode_kernel<double><<<grid, WIRE_NT, smem, s>>>(hdr, nchunks, layer_ids, dims, counts, first, idx,
                                                          static_cast<const double*>(val), static_cast<char*>(wire),
                                                          wire_capacity, wire_len, error);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return host_fail(LAGS_ERR_CUDA, std::string("lags_wire_encode: ") + cudaGetErrorString(e));
  host_count_launches(1);
  return LAGS_OK;
}

int lags_wire_decode(uint32_t mode, const void* wire, int64_t wire_len, int64_t offset, int32_t max_chunks,
                     const int64_t* first, const int32_t* caps, int64_t entry_capacity, uint32_t* layer_ids,
                     uint32_t* dims, int32_t* counts, int32_t* idx, void* val, int32_t val_dtype,
                     int32_t* nchunks_out, int64_t* end_out, uint64_t* error, lags_stream_t stream) {
  if (!wire || !layer_ids || !dims || !counts || !idx || !val || !nchunks_out || !end_out || !error)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_decode: null pointer");
  if (mode != LAGS_WIRE_MESSAGE && mode != LAGS_WIRE_CHUNK)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_decode: unknown mode");
  if (max_chunks < 1 || max_chunks > WIRE_MAX_CHUNKS)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_decode: max_chunks outside 1..4096");
  if (offset < 0 || wire_len < 0) return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_decode: negative length");
  if (val_dtype != LAGS_F32 && val_dtype != LAGS_F64)
    return host_fail(LAGS_ERR_INVALID_ARG, "lags_wire_decode: values must be LAGS_F32 or LAGS_F64");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t smem = 2 * sizeof(int64_t) * static_cast<size_t>(max_chunks);
  const int hdr = mode == LAGS_WIRE_MESSAGE ? 1 : 0;
  const char* w = static_cast<const char*>(wire);
  if (val_dtype == LAGS_F32) {
    cudaFuncSetAttribute(wire_decode_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    wire_decode_kernel<float><<<1, WIRE_NT, smem, s>>>(hdr, w, wire_len, offset, max_chunks, first, caps,
                                                      entry_capacity, layer_ids, dims, counts, idx,
                                                      static_cast<float*>(val), nchunks_out, end_out, error);
  } else {
    cudaFuncSetAttribute(wire_decode_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    wire_decode_kernel<double><<<1, WIRE_NT, smem, s>>>(hdr, w, wire_len, offset, max_chunks, first, caps,
                                                       entry_capacity, layer_ids, dims, counts, idx,
                                                       static_cast<double*>(val), nchunks_out, end_out, error);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return host_fail(LAGS_ERR_CUDA, std::string("lags_wire_decode: ") + cudaGetErrorString(e));
  host_count_launches(1);
  return LAGS_OK;
}

}  // extern "C"
