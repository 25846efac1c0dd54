// Shared device helpers for the LAGS-SGD B200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lags_b200.h"

// One layer of a bucket (device table).  Layer j occupies flat elements [offset, offset + dim)
// and output slots [slot, slot + k).
struct lags_layer_t {
  int64_t offset;
  int64_t dim;
  int32_t k;
  int32_t slot;
};

namespace lags {

// |x| as an unsigned key: monotone in magnitude for finite x and +-inf, 0 for +-0 and NaN.
// Ties on equal keys are broken by lower index (R: sparsify.py:85-87).  NaN maps to 0 (never
// selected): the reference's stable argsort of -|x| puts NaN after every number and its
// `mag > 0` filter then drops it (R: sparsify.py:87-88).
template <typename T> struct Key;
template <> struct Key<float> {
  using K = uint32_t;
  static constexpr int BITS = 31;  // sign bit dropped
  static constexpr int RB = 12;    // radix digit width -> <= 3 passes (12, 12, 7); crowded
                                   // candidate keys (common prefix skipped) usually need 2
  __device__ __forceinline__ static K of(float x) {
    const K k = __float_as_uint(x) & 0x7fffffffu;
    return k > 0x7f800000u ? 0u : k;
  }
};
template <> struct Key<double> {
  using K = unsigned long long;
  static constexpr int BITS = 63;
  static constexpr int RB = 13;  // 5 passes (13, 13, 13, 13, 11)
  __device__ __forceinline__ static K of(double x) {
    const K k = static_cast<K>(__double_as_longlong(x)) & 0x7fffffffffffffffull;
    return k > 0x7ff0000000000000ull ? 0ull : k;
  }
};

// Residual of a selected entry, acc - sent with sent = acc (R: training.py:252): +0.0 for finite
// acc, NaN for an overflowed +-inf (inf - inf), exactly as numpy computes it.
__device__ __forceinline__ float sent_residual(float x) { return __fsub_rn(x, x); }
__device__ __forceinline__ double sent_residual(double x) { return __dsub_rn(x, x); }

// total / P, the workers' mean of the decode (R: training.py:253-254).  A power-of-two P divides
// by multiplying with 2^-log2(P): both are the correctly rounded value of total * 2^-e (subnormal
// results included), so the bits match the IEEE division, which the other worker counts take.
__device__ __forceinline__ double div_workers(double total, int P) {
  if ((P & (P - 1)) == 0) return __dmul_rn(total, __longlong_as_double(static_cast<long long>(992 + __clz(P)) << 52));
  return __ddiv_rn(total, static_cast<double>(P));
}

// acc = r + alpha * g rounded twice (numpy evaluates `alpha * g` then `+`; no FMA).
__device__ __forceinline__ float accum(float r, float g, float a) { return __fadd_rn(r, __fmul_rn(a, g)); }
__device__ __forceinline__ double accum(double r, double g, double a) { return __dadd_rn(r, __dmul_rn(a, g)); }

// Programmatic dependent launch (sm_90+): wait until the preceding kernel on the stream has
// completed and its memory is visible.  A no-op for kernels launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the next kernel on the stream (launched with PDL) to be scheduled now.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ bool nonfinite(float g) { return (__float_as_uint(g) & 0x7f800000u) == 0x7f800000u; }
__device__ __forceinline__ bool nonfinite(double g) {
  return (static_cast<unsigned long long>(__double_as_longlong(g)) & 0x7ff0000000000000ull) ==
         0x7ff0000000000000ull;
}

// Block-wide exclusive scan of one uint32 per thread (NT threads, multiple of 32).
// `warp_tot` must hold 33 uint32 of shared memory.  Returns the exclusive prefix and writes the
// block total into *total.  Contains two __syncthreads().
// Inlining of the block-wide helpers (instruction footprint vs call overhead), per helper:
// LAGS_INL_<NAME> = 1 inline, 0 out of line.
#ifndef LAGS_INL_SCAN
#define LAGS_INL_SCAN 1
#endif
#ifndef LAGS_INL_FINDBIN
#define LAGS_INL_FINDBIN 1
#endif
#ifndef LAGS_INL_SUM
#define LAGS_INL_SUM 1
#endif
#ifndef LAGS_INL_OR
#define LAGS_INL_OR 1
#endif
#if LAGS_INL_SCAN
#define LAGS_SCAN_ATTR __forceinline__
#else
#define LAGS_SCAN_ATTR __noinline__
#endif
#if LAGS_INL_FINDBIN
#define LAGS_FINDBIN_ATTR __forceinline__
#else
#define LAGS_FINDBIN_ATTR __noinline__
#endif
#if LAGS_INL_SUM
#define LAGS_SUM_ATTR __forceinline__
#else
#define LAGS_SUM_ATTR __noinline__
#endif
#if LAGS_INL_OR
#define LAGS_OR_ATTR __forceinline__
#else
#define LAGS_OR_ATTR __noinline__
#endif

// Rarely executed selection paths (dense fallbacks, radix selects behind a failed histogram cut)
// are kept out of line: every path of the selection kernel runs once per launch with a cold
// instruction cache, so inlining them would only spread the hot path over more cache lines.
#ifdef LAGS_COLD_INLINE
#define LAGS_COLD __forceinline__
#else
#define LAGS_COLD __noinline__
#endif

template <int NT>
__device__ LAGS_SCAN_ATTR uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = NT / 32;
    uint32_t w = lane < NW ? warp_tot[lane] : 0u;
    uint32_t s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NW) warp_tot[lane] = s - w;  // exclusive warp prefix
    if (lane == 31) warp_tot[32] = s;
  }
  __syncthreads();
  *total = warp_tot[32];
  return warp_tot[warp] + x - v;
}

}  // namespace lags
