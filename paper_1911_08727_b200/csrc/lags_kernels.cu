// LAGS-SGD hot path for B200 (sm_100a): accumulate -> select -> compact -> decode/update.
//
// Kernels (DESIGN.md has the rooflines):
//   accum_emit_kernel     (lags_fast.cuh) fp32 accumulate + candidate emission (K1)  R: training.py:250,174
//   select_kernel         (lags_cluster.cuh) exact top-k from the candidates: 4-CTA clusters
//                         for the largest layers, persistent per-layer CTAs for the rest   R: sparsify.py:84-90
//   accum_emit64_kernel / select64_kernel (lags_f64.cuh) the same two launches for LAGS_F64 and
//                         LAGS_F32_ACC64 on 64-bit keys                             R: training.py:250-252
//   select_dense_kernel   exact dense top-k of one vector (the top_k drop-in)      R: sparsify.py:84-90
//   decode_* kernels    rank-ordered fp64 accumulation + SGD/momentum update          R: training.py:248,253-254
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "lags_common.cuh"
#include "lags_internal.h"
#include "lags_cluster.cuh"
#include "lags_f64.cuh"
#include "lags_fast.cuh"
#include "lags_select.cuh"

namespace lags {

template <typename T>
__global__ void __launch_bounds__(256) finite_kernel(const T* __restrict__ x, int64_t n, uint32_t* status) {
  bool bad = false;
  griddep_wait();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= nonfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// One CTA per layer: exact dense top-k over acc (zeroing the selected entries of acc).
template <typename T>
__global__ void __launch_bounds__(SEL_NT) select_dense_kernel(const lags_layer_t* __restrict__ layers,
                                                              lags_layer_t single, T* acc, int32_t* idx_out,
                                                              T* val_out, int32_t* count_out, int zero_selected) {
  __shared__ RadixSmem<Key<T>::RB> sm;
  const lags_layer_t L = layers ? layers[blockIdx.x] : single;
  const uint32_t cnt = exact_topk_dense<T, T>(acc + L.offset, L.dim, static_cast<uint32_t>(L.k),
                                              idx_out + L.slot, val_out + L.slot, zero_selected != 0, sm);
  if (threadIdx.x == 0) count_out[layers ? blockIdx.x : 0] = static_cast<int32_t>(cnt);
}

template <typename T>
__global__ void decompress_kernel(const int32_t* __restrict__ idx, const T* __restrict__ val,
                                  const int32_t* __restrict__ count, T* out) {
  const int32_t c = *count;
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) out[idx[j]] = val[j];
}

// ------------------------------------------------------------------------------------------
// decode + update.  Work item e = (rank p, slot s) over all layers of the bucket.
// P == 1: v[i] -= val (one kernel).  P > 1: phase A scatters each rank's values into its own
// dense plane and marks a rank bitmask; phase B lets the lowest rank holding index i add the
// planes in rank order in fp64 (R: training.py:248,253) and apply v - total / P (R: :254).
// ------------------------------------------------------------------------------------------
struct MsgView {
  const char* base;
  int64_t stride, off_cnt, off_idx, off_val;
  __device__ __forceinline__ int32_t count(int p, int j) const {
    return reinterpret_cast<const int32_t*>(base + p * stride + off_cnt)[j];
  }
  __device__ __forceinline__ int32_t idx(int p, int64_t s) const {
    return reinterpret_cast<const int32_t*>(base + p * stride + off_idx)[s];
  }
  template <typename TVal>
  __device__ __forceinline__ TVal val(int p, int64_t s) const {
    return reinterpret_cast<const TVal*>(base + p * stride + off_val)[s];
  }
};

template <typename TV, typename TVal>
__global__ void __launch_bounds__(256) decode_single_kernel(const lags_layer_t* __restrict__ layers,
                                                            const int32_t* __restrict__ slot_layer, MsgView msg,
                                                            int64_t total_k, TV* v) {
  griddep_wait();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total_k; s += stride) {
    const int j = slot_layer[s];
    const lags_layer_t L = layers[j];
    if (s - L.slot >= msg.count(0, j)) continue;
    const int64_t i = L.offset + msg.idx(0, s);
    const double total = __dadd_rn(0.0, static_cast<double>(msg.val<TVal>(0, s)));
    v[i] = static_cast<TV>(__dsub_rn(static_cast<double>(v[i]), total)  /* total / 1 == total */);
  }
}

// Work is tiled per (layer chunk, rank): CTA (t, p) handles pairs [c * DEC_NT, (c + 1) * DEC_NT)
// of rank p's list of layer j = tiles[t].x (c = tiles[t].y), one pair per thread, so a thread's
// dependent-load chain is tile -> (layer, count) -> pair -> planes (the latency-bound part).
constexpr int DEC_NT = 256;

// A decode tile with everything its threads need to address their pairs: the layer's first flat
// element and id, the tile's first message slot and entry, and how many of its DEC_NT slots lie in
// the layer (so the pair loads can be issued before the layer's count is known).
struct DecTile {
  int64_t offset;  // the layer's first flat element
  int32_t slot;    // message slot of the tile's first entry (layer slot + e0)
  int32_t layer;
  int32_t e0;      // the tile's first entry within the layer
  int32_t len;     // entries of the tile within the layer's k slots
};

template <typename TVal>
__global__ void __launch_bounds__(DEC_NT) decode_scatter_kernel(const lags_layer_t* __restrict__ layers,
                                                                const int2* __restrict__ tiles, MsgView msg, int P,
                                                                TVal* planes, int64_t n, uint32_t* mask) {
  griddep_wait();
  const int p = static_cast<int>(blockIdx.x) % P;
  const int2 tc = tiles[blockIdx.x / P];
  const lags_layer_t L = layers[tc.x];
  const int e = tc.y * DEC_NT + static_cast<int>(threadIdx.x);
  if (e >= msg.count(p, tc.x)) return;
  const int64_t s = L.slot + e;
  const int64_t i = L.offset + msg.idx(p, s);
  planes[static_cast<int64_t>(p) * n + i] = msg.val<TVal>(p, s);
  atomicOr(mask + i, 1u << p);
}

template <typename TV, typename TVal>
__global__ void __launch_bounds__(DEC_NT) decode_update_kernel(const lags_layer_t* __restrict__ layers,
                                                               const int2* __restrict__ tiles, MsgView msg, int P,
                                                               const TVal* planes, int64_t n, uint32_t* mask, TV* v) {
  griddep_wait();
  const int p = static_cast<int>(blockIdx.x) % P;
  const int2 tc = tiles[blockIdx.x / P];
  const lags_layer_t L = layers[tc.x];
  const int e = tc.y * DEC_NT + static_cast<int>(threadIdx.x);
  if (e >= msg.count(p, tc.x)) return;
  const int64_t i = L.offset + msg.idx(p, L.slot + e);
  const uint32_t bits = mask[i];
  if (bits == 0 || (__ffs(bits) - 1) != p) return;  // only the lowest holding rank applies
  const double vi = static_cast<double>(v[i]);
  double total = 0.0;
  for (uint32_t b = bits; b; b &= b - 1) {
    const int q = __ffs(b) - 1;
    total = __dadd_rn(total, static_cast<double>(planes[static_cast<int64_t>(q) * n + i]));
  }
  v[i] = static_cast<TV>(__dsub_rn(vi, div_workers(total, P)));
  mask[i] = 0u;
}

// Rank-ordered fp64 sum of the planes holding element i (bits = its rank mask): the loads of a
// batch of 8 ranks are issued together (predicated), then added in rank order (R: training.py:248,253).
template <typename TVal>
__device__ __forceinline__ double plane_sum(const TVal* planes, int64_t n, int64_t i, uint32_t bits, int P) {
  double total = 0.0;
  for (int q0 = 0; q0 < P; q0 += 8) {
    TVal x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      x[u] = (bits >> (q0 + u)) & 1u ? planes[static_cast<int64_t>(q0 + u) * n + i] : TVal(0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if ((bits >> (q0 + u)) & 1u) total = __dadd_rn(total, static_cast<double>(x[u]));
  }
  return total;
}

// Momentum update of one element: m = fl(mu m + upd), v = fl(v - m) with fp64 intermediates, upd =
// total / P (+0.0 for an element no rank sent: 0 / P without the division).
template <typename TV>
__device__ __forceinline__ void momentum_update(TV& v, TV& m, double upd, double mu) {
#ifdef LAGS_MOM_F32_PROBE  // diagnostic only (different rounding): is the fp64 arithmetic the bound?
  const float mf = __fadd_rn(__fmul_rn(static_cast<float>(mu), static_cast<float>(m)), static_cast<float>(upd));
  m = static_cast<TV>(mf);
  v = static_cast<TV>(__fsub_rn(static_cast<float>(v), mf));
  return;
#endif
  const double mnew = __dadd_rn(__dmul_rn(mu, static_cast<double>(m)), upd);
  m = static_cast<TV>(mnew);
  v = static_cast<TV>(__dsub_rn(static_cast<double>(v), mnew));
}

// The whole decode of P > 1 messages in ONE cooperative launch: phase A scatters every rank's
// pairs into its plane and marks the rank bitmask; a grid-wide barrier; phase B lets the lowest
// rank holding index i sum the planes in rank order (fp64) and apply v - total / P
// (R: training.py:248,253-254) -- each thread keeps its ITEMS (element, rank) pairs in registers
// across the barrier, so phase B starts from the mask without re-reading the messages.  With
// momentum (mu > 0) phase B is a dense pass over the bucket (16-byte vectors when v and m are
// aligned): m = mu m + total / P, v -= m.
template <typename TV, typename TVal, int ITEMS, bool MOM>
__global__ void __launch_bounds__(DEC_NT) decode_fused_kernel(const DecTile* __restrict__ tiles, int ntiles, MsgView msg,
                                                              int P, TVal* planes, int64_t n, uint32_t* mask, TV* v,
                                                              TV* mom, double mu, uint32_t* touched) {
  griddep_wait();
  const int nitems = P * ntiles;
  int64_t ii[ITEMS];
  int pp[ITEMS];
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const int c = static_cast<int>(blockIdx.x) + u * static_cast<int>(gridDim.x);
    ii[u] = -1;
    pp[u] = 0;
    if (c < nitems) {
      const int p = c % P;
      const DecTile tl = tiles[c / P];
      const int e = static_cast<int>(threadIdx.x);
      // the pair and the layer's count in one round trip (the slot is inside the layer's k slots)
      int32_t cnt = 0, ix = 0;
      TVal x = TVal(0);
      if (e < tl.len) {
        cnt = msg.count(p, tl.layer);
        ix = msg.idx(p, tl.slot + e);
        x = msg.val<TVal>(p, tl.slot + e);
      }
      if (e < tl.len && tl.e0 + e < cnt) {
        const int64_t i = tl.offset + ix;
        planes[static_cast<int64_t>(p) * n + i] = x;
        atomicOr(mask + i, 1u << p);
        if (MOM) atomicOr(touched + (i >> 5), 1u << (i & 31));  // the dense pass skips the mask
        ii[u] = i;
        pp[u] = p;
      }
    }
  }
  cooperative_groups::this_grid().sync();  // every rank's pairs are in the planes and the mask
  if (!MOM) {
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int64_t i = ii[u];
      if (i < 0) continue;
      const uint32_t bits = mask[i];
      const TV vold = v[i];  // in flight with the mask
      if (bits == 0 || (__ffs(bits) - 1) != pp[u]) continue;  // only the lowest holding rank applies
      const double vi = static_cast<double>(vold);
      const double total = plane_sum(planes, n, i, bits, P);
      v[i] = static_cast<TV>(__dsub_rn(vi, div_workers(total, P)));
      mask[i] = 0u;
    }
    return;
  }
  // dense momentum pass, one 16-byte vector of v and m per thread and iteration: the touched
  // bitmap (1 bit per element, 8 threads share a word through L1) replaces the per-element rank
  // mask, which only the touched elements read, so the pass moves 16 B per element (v and m read
  // and written); each thread clears its own bits of the bitmap (atomicAnd, touched groups only)
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  constexpr int VW = 16 / sizeof(TV);  // elements per 16-byte vector
  using VT = typename std::conditional<sizeof(TV) == 4, float4, double2>::type;
  const bool vec = ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(mom)) & 15u) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n / VW;
    VT* v4 = reinterpret_cast<VT*>(v);
    VT* m4 = reinterpret_cast<VT*>(mom);
    for (int64_t q = tid; q < nv; q += nthreads) {
      const int64_t i0 = q * VW;
      const uint32_t sh = static_cast<uint32_t>(i0 & 31);
      const uint32_t grp = (__ldg(touched + (i0 >> 5)) >> sh) & ((1u << VW) - 1u);
      VT vv = __ldcs(v4 + q), mm = __ldcs(m4 + q);
      TV* ve = reinterpret_cast<TV*>(&vv);
      TV* me = reinterpret_cast<TV*>(&mm);
#pragma unroll
      for (int u = 0; u < VW; ++u) {
        double upd = 0.0;
        if ((grp >> u) & 1u) {
          const uint32_t bits = mask[i0 + u];
          upd = div_workers(plane_sum(planes, n, i0 + u, bits, P), P);
          mask[i0 + u] = 0u;
        }
        momentum_update(ve[u], me[u], upd, mu);
      }
      __stcs(v4 + q, vv);
      __stcs(m4 + q, mm);
      if (grp) atomicAnd(touched + (i0 >> 5), ~(((1u << VW) - 1u) << sh));
    }
    done = nv * VW;
  }
  for (int64_t i = done + tid; i < n; i += nthreads) {  // unaligned buffers / the tail
    const uint32_t bits = mask[i];
    const double upd = bits ? div_workers(plane_sum(planes, n, i, bits, P), P) : 0.0;
    if (bits) {
      mask[i] = 0u;
      atomicAnd(touched + (i >> 5), ~(1u << (i & 31)));
    }
    TV vi = v[i], mi = mom[i];
    momentum_update(vi, mi, upd, mu);
    mom[i] = mi;
    v[i] = vi;
  }
}

template <typename TV, typename TVal>
__global__ void __launch_bounds__(256) decode_momentum_kernel(const TVal* planes, int64_t n, uint32_t* mask, int P,
                                                              TV* v, TV* mom, double mu) {
  griddep_wait();
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
    const double mnew =
        __dadd_rn(__dmul_rn(mu, static_cast<double>(mom[i])), div_workers(total, P));
    mom[i] = static_cast<TV>(mnew);
    v[i] = static_cast<TV>(__dsub_rn(static_cast<double>(v[i]), mnew));
  }
}

// ------------------------------------------------------------------------------------------
// diagnostics: aggregation-quality ratio delta^(l) (R: analysis.py:24-56, as the train loop
// evaluates it on the accumulated vectors, R: training.py:320-337).  acc_p = accumulated vector
// of worker p, r_p = acc_p with its selected entries zeroed (the new residual), so acc_p - r_p is
// exactly the decompressed top-k pick: total = sum_p acc_p, agg = sum_p (acc_p - r_p) in fp64 in
// worker order as the reference adds them; per task (one layer slice, one warp) the partial sums
// of (total - agg)^2 and total^2, reduced per layer in task order (deterministic).
// ------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) delta_partial_kernel(const Task* __restrict__ tasks, int ntasks,
                                                            const T* __restrict__ acc, const T* __restrict__ r,
                                                            int64_t stride, int P, double* part) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  griddep_wait();
  if (w >= ntasks) return;
  const Task tk = tasks[w];
  double num = 0.0, den = 0.0;
  for (int64_t i = tk.start + lane; i < tk.start + tk.len; i += 32) {
    double tot = static_cast<double>(acc[i]);
    double agg = __dadd_rn(0.0, __dsub_rn(tot, static_cast<double>(r[i])));
    for (int p = 1; p < P; ++p) {
      const double a = static_cast<double>(acc[p * stride + i]);
      tot = __dadd_rn(tot, a);
      agg = __dadd_rn(agg, __dsub_rn(a, static_cast<double>(r[p * stride + i])));
    }
    const double diff = __dsub_rn(tot, agg);
    num = __fma_rn(diff, diff, num);
    den = __fma_rn(tot, tot, den);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num = __dadd_rn(num, __shfl_down_sync(0xffffffffu, num, o));
    den = __dadd_rn(den, __shfl_down_sync(0xffffffffu, den, o));
  }
  if (lane == 0) {
    part[2 * w] = num;
    part[2 * w + 1] = den;
  }
}

// delta_l = ||total - agg||^2 / ((1 - k/d) ||total||^2); NaN when the denominator vanishes
// (the reference returns None there).
__global__ void delta_final_kernel(const lags_layer_t* __restrict__ layers, const int2* __restrict__ layer_tasks,
                                   int nlayers, const double* __restrict__ part, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  griddep_wait();
  if (j >= nlayers) return;
  const int2 tr = layer_tasks[j];
  double num = 0.0, den = 0.0;
  for (int t = tr.x; t < tr.y; ++t) {
    num = __dadd_rn(num, part[2 * t]);
    den = __dadd_rn(den, part[2 * t + 1]);
  }
  const lags_layer_t L = layers[j];
  const double denom =
      __dmul_rn(__dsub_rn(1.0, __ddiv_rn(static_cast<double>(L.k), static_cast<double>(L.dim))), den);
  out[j] = denom == 0.0 ? __longlong_as_double(0x7ff8000000000000ll) : __ddiv_rn(num, denom);
}

// ------------------------------------------------------------------------------------------
// residual-identity monitor (R: training.py:356-369 with the dense shadow sequence of
// R: training.py:197-200): x -= (alpha * sum_p g_p) / P every step, and on logged steps per layer
// ||mean residual||, plus ||v - x|| and max |(v - x) - mean residual| (Eq. 10: the gap between
// the sparsified and the dense sequence is exactly the mean error-feedback residual).
// ------------------------------------------------------------------------------------------
template <typename TV>
__global__ void __launch_bounds__(256) shadow_step_kernel(const TV* __restrict__ gsum, double* x, double alpha, int P,
                                                          int64_t n) {
  griddep_wait();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    x[i] = __dsub_rn(x[i], __ddiv_rn(__dmul_rn(alpha, static_cast<double>(gsum[i])), static_cast<double>(P)));
}

template <typename TV>
__global__ void __launch_bounds__(256) identity_partial_kernel(const Task* __restrict__ tasks, int ntasks,
                                                               const TV* __restrict__ v, const double* __restrict__ x,
                                                               const TV* __restrict__ rsum, int P, double* part) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  griddep_wait();
  if (w >= ntasks) return;
  const Task tk = tasks[w];
  double gsq = 0.0, msq = 0.0, dmax = 0.0;
  for (int64_t i = tk.start + lane; i < tk.start + tk.len; i += 32) {
    const double gap = __dsub_rn(static_cast<double>(v[i]), x[i]);
    const double mres = __ddiv_rn(static_cast<double>(rsum[i]), static_cast<double>(P));
    gsq = __fma_rn(gap, gap, gsq);
    msq = __fma_rn(mres, mres, msq);
    dmax = fmax(dmax, fabs(__dsub_rn(gap, mres)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gsq = __dadd_rn(gsq, __shfl_down_sync(0xffffffffu, gsq, o));
    msq = __dadd_rn(msq, __shfl_down_sync(0xffffffffu, msq, o));
    dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
  }
  if (lane == 0) {
    part[3 * w] = gsq;
    part[3 * w + 1] = msq;
    part[3 * w + 2] = dmax;
  }
}

// out[j] = sum of mean-residual squares of layer j; out[L] = sum of gap squares; out[L+1] = max
// deviation (one CTA, deterministic task order).
__global__ void identity_final_kernel(const int2* __restrict__ layer_tasks, int nlayers,
                                      const double* __restrict__ part, double* out) {
  griddep_wait();
  for (int j = threadIdx.x; j < nlayers; j += blockDim.x) {
    const int2 tr = layer_tasks[j];
    double msq = 0.0;
    for (int t = tr.x; t < tr.y; ++t) msq = __dadd_rn(msq, part[3 * t + 1]);
    out[j] = msq;
  }
  if (threadIdx.x == 0) {
    double gsq = 0.0, dmax = 0.0;
    for (int j = 0; j < nlayers; ++j) {
      const int2 tr = layer_tasks[j];
      for (int t = tr.x; t < tr.y; ++t) {
        gsq = __dadd_rn(gsq, part[3 * t]);
        dmax = fmax(dmax, part[3 * t + 2]);
      }
    }
    out[nlayers] = gsq;
    out[nlayers + 1] = dmax;
  }
}

// acc_p[L.offset + idx] = val for every sent pair of message p (acc_p pre-filled with r_p).
template <typename T>
__global__ void __launch_bounds__(256) reconstruct_kernel(const lags_layer_t* __restrict__ layers,
                                                          const int32_t* __restrict__ slot_layer, MsgView msg,
                                                          int64_t total_k, int P, T* acc, int64_t stride) {
  griddep_wait();
  const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total_k * P; e += gs) {
    const int p = static_cast<int>(e / total_k);
    const int64_t s = e - static_cast<int64_t>(p) * total_k;
    const int j = slot_layer[s];
    const lags_layer_t L = layers[j];
    if (s - L.slot >= msg.count(p, j)) continue;
    acc[p * stride + L.offset + msg.idx(p, s)] = msg.val<T>(p, s);
  }
}

}  // namespace lags

// ==========================================================================================
// host side
// ==========================================================================================

using namespace lags;

struct lags_bucket {
  int32_t dtype = 0, nlayers = 0, ntasks = 0, max_world = 1, cap = 0, smem_keys = 0;
  int64_t n_total = 0, total_k = 0;
  int64_t off_cnt = 0, off_idx = 0, off_val = 0, msg_bytes = 0;
  // device pointers inside the caller's memory
  lags_layer_t* layers = nullptr;
  int2* layer_tasks = nullptr;
  FastState* state = nullptr;
  Task* tasks = nullptr;
  int32_t* slot_layer = nullptr;
  int32_t* cand_cnt = nullptr;
  int32_t* cand_idx = nullptr;
  float* cand_val = nullptr;   // LAGS_F32 candidate values (cand_val64 for LAGS_F64 / LAGS_F32_ACC64)
  double* cand_val64 = nullptr;
  double* gval64 = nullptr;
  State64* state64 = nullptr;   // LAGS_F64 / LAGS_F32_ACC64 selection state
  int32_t* gidx = nullptr;
  float* gval = nullptr;
  double* acc64 = nullptr;
  uint32_t* mask = nullptr;
  char* planes = nullptr;
  int32_t* order = nullptr;  // layers by decreasing selection work, group by group (persistent-role schedule)
  int2* tiles_dec = nullptr;  // decode tiles: (layer, chunk of DEC_NT slots)
  DecTile* dtiles = nullptr;  // the same tiles with their layer offset / slot (fused decode)
  int dec_tiles = 0;
  double* delta_part = nullptr;  // [2 * ntasks] lags_bucket_delta partial sums
  uint32_t* hist = nullptr;       // fp32: per-layer candidate-key histograms (K1 -> select_kernel)
  uint32_t* touched = nullptr;    // decode with momentum: one bit per element sent by any rank
  bool r_stream = true;           // K1 streams r with evict-first priority (r larger than half the L2)
  bool k1_wide = false;           // K1 with 2 * K1_UNROLL loads in flight (fuller waves for this bucket)
  bool k1_cta = false;            // K1 in its CTA form (Plan::k1_cta)
  // selection groups of an fp32 bucket (plan_groups): 0 persistent role, 1 cluster role, 2 warp
  // role; each group's tasks and `order` entries are contiguous
  struct Group {
    int task_base = 0, ntasks = 0;    // contiguous range of the task table
    int order_base = 0, nlayers = 0;  // contiguous range of `order`
  };
  Group grp[3];
  SelectCounters sel_ctr{};  // per-call selection counter (persistent role)
  cudaEvent_t probe_before = nullptr, probe_after = nullptr;  // caller-owned, optional
  float* const* grad_table = nullptr;  // caller-owned device array of per-layer gradient pointers
};

namespace {
thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
}  // namespace

int lags::host_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
void lags::host_count_launches(int n) {
  g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed);
}

namespace {
int fail(int code, const std::string& msg) { return host_fail(code, msg); }

int cuda_check(const char* where, int launches = 1) {
  g_launches.fetch_add(static_cast<unsigned long long>(launches), std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return LAGS_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int num_sms();
// Resident warps of K1 (the narrow unroll) over the whole device: one wave of tasks.
int64_t k1_resident_warps() {
  static int64_t w = 0;
  if (w == 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, accum_emit_kernel<false, true>, K1_WARPS * 32, 0) !=
            cudaSuccess ||
        occ <= 0) {
      cudaGetLastError();
      occ = 3;  // 80 registers, 8-warp CTAs
    }
    w = static_cast<int64_t>(occ) * K1_WARPS * num_sms();
  }
  return w;
}

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
  const int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

bool valid_dtype(int32_t dtype) { return dtype == LAGS_F32 || dtype == LAGS_F64 || dtype == LAGS_F32_ACC64; }
size_t val_size(int32_t dtype) { return dtype == LAGS_F32 ? 4 : 8; }

// Shared-memory staging words of select_kernel: the device's opt-in maximum per block minus the
// kernel's static shared memory (B200: ~48 k words = ~190 KB).
int select_smem_words_max() {
  static int words = 0;
  if (words == 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, select_kernel);
    words = static_cast<int>((static_cast<size_t>(optin) - fa.sharedSizeBytes - 1024) / sizeof(uint32_t)) / 1024 * 1024;
    if (words < 16384) words = 16384;
  }
  return words;
}

// Device memory layout shared by lags_bucket_device_bytes and lags_bucket_create.
struct Plan {
  int64_t n_total = 0, total_k = 0;
  int32_t ntasks = 0, cap = 0, task_elems = TASK_ELEMS;
  bool k1_cta = false;  // K1 in its CTA form (accum_emit_cta_kernel, K1C_TASK-element tasks)
  size_t o_layers = 0, o_ltasks = 0, o_state = 0, o_tasks = 0, o_slot = 0, o_ccnt = 0, o_cidx = 0, o_cval = 0,
         o_gidx = 0, o_gval = 0, o_acc = 0, o_mask = 0, o_planes = 0, o_order = 0, o_ctr = 0, o_delta = 0, o_tiles = 0,
         o_hist = 0, o_touched = 0, o_state64 = 0, o_dtiles = 0, bytes = 0;
  int32_t ntiles = 0;
};

int make_plan(int32_t dtype, const int64_t* dims, const int32_t* ks, int32_t L, int32_t max_world, Plan* p) {
  if (!valid_dtype(dtype)) return fail(LAGS_ERR_INVALID_ARG, "unknown dtype");
  if (!dims || !ks || L <= 0) return fail(LAGS_ERR_INVALID_ARG, "empty bucket");
  if (max_world < 1 || max_world > 32) return fail(LAGS_ERR_INVALID_ARG, "max_world must be in 1..32");
  // task size: TASK_ELEMS, smaller for small buckets so that K1 still has about a warp per SM
  // slot (ResNet-20's 0.27 M elements in 8192-element tasks were 34 warps: 20 us of latency)
  int64_t n_all = 0;
  for (int j = 0; j < L; ++j) n_all += std::max<int64_t>(dims[j], 0);
  int task = TASK_ELEMS;
  while (task > MIN_TASK_ELEMS && n_all / task < static_cast<int64_t>(num_sms()) * K1_WARPS) task >>= 1;
#ifndef LAGS_NO_K1_CTA
  // large fp32 buckets: K1's CTA form, one short CTA per K1C_TASK-element task
  if (dtype == LAGS_F32 && task == TASK_ELEMS) {
    task = K1C_TASK;
    p->k1_cta = true;
  }
#endif
#ifndef LAGS_NO_WAVE_FIT
  // a bucket that fits one wave of resident K1 warps: the smallest task (multiple of 256 elements)
  // that still fits, so every warp streams about the same bytes and the wave is full (ResNet-50:
  // 3120 tasks of 8192 for 3552 warp slots -> 7168-element tasks)
  if (task == TASK_ELEMS && !p->k1_cta) {
    auto ntasks_for = [&](int t) {
      int64_t c = 0;
      for (int j = 0; j < L; ++j) c += (std::max<int64_t>(dims[j], 1) + t - 1) / t;
      return c;
    };
    const int64_t slots = k1_resident_warps();
    if (ntasks_for(task) <= slots)
      while (task - 256 >= MIN_TASK_ELEMS && ntasks_for(task - 256) <= slots) task -= 256;
  }
#endif
  p->task_elems = task;
  double max_per_task = 0.0;  // expected selected entries in one task of a layer
  for (int j = 0; j < L; ++j) {
    if (dims[j] < 1) return fail(LAGS_ERR_STRUCTURE, "layer " + std::to_string(j + 1) + ": dim must be positive");
    if (dims[j] > 0x7fffffffLL) return fail(LAGS_ERR_INVALID_ARG, "layer dim exceeds the int32 index range");
    if (ks[j] < 1 || ks[j] > dims[j])
      return fail(LAGS_ERR_K_OUT_OF_RANGE, "k=" + std::to_string(ks[j]) + " outside 1.." + std::to_string(dims[j]));
    p->n_total += dims[j];
    p->total_k += ks[j];
    p->ntasks += static_cast<int32_t>((dims[j] + task - 1) / task);
    p->ntiles += (ks[j] + DEC_NT - 1) / DEC_NT;
    max_per_task = std::max(max_per_task, static_cast<double>(ks[j]) * std::min<int64_t>(dims[j], task) / dims[j]);
  }
  // per-task candidate capacity: 16x the expected PRED_FACTOR * (selected per task), power of two
  // in [256, TASK]
  const double want = 16.0 * PRED_FACTOR * max_per_task;
  int cap = 256;
  while (cap < want && cap < task) cap <<= 1;
  p->cap = cap;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  const size_t nt = static_cast<size_t>(p->ntasks), cp = static_cast<size_t>(p->cap);
  p->o_layers = take(sizeof(lags_layer_t) * L);
  p->o_ltasks = take(sizeof(int2) * L);
  p->o_state = take(sizeof(FastState) * L);
  p->o_tasks = take(sizeof(Task) * nt);
  p->o_slot = take(sizeof(int32_t) * static_cast<size_t>(p->total_k));
  p->o_ccnt = take(sizeof(int32_t) * nt);
  p->o_cidx = take(sizeof(int32_t) * nt * cp);
  p->o_cval = take(val_size(dtype) * nt * cp);
  p->o_gidx = take(sizeof(int32_t) * nt * cp);
  p->o_gval = take(val_size(dtype) * nt * cp);
  p->o_state64 = take(dtype != LAGS_F32 ? sizeof(State64) * L : 0);
  p->o_acc = take(dtype == LAGS_F32_ACC64 ? sizeof(double) * static_cast<size_t>(p->n_total) : 0);
  p->o_mask = take(sizeof(uint32_t) * static_cast<size_t>(p->n_total));
  p->o_planes = take(val_size(dtype) * static_cast<size_t>(p->n_total) * static_cast<size_t>(max_world));
  p->o_order = take(sizeof(int32_t) * L);
  p->o_delta = take(3 * sizeof(double) * nt);  // delta (2 per task) / identity monitor (3 per task)
  p->o_tiles = take(sizeof(int2) * static_cast<size_t>(p->ntiles));
  const bool f32 = dtype == LAGS_F32;
  p->o_ctr = take(f32 ? 2 * sizeof(uint32_t) : 0);  // selection counter (SelectCounters) + fused-push CTA count
  p->o_hist = take(f32 ? sizeof(uint32_t) * HIST_BINS * static_cast<size_t>(L) : 0);
  p->o_touched = take(sizeof(uint32_t) * static_cast<size_t>(p->n_total / 32 + 1));
  p->o_dtiles = take(sizeof(DecTile) * static_cast<size_t>(p->ntiles));
  p->bytes = o;
  return LAGS_OK;
}

// Selection groups of an fp32 bucket: 0 = one CTA per layer (select_kernel's persistent role),
// 1 = the largest layers, one thread-block cluster per layer (select_kernel's cluster role),
// 2 = tiny layers (d <= WARP_MAX_DIM) with k <= WARP_TOPK, one warp per layer (select_kernel's warp
// role; a warp's two passes over a 4096-element layer took longer than a whole CTA's dense path).
std::vector<int> plan_groups(const int64_t* dims, const int32_t* ks, int L) {
  std::vector<int> gid(L, 0);
  for (int j = 0; j < L; ++j) {
    if (dims[j] > SMALL_LAYER && ks[j] >= CLUSTER_MIN_K) gid[j] = 1;
    else if (dims[j] <= WARP_MAX_DIM && ks[j] <= WARP_TOPK) gid[j] = 2;
  }
  return gid;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool aligned_to(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while the
// previous kernel on the stream drains; it calls griddep_wait() before touching its inputs.
// The same with a thread-block cluster size (1 = no clusters).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace

extern "C" {

int lags_abi_version(void) { return 3; }
const char* lags_last_error(void) { return g_last_error.c_str(); }
unsigned long long lags_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

size_t lags_bucket_device_bytes(int32_t dtype, const int64_t* dims, const int32_t* ks, int32_t nlayers,
                                int32_t max_world) {
  Plan p;
  if (make_plan(dtype, dims, ks, nlayers, max_world, &p) != LAGS_OK) return 0;
  return p.bytes + 256;  // slack for aligning the caller's pointer
}

int lags_bucket_create(int32_t dtype, const int64_t* dims, const int32_t* ks, int32_t nlayers, int32_t max_world,
                       void* device_mem, size_t bytes, lags_stream_t stream, lags_bucket_t** out) {
  if (!out || !device_mem) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_create: null pointer");
  Plan p;
  const int rc = make_plan(dtype, dims, ks, nlayers, max_world, &p);
  if (rc) return rc;
  char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(device_mem), 256));
  if (base + p.bytes > static_cast<char*>(device_mem) + bytes)
    return fail(LAGS_ERR_WORKSPACE, "lags_bucket_create: device memory too small");
  lags_bucket* b = new lags_bucket();
  b->dtype = dtype;
  b->nlayers = nlayers;
  b->ntasks = p.ntasks;
  b->max_world = max_world;
  b->cap = p.cap;
  b->n_total = p.n_total;
  b->total_k = p.total_k;
  b->layers = reinterpret_cast<lags_layer_t*>(base + p.o_layers);
  b->layer_tasks = reinterpret_cast<int2*>(base + p.o_ltasks);
  b->state = reinterpret_cast<FastState*>(base + p.o_state);
  b->tasks = reinterpret_cast<Task*>(base + p.o_tasks);
  b->slot_layer = reinterpret_cast<int32_t*>(base + p.o_slot);
  b->cand_cnt = reinterpret_cast<int32_t*>(base + p.o_ccnt);
  b->cand_idx = reinterpret_cast<int32_t*>(base + p.o_cidx);
  b->cand_val = reinterpret_cast<float*>(base + p.o_cval);
  b->gidx = reinterpret_cast<int32_t*>(base + p.o_gidx);
  b->gval = reinterpret_cast<float*>(base + p.o_gval);
  b->cand_val64 = reinterpret_cast<double*>(base + p.o_cval);
  b->gval64 = reinterpret_cast<double*>(base + p.o_gval);
  b->state64 = dtype != LAGS_F32 ? reinterpret_cast<State64*>(base + p.o_state64) : nullptr;
  b->acc64 = reinterpret_cast<double*>(base + p.o_acc);
  b->mask = reinterpret_cast<uint32_t*>(base + p.o_mask);
  b->planes = base + p.o_planes;
  b->order = reinterpret_cast<int32_t*>(base + p.o_order);
  b->delta_part = reinterpret_cast<double*>(base + p.o_delta);
  b->tiles_dec = reinterpret_cast<int2*>(base + p.o_tiles);
  b->dtiles = reinterpret_cast<DecTile*>(base + p.o_dtiles);
  b->dec_tiles = p.ntiles;
  b->sel_ctr.work = reinterpret_cast<uint32_t*>(base + p.o_ctr);
  b->hist = dtype == LAGS_F32 ? reinterpret_cast<uint32_t*>(base + p.o_hist) : nullptr;
  b->touched = reinterpret_cast<uint32_t*>(base + p.o_touched);
  b->off_cnt = 0;
  b->off_idx = static_cast<int64_t>(align_up(4 * static_cast<size_t>(nlayers), 16));
  b->off_val = static_cast<int64_t>(align_up(b->off_idx + 4 * static_cast<size_t>(p.total_k), 16));
  b->msg_bytes = static_cast<int64_t>(align_up(b->off_val + val_size(dtype) * static_cast<size_t>(p.total_k), 16));
  // host tables.  fp32 buckets are split into selection groups (plan_groups); the task table holds
  // them group after group, so each group's tasks (and candidate lists) are one contiguous range.
  const std::vector<int> gid = dtype == LAGS_F32 ? plan_groups(dims, ks, nlayers) : std::vector<int>(nlayers, 0);
  std::vector<lags_layer_t> layers(nlayers);
  std::vector<int2> ltasks(nlayers);
  std::vector<Task> tasks;
  std::vector<int32_t> slot_layer(static_cast<size_t>(p.total_k));
  std::vector<int64_t> offs(nlayers);
  tasks.reserve(p.ntasks);
  int64_t off = 0, slot = 0;
  for (int j = 0; j < nlayers; ++j) {
    layers[j] = lags_layer_t{off, dims[j], ks[j], static_cast<int32_t>(slot)};
    offs[j] = off;
    for (int32_t q = 0; q < ks[j]; ++q) slot_layer[slot + q] = j;
    off += dims[j];
    slot += ks[j];
  }
  for (int g = 0; g < 3; ++g) {
    b->grp[g].task_base = static_cast<int>(tasks.size());
    for (int j = 0; j < nlayers; ++j) {
      if (gid[j] != g) continue;
      ltasks[j].x = static_cast<int>(tasks.size());
      for (int64_t s = 0; s < dims[j]; s += p.task_elems)
        tasks.push_back(Task{offs[j] + s, static_cast<int32_t>(std::min<int64_t>(p.task_elems, dims[j] - s)), j});
      ltasks[j].y = static_cast<int>(tasks.size());
    }
    b->grp[g].ntasks = static_cast<int>(tasks.size()) - b->grp[g].task_base;
  }
  // schedule of the selection kernel's persistent role: longest (estimated) work first, group by group
  std::vector<int32_t> order;
  std::vector<double> cost(nlayers);
  for (int j = 0; j < nlayers; ++j)
    cost[j] = dims[j] <= SMALL_LAYER ? 5.0 * dims[j] : 40.0 * ks[j] + 64.0 * (ltasks[j].y - ltasks[j].x);
  for (int g = 0; g < 3; ++g) {
    b->grp[g].order_base = static_cast<int>(order.size());
    std::vector<int32_t> og;
    for (int j = 0; j < nlayers; ++j)
      if (gid[j] == g) og.push_back(j);
    std::stable_sort(og.begin(), og.end(), [&](int a, int c) { return cost[a] > cost[c]; });
    order.insert(order.end(), og.begin(), og.end());
    b->grp[g].nlayers = static_cast<int>(og.size());
  }
  std::vector<int2> tiles;  // decode tiles
  std::vector<DecTile> dtiles;
  for (int j = 0; j < nlayers; ++j)
    for (int c = 0; c * DEC_NT < ks[j]; ++c) {
      tiles.push_back(make_int2(j, c));
      dtiles.push_back(DecTile{offs[j], static_cast<int32_t>(layers[j].slot + c * DEC_NT), j, c * DEC_NT,
                               std::min(DEC_NT, ks[j] - c * DEC_NT)});
    }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool ok =
      cudaMemcpyAsync(b->layers, layers.data(), sizeof(lags_layer_t) * nlayers, cudaMemcpyHostToDevice, s) ==
          cudaSuccess &&
      cudaMemcpyAsync(b->layer_tasks, ltasks.data(), sizeof(int2) * nlayers, cudaMemcpyHostToDevice, s) ==
          cudaSuccess &&
      cudaMemcpyAsync(b->tasks, tasks.data(), sizeof(Task) * tasks.size(), cudaMemcpyHostToDevice, s) == cudaSuccess &&
      cudaMemcpyAsync(b->slot_layer, slot_layer.data(), sizeof(int32_t) * slot_layer.size(), cudaMemcpyHostToDevice,
                      s) == cudaSuccess &&
      cudaMemcpyAsync(b->order, order.data(), sizeof(int32_t) * nlayers, cudaMemcpyHostToDevice, s) ==
          cudaSuccess &&
      cudaMemcpyAsync(b->dtiles, dtiles.data(), sizeof(DecTile) * dtiles.size(), cudaMemcpyHostToDevice, s) ==
          cudaSuccess &&
      cudaMemcpyAsync(b->tiles_dec, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, s) ==
          cudaSuccess &&
      cudaMemsetAsync(b->state, 0, sizeof(FastState) * nlayers, s) == cudaSuccess &&
      (dtype == LAGS_F32 || cudaMemsetAsync(b->state64, 0, sizeof(State64) * nlayers, s) == cudaSuccess) &&
      cudaMemsetAsync(b->mask, 0, sizeof(uint32_t) * static_cast<size_t>(p.n_total), s) == cudaSuccess &&
      cudaMemsetAsync(b->touched, 0, sizeof(uint32_t) * static_cast<size_t>(p.n_total / 32 + 1), s) == cudaSuccess &&
      (dtype != LAGS_F32 || cudaMemsetAsync(b->sel_ctr.work, 0, 2 * sizeof(uint32_t), s) == cudaSuccess) &&
      (dtype != LAGS_F32 ||
       cudaMemsetAsync(b->hist, 0, sizeof(uint32_t) * HIST_BINS * static_cast<size_t>(nlayers), s) == cudaSuccess) &&
      cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) {
    delete b;
    return cuda_check("lags_bucket_create upload", 0);
  }
  if (dtype == LAGS_F32) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
#ifdef LAGS_NO_RSTREAM
    b->r_stream = false;
#else
    b->r_stream = static_cast<int64_t>(p.n_total) * 4 > static_cast<int64_t>(l2 > 0 ? l2 : (126 << 20)) / 2;
#endif
    b->k1_cta = p.k1_cta;
    // K1 runs one warp per task in waves of the resident warps; a partial last wave streams at a
    // fraction of the bandwidth.  Take the wider unroll when its waves are fuller (measured:
    // ResNet-50's 3120 tasks fit one 80-register wave, 68.8 vs 79.1 us; VGG-16's 1800 tasks and
    // LSTM's 8060 fill the 116-register waves better, 48.9 -> 45.7 and 187.8 -> 182.9 us).
    {
      int occ_n = 0, occ_w = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_n, accum_emit_kernel<false, true>, K1_WARPS * 32, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, accum_emit_kernel<false, true, 2 * K1_UNROLL>,
                                                    K1_WARPS * 32, 0);
      auto fill = [&](int occ) {
        const int64_t slots = static_cast<int64_t>(std::max(occ, 1)) * K1_WARPS * num_sms();
        const int64_t waves = (p.ntasks + slots - 1) / slots;
        return static_cast<double>(p.ntasks) / static_cast<double>(waves * slots);
      };
      b->k1_wide = occ_w > 0 && fill(occ_w) > fill(occ_n) + 0.05;
    }
    const int smem = select_smem_words_max() * static_cast<int>(sizeof(uint32_t));
    if (cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(select_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 0) != cudaSuccess) {
      delete b;
      return cuda_check("select kernel attributes", 0);
    }
    // shared-memory staging sized to the bucket: small layers are staged whole; a candidate set
    // (~2k at the adaptive margin) needs value + index words, a cluster layer m + 2 * m_max;
    // bigger sets fall back to global scratch.  Smaller staging leaves room for backprop kernels
    // co-resident on the SM when the compress runs beside them.
    int64_t words = 4096;
    for (int j = 0; j < nlayers; ++j)
      words = std::max<int64_t>(words, dims[j] <= SMALL_LAYER ? dims[j] : (15 * static_cast<int64_t>(ks[j])) / 2);
    b->smem_keys = static_cast<int>(std::min<int64_t>(align_up(static_cast<size_t>(words), 1024), select_smem_words_max()));
  }
  if (dtype != LAGS_F32) {
    static int words64 = 0;  // the device's opt-in shared memory minus select64_kernel's static part
    if (words64 == 0) {
      int dev = 0, optin = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, select64_kernel);
      words64 = std::max(4096, static_cast<int>((static_cast<size_t>(optin) - fa.sharedSizeBytes - 1024) / 4) / 1024 * 1024);
      if (cudaFuncSetAttribute(select64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, words64 * 4) != cudaSuccess) {
        delete b;
        return cuda_check("select64 kernel attributes", 0);
      }
    }
    // candidate staging: value (2 words) + index per candidate, ~2.5 k of them at the adaptive margin
    int64_t words = 4096;
    for (int j = 0; j < nlayers; ++j) words = std::max<int64_t>(words, 3 * ((5 * static_cast<int64_t>(ks[j])) / 2) + 8);
    b->smem_keys = static_cast<int>(std::min<int64_t>(align_up(static_cast<size_t>(words), 1024), words64));
  }
  *out = b;
  return LAGS_OK;
}

void lags_bucket_destroy(lags_bucket_t* bucket) { delete bucket; }

int lags_bucket_message_layout(const lags_bucket_t* b, int64_t* off_counts, int64_t* off_idx, int64_t* off_val,
                               int64_t* msg_bytes) {
  if (!b) return fail(LAGS_ERR_INVALID_ARG, "null bucket");
  if (off_counts) *off_counts = b->off_cnt;
  if (off_idx) *off_idx = b->off_idx;
  if (off_val) *off_val = b->off_val;
  if (msg_bytes) *msg_bytes = b->msg_bytes;
  return LAGS_OK;
}

// compress of one worker; v_update (nullable, LAGS_F32 only) fuses the P = 1 update into the
// selection epilogue (lags_bucket_step_local).
static int compress_impl(lags_bucket_t* b, void* g, void* r, double alpha, void* msg, uint32_t* status,
                         uint32_t flags, void* v_update, lags_stream_t stream, const lags_peer_push_t* peer = nullptr) {
  const bool table = b && b->grad_table && b->dtype == LAGS_F32;
  if (!b || (!g && !table) || !r || !msg || !status)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_compress: null pointer");
  if (table) g = nullptr;  // the per-layer table replaces the flat gradient
  // g / r / v need only their element alignment (the streaming pass peels a scalar head up to
  // 16 bytes); the message is the library's own layout and stays 16-byte aligned
  const size_t ea = b->dtype == LAGS_F64 ? 8 : 4;
  if ((g && !aligned_to(g, ea)) || !aligned_to(r, ea) || (v_update && !aligned_to(v_update, ea)) || !aligned16(msg))
    return fail(LAGS_ERR_INVALID_ARG,
                "lags_bucket_compress: g / r / v must be element-aligned and msg 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* m = static_cast<char*>(msg);
  int32_t* cnt = reinterpret_cast<int32_t*>(m + b->off_cnt);
  int32_t* idx = reinterpret_cast<int32_t*>(m + b->off_idx);
  if (b->dtype == LAGS_F32) {
    const bool exact = (flags & LAGS_COMPRESS_EXACT) != 0;
    const float a = static_cast<float>(alpha);  // numpy casts a Python float to float32 (NEP 50)
    float* rr = static_cast<float*>(r);
    float* gg = static_cast<float*>(g);
    float* vals = reinterpret_cast<float*>(m + b->off_val);
    float* vu = static_cast<float*>(v_update);
    const int fe = exact ? 1 : 0;
    const bool zg = (flags & LAGS_COMPRESS_ZERO_GRAD) != 0;
    // K1 over every task (candidate lists indexed by global task id)
    const lags_bucket::Group& G0 = b->grp[0];
    const lags_bucket::Group& G1 = b->grp[1];
    const lags_bucket::Group& G2 = b->grp[2];
    const int ntasks = G0.ntasks + G1.ntasks + G2.ntasks;
    const int blocks = (ntasks + K1_WARPS - 1) / K1_WARPS;
    cudaError_t e = cudaSuccess;
    if (b->probe_before) e = cudaEventRecord(b->probe_before, s);
    if (e == cudaSuccess && b->k1_cta) {
      auto kern = zg ? (b->r_stream ? accum_emit_cta_kernel<true, true> : accum_emit_cta_kernel<true, false>)
                     : (b->r_stream ? accum_emit_cta_kernel<false, true> : accum_emit_cta_kernel<false, false>);
      e = launch_pdl(kern, dim3(ntasks), dim3(K1C_NT), 0, s, b->tasks, ntasks, b->layers, b->state, gg,
                     b->grad_table, rr, a, b->cap, b->cand_idx, b->cand_val, b->cand_cnt, status, b->sel_ctr.work,
                     b->hist);
    } else if (e == cudaSuccess) {
      auto kern = b->k1_wide
                      ? (zg ? (b->r_stream ? accum_emit_kernel<true, true, 2 * K1_UNROLL>
                                           : accum_emit_kernel<true, false, 2 * K1_UNROLL>)
                            : (b->r_stream ? accum_emit_kernel<false, true, 2 * K1_UNROLL>
                                           : accum_emit_kernel<false, false, 2 * K1_UNROLL>))
                      : (zg ? (b->r_stream ? accum_emit_kernel<true, true> : accum_emit_kernel<true, false>)
                            : (b->r_stream ? accum_emit_kernel<false, true> : accum_emit_kernel<false, false>));
      e = launch_pdl(kern, dim3(blocks), dim3(K1_WARPS * 32), 0, s, b->tasks, ntasks, b->layers, b->state, gg,
                     b->grad_table, rr, a, b->cap, b->cand_idx, b->cand_val, b->cand_cnt, status, b->sel_ctr.work,
                     b->hist);
    }
    if (e == cudaSuccess && b->probe_after) e = cudaEventRecord(b->probe_after, s);
    if (e == cudaSuccess) {
      // the selection: one launch (PDL behind K1).  Group 1 (the largest layers): one 4-CTA
      // cluster each; group 2 (tiny layers): one warp each; group 0: persistent CTAs, one wave
      // on the SMs the others leave free.
      const int ncl = G1.nlayers;
      const int cl = ncl > 0 ? CLUSTER : 1;
      const int tiny_ctas = (G2.nlayers + SEL_NT / 32 - 1) / (SEL_NT / 32);
      const int fixed = ncl * CLUSTER + tiny_ctas;
      const int per = std::min(G0.nlayers, std::max(SEL_MINB * num_sms() - fixed, num_sms() / 2));
      const int grid = (fixed + per + cl - 1) / cl * cl;  // a whole number of clusters
      PeerPush pp{};
      if (peer) {
        pp.bases = static_cast<const uint64_t*>(peer->bases);
        pp.P = peer->P;
        pp.rank = peer->rank;
        pp.G = peer->ctas_per_peer;
        pp.flags_bytes = peer->flags_bytes;
        pp.msg_bytes = b->msg_bytes;
        pp.off_cnt = b->off_cnt;
        pp.off_idx = b->off_idx;
        pp.off_val = b->off_val;
        pp.epoch = static_cast<const uint32_t*>(peer->epoch);
        pp.done = b->sel_ctr.work + 1;
      }
      e = launch_pdl_cluster(select_kernel, dim3(grid), dim3(SEL_NT), static_cast<size_t>(b->smem_keys) * 4, s, cl,
                             b->layers, b->layer_tasks, b->order + G1.order_base, ncl, b->order + G2.order_base,
                             G2.nlayers, b->order + G0.order_base, G0.nlayers, b->state, b->cand_cnt, b->cand_idx,
                             b->cand_val, b->cap, b->gidx, b->gval, rr, idx, vals, cnt, b->smem_keys, fe, b->sel_ctr, vu,
                             b->hist, pp);
    }
    const int launches = 2;
    if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string("compress launch: ") + cudaGetErrorString(e));

    return cuda_check("lags_bucket_compress(f32)", launches);
  }
  if (v_update) return fail(LAGS_ERR_INVALID_ARG, "fused single-rank update needs an LAGS_F32 bucket");
  // LAGS_F64 / LAGS_F32_ACC64: K1 (candidates above the predicted threshold) + one CTA per layer;
  // the mixed mode keeps the fp64 acc in the bucket memory and its fp32 residual in r
  const int ntasks = b->ntasks;
  const int blocks = (ntasks + K1_WARPS - 1) / K1_WARPS;
  const bool zg = (flags & LAGS_COMPRESS_ZERO_GRAD) != 0;
  const bool mixed = b->dtype == LAGS_F32_ACC64;
  double* acc = mixed ? b->acc64 : static_cast<double*>(r);
  cudaError_t e;
  if (mixed) {
    float* rr = static_cast<float*>(r);
    float* gg = static_cast<float*>(g);
    e = launch_pdl(zg ? accum_emit64_kernel<true, float> : accum_emit64_kernel<false, float>, dim3(blocks),
                   dim3(K1_WARPS * 32), 0, s, b->tasks, ntasks, b->layers, b->state64, gg, rr, b->acc64, alpha,
                   b->cap, b->cand_idx, b->cand_val64, b->cand_cnt, status);
  } else {
    double* rr = static_cast<double*>(r);
    double* gg = static_cast<double*>(g);
    e = launch_pdl(zg ? accum_emit64_kernel<true, double> : accum_emit64_kernel<false, double>, dim3(blocks),
                   dim3(K1_WARPS * 32), 0, s, b->tasks, ntasks, b->layers, b->state64, gg, rr,
                   static_cast<double*>(nullptr), alpha, b->cap, b->cand_idx, b->cand_val64, b->cand_cnt, status);
  }
  if (e == cudaSuccess)
    e = launch_pdl(select64_kernel, dim3(b->nlayers), dim3(SEL_NT), static_cast<size_t>(b->smem_keys) * 4, s,
                   b->layers, b->layer_tasks, b->state64, b->cand_cnt, b->cand_idx, b->cand_val64, b->cap, b->gidx,
                   b->gval64, acc, idx, reinterpret_cast<double*>(m + b->off_val), cnt, b->smem_keys,
                   (flags & LAGS_COMPRESS_EXACT) ? 1 : 0, mixed ? static_cast<float*>(r) : static_cast<float*>(nullptr),
                   static_cast<const int32_t*>(b->order));
  if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string("compress(f64) launch: ") + cudaGetErrorString(e));
  return cuda_check(mixed ? "lags_bucket_compress(f32/acc64)" : "lags_bucket_compress(f64)", 2);
}

}  // extern "C"

namespace {
// Cooperative launch of decode_fused_kernel<TV, TVal, ITEMS> (grid <= co-resident CTAs), with
// programmatic dependent launch when the driver takes both attributes.
template <typename TV, typename TVal, int ITEMS, bool MOM>
cudaError_t launch_fused_decode(lags_bucket_t* b, const MsgView& mv, int32_t P, int grid, void* v, void* momentum,
                                double mu, cudaStream_t s) {
  auto kern = decode_fused_kernel<TV, TVal, ITEMS, MOM>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(DEC_NT);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const DecTile* tiles = b->dtiles;
  const int ntiles = b->dec_tiles;
  TVal* planes = reinterpret_cast<TVal*>(b->planes);
  const int64_t n = b->n_total;
  uint32_t* mask = b->mask;
  TV* vv = static_cast<TV*>(v);
  TV* mm = static_cast<TV*>(momentum);
  uint32_t* touched = b->touched;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tiles, ntiles, mv, static_cast<int>(P), planes, n, mask, vv, mm, mu,
                                     touched);
  if (e != cudaSuccess) {  // without PDL
    cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tiles, ntiles, mv, static_cast<int>(P), planes, n, mask, vv, mm, mu, touched);
  }
  return e;
}

// Largest cooperative grid of decode_fused_kernel (co-resident CTAs on the device).
template <typename TV, typename TVal, bool MOM>
int fused_decode_grid() {
  static int grid = 0;
  if (grid == 0) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_fused_kernel<TV, TVal, 1, MOM>, DEC_NT, 0);
    int per8 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per8, decode_fused_kernel<TV, TVal, 8, MOM>, DEC_NT, 0);
    grid = std::max(1, std::min(per, per8)) * num_sms();
  }
  return grid;
}

template <typename TV, typename TVal, bool MOM>
cudaError_t fused_decode(lags_bucket_t* b, const MsgView& mv, int32_t P, void* v, void* momentum, double mu,
                         cudaStream_t s) {
  const int cap = fused_decode_grid<TV, TVal, MOM>();
  const int64_t nitems = static_cast<int64_t>(P) * b->dec_tiles;
  const int items = static_cast<int>((nitems + cap - 1) / cap);
  // momentum: the dense pass wants every co-resident CTA; otherwise one CTA per work item
  const int grid = MOM ? cap : static_cast<int>(std::min<int64_t>(nitems, cap));
  if (items <= 1) return launch_fused_decode<TV, TVal, 1, MOM>(b, mv, P, grid, v, momentum, mu, s);
  if (items <= 2) return launch_fused_decode<TV, TVal, 2, MOM>(b, mv, P, grid, v, momentum, mu, s);
  if (items <= 4) return launch_fused_decode<TV, TVal, 4, MOM>(b, mv, P, grid, v, momentum, mu, s);
  if (items <= 8) return launch_fused_decode<TV, TVal, 8, MOM>(b, mv, P, grid, v, momentum, mu, s);
  return cudaErrorNotSupported;  // more than 8 pairs per thread of a co-resident grid
}

template <typename TV, typename TVal>
int decode_impl(lags_bucket_t* b, const MsgView& mv, int32_t P, void* v, void* momentum, double mu, cudaStream_t s) {
  const int64_t n = b->n_total, S = b->total_k;
  const int gwork = stream_grid(S * P, 256, 8);
  TVal* planes = reinterpret_cast<TVal*>(b->planes);
  if (P > 1 || mu != 0.0) {  // one cooperative launch: scatter, grid barrier, update
    const cudaError_t e = mu != 0.0 ? fused_decode<TV, TVal, true>(b, mv, P, v, momentum, mu, s)
                                    : fused_decode<TV, TVal, false>(b, mv, P, v, momentum, mu, s);
    if (e == cudaSuccess) return cuda_check("decode(fused)", 1);
    if (e != cudaErrorNotSupported)
      return fail(LAGS_ERR_CUDA, std::string("fused decode launch: ") + cudaGetErrorString(e));
    // more than 8 pairs per thread of a co-resident grid: the two-kernel decode below
  }
  if (mu != 0.0) {
    decode_scatter_kernel<TVal><<<P * b->dec_tiles, DEC_NT, 0, s>>>(b->layers, b->tiles_dec, mv, P, planes, n, b->mask);
    decode_momentum_kernel<TV, TVal><<<stream_grid(n, 256, 8), 256, 0, s>>>(
        planes, n, b->mask, P, static_cast<TV*>(v), static_cast<TV*>(momentum), mu);
    return cuda_check("decode(momentum)", 2);
  }
  cudaError_t e;
  if (P == 1) {
    e = launch_pdl(decode_single_kernel<TV, TVal>, dim3(gwork), dim3(256), 0, s, b->layers, b->slot_layer, mv, S,
                   static_cast<TV*>(v));
    if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    return cuda_check("decode(single)", 1);
  }
  e = launch_pdl(decode_scatter_kernel<TVal>, dim3(P * b->dec_tiles), dim3(DEC_NT), 0, s, b->layers, b->tiles_dec, mv,
                 P, planes, n, b->mask);
  if (e == cudaSuccess)
    e = launch_pdl(decode_update_kernel<TV, TVal>, dim3(P * b->dec_tiles), dim3(DEC_NT), 0, s, b->layers,
                   b->tiles_dec, mv, P, static_cast<const TVal*>(planes), n, b->mask, static_cast<TV*>(v));
  if (e != cudaSuccess) return fail(LAGS_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  return cuda_check("decode", 2);
}
}  // namespace

extern "C" {

int lags_bucket_decode_update(lags_bucket_t* b, const void* msgs, int64_t msg_stride, int32_t P, void* v,
                              void* momentum, double mu, uint32_t flags, lags_stream_t stream) {
  if (!b || !msgs || !v) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_decode_update: null pointer");
  if (P < 1 || P > b->max_world)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_decode_update: P outside 1..max_world");
  if (P > 1 && msg_stride < b->msg_bytes)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_decode_update: msg_stride smaller than a message");
  if (mu != 0.0 && !momentum)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_decode_update: mu != 0 needs a momentum buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const MsgView mv{static_cast<const char*>(msgs), msg_stride, b->off_cnt, b->off_idx, b->off_val};
  if (flags & LAGS_DECODE_V64) {
    if (b->dtype == LAGS_F32) return decode_impl<double, float>(b, mv, P, v, momentum, mu, s);
    return decode_impl<double, double>(b, mv, P, v, momentum, mu, s);
  }
  if (b->dtype == LAGS_F32) return decode_impl<float, float>(b, mv, P, v, momentum, mu, s);
  if (b->dtype == LAGS_F64) return decode_impl<double, double>(b, mv, P, v, momentum, mu, s);
  return decode_impl<float, double>(b, mv, P, v, momentum, mu, s);
}

int lags_bucket_compress(lags_bucket_t* b, void* g, void* r, double alpha, void* msg, uint32_t* status,
                         uint32_t flags, lags_stream_t stream) {
  return compress_impl(b, g, r, alpha, msg, status, flags, nullptr, stream);
}

int lags_bucket_compress_push(lags_bucket_t* b, void* g, void* r, double alpha, void* msg, uint32_t* status,
                              uint32_t flags, const lags_peer_push_t* peer, lags_stream_t stream) {
  if (!b || !peer || !peer->bases || !peer->epoch || peer->P < 1 || peer->rank < 0 || peer->rank >= peer->P ||
      peer->ctas_per_peer < 1 || (peer->flags_bytes & 255) ||
      peer->flags_bytes < static_cast<uint64_t>(peer->P) * peer->ctas_per_peer * 4u)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_compress_push: bad peer description");
  if (b->dtype != LAGS_F32) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_compress_push: LAGS_F32 buckets only");
  return compress_impl(b, g, r, alpha, msg, status, flags, nullptr, stream, peer);
}

constexpr int64_t FUSE_P1_MAX_K = 49152;  // fused P = 1 update up to this many selected entries

int lags_bucket_step_local(lags_bucket_t* b, void* g, void* r, double alpha, void* v, void* msg, uint32_t* status,
                           uint32_t flags, lags_stream_t stream) {
  if (!v || !b) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_step_local: null pointer");
  // parity modes, and fp32 buckets selecting many entries: compress, then the ordinary P = 1
  // decode.  The fused update keeps a layer's scattered weight reads / writes on the CTAs that
  // select it: fewer launches for small selections (ResNet-50 at rho = 0.001: 69.8 vs 72.0 us),
  // but a few CTAs' memory pipes for large ones (rho = 0.01: 114.3 vs 110.5 us over all SMs).
  if (b->dtype != LAGS_F32 || b->total_k > FUSE_P1_MAX_K) {
    const int rc = lags_bucket_compress(b, g, r, alpha, msg, status, flags, stream);
    if (rc != LAGS_OK) return rc;
    return lags_bucket_decode_update(b, msg, b->msg_bytes, 1, v, nullptr, 0.0, 0, stream);
  }
  return compress_impl(b, g, r, alpha, msg, status, flags, v, stream);
}

int lags_bucket_set_probe_events(lags_bucket_t* b, void* before, void* after) {
  if (!b) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_set_probe_events: null bucket");
  b->probe_before = static_cast<cudaEvent_t>(before);
  b->probe_after = static_cast<cudaEvent_t>(after);
  return LAGS_OK;
}

int lags_bucket_set_grad_table(lags_bucket_t* b, const void* table) {
  if (!b) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_set_grad_table: null bucket");
  if (table && b->dtype != LAGS_F32)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_set_grad_table: LAGS_F32 buckets only");
  b->grad_table = static_cast<float* const*>(table);
  return LAGS_OK;
}

int lags_bucket_stats(const lags_bucket_t* b, uint32_t* out, lags_stream_t stream) {
  if (!b || !out) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_stats: null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (b->state64) {  // 64-bit-key buckets: {thr high word, fallbacks, last candidates, calls, 0, path, 0...}
    std::vector<State64> st(b->nlayers);
    if (cudaMemcpyAsync(st.data(), b->state64, sizeof(State64) * b->nlayers, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return cuda_check("lags_bucket_stats", 0);
    for (int j = 0; j < b->nlayers; ++j) {
      uint32_t* o = out + static_cast<size_t>(j) * LAGS_STATS_WORDS;
      std::fill(o, o + LAGS_STATS_WORDS, 0u);
      o[0] = static_cast<uint32_t>(st[j].thr >> 32);
      o[1] = st[j].fallbacks;
      o[2] = st[j].last_cands;
      o[3] = st[j].calls;
      o[5] = st[j].path;
    }
    return LAGS_OK;
  }
  if (cudaMemcpyAsync(out, b->state, sizeof(FastState) * b->nlayers, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return cuda_check("lags_bucket_stats", 0);
  return LAGS_OK;
}

int lags_bucket_reconstruct(const lags_bucket_t* b, const void* msgs, int64_t msg_stride, int32_t P, const void* r,
                            void* acc, int64_t plane_stride, lags_stream_t stream) {
  if (!b || !msgs || !r || !acc) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_reconstruct: null pointer");
  if (b->dtype == LAGS_F32_ACC64) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_reconstruct: LAGS_F32 or LAGS_F64 bucket");
  if (P < 1 || plane_stride < b->n_total || msg_stride < b->msg_bytes)
    return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_reconstruct: bad P or strides");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = b->dtype == LAGS_F64 ? 8 : 4;
  if (cudaMemcpy2DAsync(acc, es * plane_stride, r, es * plane_stride, es * b->n_total, P, cudaMemcpyDeviceToDevice,
                        s) != cudaSuccess)
    return cuda_check("lags_bucket_reconstruct copy", 0);
  const MsgView mv{static_cast<const char*>(msgs), msg_stride, b->off_cnt, b->off_idx, b->off_val};
  const int grid = stream_grid(b->total_k * P, 256, 8);
  if (b->dtype == LAGS_F64)
    reconstruct_kernel<double><<<grid, 256, 0, s>>>(b->layers, b->slot_layer, mv, b->total_k, P,
                                                    static_cast<double*>(acc), plane_stride);
  else
    reconstruct_kernel<float><<<grid, 256, 0, s>>>(b->layers, b->slot_layer, mv, b->total_k, P,
                                                   static_cast<float*>(acc), plane_stride);
  return cuda_check("reconstruct_kernel");
}

int lags_bucket_delta(const lags_bucket_t* b, const void* acc, const void* r, int64_t plane_stride, int32_t P,
                      double* out, lags_stream_t stream) {
  if (!b || !acc || !r || !out) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_delta: null pointer");
  if (b->dtype == LAGS_F32_ACC64) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_delta: LAGS_F32 or LAGS_F64 bucket");
  if (P < 1 || plane_stride < b->n_total) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_delta: bad P or stride");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = (b->ntasks + 7) / 8;
  if (b->dtype == LAGS_F64)
    delta_partial_kernel<double><<<blocks, 256, 0, s>>>(b->tasks, b->ntasks, static_cast<const double*>(acc),
                                                        static_cast<const double*>(r), plane_stride, P, b->delta_part);
  else
    delta_partial_kernel<float><<<blocks, 256, 0, s>>>(b->tasks, b->ntasks, static_cast<const float*>(acc),
                                                       static_cast<const float*>(r), plane_stride, P, b->delta_part);
  delta_final_kernel<<<(b->nlayers + 127) / 128, 128, 0, s>>>(b->layers, b->layer_tasks, b->nlayers, b->delta_part,
                                                              out);
  return cuda_check("delta kernels", 2);
}

int lags_bucket_shadow_step(const lags_bucket_t* b, const void* g_sum, double* x, double alpha, int32_t P,
                            lags_stream_t stream) {
  if (!b || !g_sum || !x) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_shadow_step: null pointer");
  if (P < 1) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_shadow_step: P must be >= 1");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = stream_grid(b->n_total, 256, 8);
  if (b->dtype == LAGS_F64)
    shadow_step_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(g_sum), x, alpha, P, b->n_total);
  else
    shadow_step_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(g_sum), x, alpha, P, b->n_total);
  return cuda_check("shadow_step_kernel");
}

int lags_bucket_identity(const lags_bucket_t* b, const void* v, const double* x, const void* r_sum, int32_t P,
                         double* out, lags_stream_t stream) {
  if (!b || !v || !x || !r_sum || !out) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_identity: null pointer");
  if (P < 1) return fail(LAGS_ERR_INVALID_ARG, "lags_bucket_identity: P must be >= 1");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = (b->ntasks + 7) / 8;
  if (b->dtype == LAGS_F64)
    identity_partial_kernel<double><<<blocks, 256, 0, s>>>(b->tasks, b->ntasks, static_cast<const double*>(v), x,
                                                           static_cast<const double*>(r_sum), P, b->delta_part);
  else
    identity_partial_kernel<float><<<blocks, 256, 0, s>>>(b->tasks, b->ntasks, static_cast<const float*>(v), x,
                                                          static_cast<const float*>(r_sum), P, b->delta_part);
  identity_final_kernel<<<1, 256, 0, s>>>(b->layer_tasks, b->nlayers, b->delta_part, out);
  return cuda_check("identity kernels", 2);
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
  if (dtype != LAGS_F32 && dtype != LAGS_F64)
    return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: dtype must be F32 or F64");
  if (!x || !idx_out || !val_out || !count_out || !workspace)
    return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: null pointer");
  if (dim <= 0) return fail(LAGS_ERR_INVALID_ARG, "input must be a non-empty 1-D array");
  if (k < 1 || k > dim)
    return fail(LAGS_ERR_K_OUT_OF_RANGE, "k=" + std::to_string(k) + " outside 1.." + std::to_string(dim));
  if (dim > 0x7fffffffLL) return fail(LAGS_ERR_INVALID_ARG, "lags_top_k: dim exceeds the int32 index range");
  if (workspace_bytes < lags_top_k_workspace_bytes(dtype, dim))
    return fail(LAGS_ERR_WORKSPACE, "lags_top_k: workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == LAGS_F64 ? 8 : 4;
  void* copy = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 256));
  if (cudaMemcpyAsync(copy, x, static_cast<size_t>(dim) * es, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return cuda_check("lags_top_k copy", 0);
  const lags_layer_t one{0, dim, k, 0};
  if (dtype == LAGS_F32)
    select_dense_kernel<float><<<1, SEL_NT, 0, s>>>(nullptr, one, static_cast<float*>(copy), idx_out,
                                                    static_cast<float*>(val_out), count_out, 0);
  else
    select_dense_kernel<double><<<1, SEL_NT, 0, s>>>(nullptr, one, static_cast<double*>(copy), idx_out,
                                                     static_cast<double*>(val_out), count_out, 0);
  return cuda_check("select_dense_kernel(top_k)");
}

int lags_decompress(int32_t dtype, const int32_t* idx, const void* val, const int32_t* count, int64_t dim, void* out,
                    lags_stream_t stream) {
  if (dtype != LAGS_F32 && dtype != LAGS_F64)
    return fail(LAGS_ERR_INVALID_ARG, "lags_decompress: dtype must be F32 or F64");
  if (!idx || !val || !count || !out || dim <= 0) return fail(LAGS_ERR_INVALID_ARG, "lags_decompress: bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == LAGS_F64 ? 8 : 4;
  if (cudaMemsetAsync(out, 0, static_cast<size_t>(dim) * es, s) != cudaSuccess)
    return cuda_check("lags_decompress memset", 0);
  if (dtype == LAGS_F32)
    decompress_kernel<float><<<64, 256, 0, s>>>(idx, static_cast<const float*>(val), count, static_cast<float*>(out));
  else
    decompress_kernel<double><<<64, 256, 0, s>>>(idx, static_cast<const double*>(val), count,
                                                 static_cast<double*>(out));
  return cuda_check("decompress_kernel");
}

}  // extern "C"

#ifdef LAGS_DBG_STAMPS
// Diagnostic builds only: the phase stamps of the first cluster layer ([rank][clock|globaltimer][16]).
extern "C" int lags_dbg_stamps_read(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, lags::lags_dbg_stamps, sizeof(lags::lags_dbg_stamps)));
}
extern "C" int lags_dbg_s64_read(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, lags::lags_dbg_s64, sizeof(lags::lags_dbg_s64)));
}
extern "C" int lags_dbg_sp_read(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, lags::lags_dbg_sp, sizeof(lags::lags_dbg_sp)));
}
extern "C" int lags_dbg_cstamps_read(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, lags::lags_dbg_cstamps, sizeof(lags::lags_dbg_cstamps)));
}
#endif
