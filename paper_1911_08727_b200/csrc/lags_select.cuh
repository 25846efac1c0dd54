// Exact per-layer top-k selection + ordered compaction, one CTA per layer.
//
// Replaces R: sparsify.py:84-90 (|x|, stable argsort, drop zeros, sort indices) and the residual
// rule of R: training.py:252 (selected residual entries become +0.0).  Selection works on the
// magnitude key (Key<T>): the k largest keys win, ties go to the lower index, key == 0 is never
// selected.  Output indices are produced in ascending order by an ordered block scan.
#pragma once
#include "lags_common.cuh"

namespace lags {

constexpr int SEL_NT = 1024;  // threads per selection CTA
constexpr int SEL_VEC = 4;    // consecutive elements per thread per compaction chunk

// Radix-select result for one layer: select key with (key & pmask) > prefix, plus the first
// `need_eq` (in index order) with (key & pmask) == prefix.
template <typename K>
struct SelectThreshold {
  K prefix;
  K pmask;
  uint32_t n_gt;
  uint32_t need_eq;
};

// Shared memory for one selection CTA.
template <typename T>
struct SelectSmem {
  static constexpr int NB = 1 << Key<T>::RB;
  uint32_t hist[NB];
  uint32_t warp_tot[33];
  typename Key<T>::K prefix, pmask;
  uint32_t n_gt, rank, bin_count;
  int found;
};

// Find the digit bin holding the rank-th largest (1-based) among the histogram; descending scan.
template <typename T>
__device__ __forceinline__ void find_bin(SelectSmem<T>& sm, uint32_t rank, uint32_t* bin, uint32_t* above,
                                         uint32_t* in_bin) {
  constexpr int NB = SelectSmem<T>::NB;
  constexpr int PER = NB / SEL_NT;  // bins per thread (2 for fp32, 8 for fp64)
  const int t = threadIdx.x;
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) s += sm.hist[NB - 1 - t * PER - q];
  uint32_t tot;
  uint32_t ex = block_exclusive_scan<SEL_NT>(s, sm.warp_tot, &tot);
  if (ex < rank && rank <= ex + s) {
    uint32_t c = ex;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = NB - 1 - t * PER - q;
      const uint32_t h = sm.hist[b];
      if (rank <= c + h) {
        sm.bin_count = h;
        sm.n_gt = c;  // temporarily: count strictly above bin b within the prefix
        sm.found = b;
        break;
      }
      c += h;
    }
  }
  __syncthreads();
  *bin = static_cast<uint32_t>(sm.found);
  *above = sm.n_gt;
  *in_bin = sm.bin_count;
  __syncthreads();
}

// Multi-pass radix select over data[0:d) (global memory).  All threads return the same result.
template <typename T>
__device__ SelectThreshold<typename Key<T>::K> radix_select(const T* data, int64_t d, uint32_t k,
                                                            SelectSmem<T>& sm) {
  using K = typename Key<T>::K;
  constexpr int BITS = Key<T>::BITS, RB = Key<T>::RB, NB = SelectSmem<T>::NB;
  SelectThreshold<K> th;
  if (static_cast<int64_t>(k) >= d) {  // everything nonzero is selected
    th.prefix = 0;
    th.pmask = ~K(0);
    th.n_gt = 0;
    th.need_eq = 0;
    return th;
  }
  K prefix = 0, pmask = 0;
  uint32_t rank = k, n_gt = 0;
  int shift = BITS - RB, width = RB;
  while (true) {
    for (int b = threadIdx.x; b < NB; b += SEL_NT) sm.hist[b] = 0;
    __syncthreads();
    const K dmask = (K(1) << width) - 1;
    for (int64_t i = threadIdx.x; i < d; i += SEL_NT) {
      const K key = Key<T>::of(data[i]);
      if ((key & pmask) == prefix) atomicAdd(&sm.hist[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    uint32_t b, above, in_bin;
    find_bin<T>(sm, rank, &b, &above, &in_bin);
    prefix |= K(b) << shift;
    pmask |= dmask << shift;
    n_gt += above;
    rank -= above;
    if (shift == 0) break;
    if (in_bin == rank && prefix != 0) break;  // the whole bin is taken: no need to resolve lower bits
    const int ns = shift > RB ? shift - RB : 0;
    width = shift - ns;
    shift = ns;
  }
  th.prefix = prefix;
  th.pmask = pmask;
  th.n_gt = n_gt;
  // prefix == 0 only survives to full resolution (the early exit requires prefix != 0); a zero
  // threshold means "every nonzero key": zeros are never selected (R: sparsify.py:88).
  th.need_eq = prefix == 0 ? 0u : rank;
  return th;
}

// Ordered compaction of data[0:d) under threshold `th`: writes ascending local indices and
// values of the selected entries into idx_out/val_out, optionally zeroes them in `data`
// (the residual rule), returns the count (all threads).
template <typename T>
__device__ uint32_t ordered_compact(T* data, int64_t d, const SelectThreshold<typename Key<T>::K>& th,
                                    int32_t* idx_out, T* val_out, bool zero_selected, SelectSmem<T>& sm) {
  using K = typename Key<T>::K;
  uint32_t carry_gt = 0, carry_eq = 0;
  const int64_t chunk = static_cast<int64_t>(SEL_NT) * SEL_VEC;
  for (int64_t base = 0; base < d; base += chunk) {
    const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * SEL_VEC;
    T x[SEL_VEC];
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int v = 0; v < SEL_VEC; ++v) {
      const int64_t i = i0 + v;
      x[v] = i < d ? data[i] : T(0);
      const K key = Key<T>::of(x[v]);
      const K hi = key & th.pmask;
      if (i < d && key != 0) {
        if (hi > th.prefix) gtm |= 1u << v;
        else if (hi == th.prefix) eqm |= 1u << v;
      }
    }
    const uint32_t packed = (static_cast<uint32_t>(__popc(eqm)) << 16) | static_cast<uint32_t>(__popc(gtm));
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<SEL_NT>(packed, sm.warp_tot, &tot);
    uint32_t gt_before = carry_gt + (ex & 0xffffu);
    uint32_t eq_before = carry_eq + (ex >> 16);
    if (gtm | eqm) {
#pragma unroll
      for (int v = 0; v < SEL_VEC; ++v) {
        const bool g = (gtm >> v) & 1u, e = (eqm >> v) & 1u;
        bool take = g || (e && eq_before < th.need_eq);
        if (take) {
          const uint32_t pos = gt_before + min(eq_before, th.need_eq);
          idx_out[pos] = static_cast<int32_t>(i0 + v);
          val_out[pos] = x[v];
          if (zero_selected) data[i0 + v] = T(0);  // acc - acc == +0.0 (R: training.py:252)
        }
        gt_before += g;
        eq_before += e;
      }
    }
    carry_gt += tot & 0xffffu;
    carry_eq += tot >> 16;
    __syncthreads();  // warp_tot reuse by the next scan
  }
  return carry_gt + min(carry_eq, th.need_eq);
}

}  // namespace lags
