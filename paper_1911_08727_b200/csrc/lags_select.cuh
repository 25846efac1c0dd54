// Exact top-k selection machinery (one CTA): radix select on magnitude keys + ordered compaction.
//
// Replaces R: sparsify.py:84-90 (|x|, stable argsort, drop zeros, sort indices) and the residual
// rule of R: training.py:252 (selected residual entries become +0.0).  The k largest keys win,
// ties go to the lower index (= earlier position in the scanned order), key == 0 is never
// selected.  Output indices come out ascending because the compaction is an ordered block scan.
#pragma once
#include "lags_common.cuh"

namespace lags {

#ifndef LAGS_SEL_NT
#define LAGS_SEL_NT 512
#endif
#ifndef LAGS_SEL_MINB
#define LAGS_SEL_MINB 1
#endif
constexpr int SEL_NT = LAGS_SEL_NT;      // threads per selection CTA (512 measured faster than 1024)
constexpr int SEL_MINB = LAGS_SEL_MINB;  // selection CTAs resident per SM (launch bounds)
#ifndef LAGS_SEL_VEC
#define LAGS_SEL_VEC 4
#endif
#ifndef LAGS_UPDATE_B
#define LAGS_UPDATE_B 4
#endif
constexpr int SEL_VEC = LAGS_SEL_VEC;        // consecutive elements per thread per compaction chunk
constexpr int UPDATE_B = LAGS_UPDATE_B;      // weight loads in flight per thread in the P = 1 update

// Select (key & pmask) > prefix, plus the first `need_eq` (in scan order) with
// (key & pmask) == prefix.  `full_key` is the resolved threshold (valid when pmask is full).
template <typename K>
struct SelectThreshold {
  K prefix;
  K pmask;
  uint32_t n_gt;
  uint32_t need_eq;
};

template <int RB>
struct RadixSmem {
  static constexpr int NB = 1 << RB;
  alignas(16) uint32_t hist[NB];
  uint32_t warp_tot[33];
  uint32_t above, bin_count;
  int found;
  uint32_t found2[2], above2[2], count2[2];  // find_bin2
  uint32_t list_n, list_key, list_gt;         // bin-list finish of radix_select_dual
  uint32_t diff_acc;                          // key ^ key0 OR-accumulated by the candidate gathers
  uint32_t gtb;                               // candidates above the histogram cut (gathers)
  uint32_t dbg;                               // -DLAGS_DBG_SELECT: radix_select_dual's shape
};

// Thread t's PER contiguous bins in descending order, h[q] = H[NB - 1 - t * PER - q], read as
// 16-byte vectors (H 16-byte aligned): a scalar read at a stride of PER words was a PER-way bank
// conflict per load.
template <int NB, int PER>
__device__ __forceinline__ void load_bins_desc(const uint32_t* H, int t, uint32_t (&h)[PER]) {
  static_assert(PER % 4 == 0, "whole 16-byte vectors per thread");
  const uint4* v = reinterpret_cast<const uint4*>(H + NB - PER * (t + 1));
#pragma unroll
  for (int c = 0; c < PER / 4; ++c) {
    const uint4 x = v[c];
    h[PER - 1 - 4 * c] = x.x;
    h[PER - 2 - 4 * c] = x.y;
    h[PER - 3 - 4 * c] = x.z;
    h[PER - 4 - 4 * c] = x.w;
  }
}

// Bin holding the rank-th largest (1-based) of the histogram (descending scan).  All threads.
// `hist` (shared, NB bins, 16-byte aligned) defaults to sm.hist.
template <int RB>
__device__ LAGS_FINDBIN_ATTR void find_bin(RadixSmem<RB>& sm, uint32_t rank, uint32_t* bin, uint32_t* above,
                                         uint32_t* in_bin, const uint32_t* hist = nullptr) {
  constexpr int NB = RadixSmem<RB>::NB;
  constexpr int PER = NB / SEL_NT;  // 8 (fp32) or 16 (fp64) bins per thread at 512 threads
  const uint32_t* H = hist ? hist : sm.hist;
  const int t = threadIdx.x;
  uint32_t h[PER];
  load_bins_desc<NB, PER>(H, t, h);
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) s += h[q];
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<SEL_NT>(s, sm.warp_tot, &tot);
  if (ex < rank && rank <= ex + s) {
    uint32_t c = ex;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (rank <= c + h[q]) {
        sm.bin_count = h[q];
        sm.above = c;
        sm.found = NB - 1 - t * PER - q;
        break;
      }
      c += h[q];
    }
  }
  __syncthreads();
  *bin = static_cast<uint32_t>(sm.found);
  *above = sm.above;
  *in_bin = sm.bin_count;
  __syncthreads();
}

// Both ranks' bins in one scan of the histogram (the first pass of a dual select, where both
// ranks share the prefix).  bin/above/in_bin are arrays of 2.  All threads.
template <int RB>
__device__ LAGS_FINDBIN_ATTR void find_bin2(RadixSmem<RB>& sm, const uint32_t* H, uint32_t r0, uint32_t r1,
                                          uint32_t* bin, uint32_t* above, uint32_t* in_bin) {
  constexpr int NB = RadixSmem<RB>::NB;
  constexpr int PER = NB / SEL_NT;
  const int t = threadIdx.x;
  uint32_t h[PER];
  load_bins_desc<NB, PER>(H, t, h);
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) s += h[q];
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<SEL_NT>(s, sm.warp_tot, &tot);
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const uint32_t r = w ? r1 : r0;
    if (ex < r && r <= ex + s) {
      uint32_t c = ex;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        if (r <= c + h[q]) {
          sm.count2[w] = h[q];
          sm.above2[w] = c;
          sm.found2[w] = static_cast<uint32_t>(NB - 1 - t * PER - q);
          break;
        }
        c += h[q];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    bin[w] = sm.found2[w];
    above[w] = sm.above2[w];
    in_bin[w] = sm.count2[w];
  }
  __syncthreads();
}

// Multi-pass radix select over m keys produced by key_at(i).  Returns the threshold of the
// k largest.  If pred_rank > 0, *pred_key receives the lower edge of the first-digit bin that
// holds the pred_rank-th largest key (used to predict next call's candidate threshold).
// Block-wide OR of one key per thread (all threads get the result).  Uses sm.warp_tot.
template <typename K, int RB>
__device__ LAGS_OR_ATTR K block_or(K v, RadixSmem<RB>& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(v));
  uint32_t hi = sizeof(K) > 4 ? __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(static_cast<uint64_t>(v) >> 32)) : 0u;
  __syncthreads();
  if (lane == 0) {
    sm.warp_tot[warp] = lo;
  }
  __syncthreads();
  lo = 0;
  for (int w = 0; w < SEL_NT / 32; ++w) lo |= sm.warp_tot[w];
  __syncthreads();
  if (sizeof(K) > 4) {
    if (lane == 0) sm.warp_tot[warp] = hi;
    __syncthreads();
    hi = 0;
    for (int w = 0; w < SEL_NT / 32; ++w) hi |= sm.warp_tot[w];
    __syncthreads();
  }
  return static_cast<K>((static_cast<uint64_t>(hi) << 32) | lo);
}

// skip_common_prefix: first OR-reduce key ^ key(0) over all m keys and start the radix passes
// below the highest differing bit (cheap when keys live in shared memory and crowd together).
template <typename K, int BITS, int RB, typename KeyAt>
__device__ SelectThreshold<K> radix_select(KeyAt key_at, int64_t m, uint32_t k, RadixSmem<RB>& sm,
                                           uint32_t pred_rank = 0, K* pred_key = nullptr,
                                           bool skip_common_prefix = false) {
  constexpr int NB = RadixSmem<RB>::NB;
  constexpr K FULL = (K(1) << BITS) - 1;
  SelectThreshold<K> th;
  K prefix = 0, pmask = 0;
  uint32_t rank = k, n_gt = 0;
  int shift = BITS - RB, width = RB;
  bool first = true;
  if (static_cast<int64_t>(k) >= m && pred_rank == 0) {  // everything nonzero is selected
    th.prefix = 0;
    th.pmask = ~K(0);
    th.n_gt = 0;
    th.need_eq = 0;
    return th;
  }
  if (static_cast<int64_t>(rank) > m) rank = static_cast<uint32_t>(m);
  if (skip_common_prefix) {
    const K key0 = key_at(0);
    K diff = 0;
    for (int64_t i = threadIdx.x; i < m; i += SEL_NT) diff |= key_at(i) ^ key0;
    diff = block_or<K, RB>(diff, sm);
    if (diff == 0) {  // all keys equal
      pmask = FULL;
      prefix = key0;
      shift = 0;
      width = 0;
      if (pred_rank > 0 && pred_key) *pred_key = key0;
    } else {
      const int h = sizeof(K) > 4 ? 63 - __clzll(static_cast<long long>(diff)) : 31 - __clz(static_cast<int>(diff));
      const K low = (K(1) << (h + 1)) - 1;
      pmask = FULL & ~low;
      prefix = key0 & pmask;
      shift = h + 1 > RB ? h + 1 - RB : 0;
      width = h + 1 - shift;
    }
  }
  while (width > 0) {
    for (int b = threadIdx.x; b < NB; b += SEL_NT) sm.hist[b] = 0;
    __syncthreads();
    const K dmask = (K(1) << width) - 1;
    const int lane = threadIdx.x & 31;
    (void)lane;
    for (int64_t i = threadIdx.x; i < m; i += SEL_NT) {
      const K key = key_at(i);
      if ((key & pmask) == prefix) atomicAdd(&sm.hist[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    uint32_t b, above, in_bin;
    if (first && pred_rank > 0) {
      const uint32_t pr = static_cast<int64_t>(pred_rank) < m ? pred_rank : static_cast<uint32_t>(m);
      find_bin<RB>(sm, pr, &b, &above, &in_bin);
      *pred_key = prefix | (K(b) << shift);
    }
    first = false;
    find_bin<RB>(sm, rank, &b, &above, &in_bin);
    prefix |= K(b) << shift;
    pmask |= dmask << shift;
    n_gt += above;
    rank -= above;
    if (shift == 0) break;
    if (in_bin == rank && prefix != 0) break;  // the whole bin is taken: lower bits irrelevant
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
  if (static_cast<int64_t>(k) >= m) {  // pred-only call: select every nonzero
    th.prefix = 0;
    th.pmask = ~K(0);
    th.n_gt = 0;
    th.need_eq = 0;
  }
  return th;
}

// Ordered compaction of m entries (scan order = ascending index) under threshold th.
// load(i, &key, &val, &index) fetches entry i; emit(pos, i, index, val) writes selected entry i
// to output position pos.  Returns the selected count (all threads).
// carry_gt0 / carry_eq0: counts of gt / eq entries before entry 0 (multi-CTA compaction).
// Without a prefetch functor the emit is emit(pos, i, index, val).  ordered_compact_pf takes
// pf(i, index) -> W, called for every entry at or above the threshold BEFORE the block scan (so its
// loads are in flight across the scan's barriers), and calls emit(pos, i, index, val, w).
struct NoPrefetch {
  __device__ __forceinline__ float operator()(int64_t, int64_t) const { return 0.0f; }
};

template <typename K, typename T, typename Load, typename Emit, int RB, typename Pf = NoPrefetch>
__device__ uint32_t ordered_compact_pf(int64_t m, const SelectThreshold<K>& th, Load load, Emit emit,
                                       RadixSmem<RB>& sm, uint32_t carry_gt0, uint32_t carry_eq0, Pf pf) {
  uint32_t carry_gt = carry_gt0, carry_eq = carry_eq0;
  const int64_t chunk = static_cast<int64_t>(SEL_NT) * SEL_VEC;
  for (int64_t base = 0; base < m; base += chunk) {
    const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * SEL_VEC;
    T x[SEL_VEC];
    int64_t ix[SEL_VEC];
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int v = 0; v < SEL_VEC; ++v) {
      const int64_t i = i0 + v;
      K key = 0;
      x[v] = T(0);
      ix[v] = 0;
      if (i < m) load(i, &key, &x[v], &ix[v]);
      const K hi = key & th.pmask;
      if (key != 0) {
        if (hi > th.prefix) gtm |= 1u << v;
        else if (hi == th.prefix) eqm |= 1u << v;
      }
    }
    decltype(pf(0, 0)) w[SEL_VEC];
#pragma unroll
    for (int v = 0; v < SEL_VEC; ++v) w[v] = ((gtm | eqm) >> v) & 1u ? pf(i0 + v, ix[v]) : decltype(pf(0, 0))(0);
    const uint32_t packed = (static_cast<uint32_t>(__popc(eqm)) << 16) | static_cast<uint32_t>(__popc(gtm));
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<SEL_NT>(packed, sm.warp_tot, &tot);
    uint32_t gt_before = carry_gt + (ex & 0xffffu);
    uint32_t eq_before = carry_eq + (ex >> 16);
    if (gtm | eqm) {
#pragma unroll
      for (int v = 0; v < SEL_VEC; ++v) {
        const bool g = (gtm >> v) & 1u, e = (eqm >> v) & 1u;
        if (g || (e && eq_before < th.need_eq)) emit(gt_before + min(eq_before, th.need_eq), i0 + v, ix[v], x[v], w[v]);
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

template <typename K, typename T, typename Load, typename Emit, int RB>
__device__ uint32_t ordered_compact(int64_t m, const SelectThreshold<K>& th, Load load, Emit emit,
                                    RadixSmem<RB>& sm, uint32_t carry_gt0 = 0, uint32_t carry_eq0 = 0) {
  uint32_t carry_gt = carry_gt0, carry_eq = carry_eq0;
  const int64_t chunk = static_cast<int64_t>(SEL_NT) * SEL_VEC;
  for (int64_t base = 0; base < m; base += chunk) {
    const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * SEL_VEC;
    T x[SEL_VEC];
    int64_t ix[SEL_VEC];
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int v = 0; v < SEL_VEC; ++v) {
      const int64_t i = i0 + v;
      K key = 0;
      x[v] = T(0);
      ix[v] = 0;
      if (i < m) load(i, &key, &x[v], &ix[v]);
      const K hi = key & th.pmask;
      if (key != 0) {
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
        if (g || (e && eq_before < th.need_eq)) emit(gt_before + min(eq_before, th.need_eq), i0 + v, ix[v], x[v]);
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

// Exact top-k of dense data[0:d) (global memory) by one CTA: select + ordered compaction,
// optionally zeroing the selected entries in place.  Returns count; *pred receives the
// predicted candidate threshold for rank pred_rank (if pred_rank > 0).
template <typename T, typename TOut>
__device__ uint32_t exact_topk_dense(T* data, int64_t d, uint32_t k, int32_t* idx_out, TOut* val_out,
                                     bool zero_selected, RadixSmem<Key<T>::RB>& sm, uint32_t pred_rank = 0,
                                     typename Key<T>::K* pred = nullptr) {
  using K = typename Key<T>::K;
  auto key_at = [data](int64_t i) { return Key<T>::of(data[i]); };
  const auto th = radix_select<K, Key<T>::BITS, Key<T>::RB>(key_at, d, k, sm, pred_rank, pred);
  auto load = [data](int64_t i, K* key, T* x, int64_t* ix) {
    *x = data[i];
    *key = Key<T>::of(*x);
    *ix = i;
  };
  auto emit = [=](uint32_t pos, int64_t i, int64_t ix, T x) {
    idx_out[pos] = static_cast<int32_t>(ix);
    val_out[pos] = static_cast<TOut>(x);
    if (zero_selected) data[i] = sent_residual(x);  // acc - acc (R: training.py:252)
  };
  return ordered_compact<K, T>(d, th, load, emit, sm);
}

}  // namespace lags
