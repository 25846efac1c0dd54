// fp64 fast path (LAGS_F64, the reference's default LayeredVector dtype, R: layered.py:88-90):
// the same two-launch structure as the fp32 path on 64-bit keys.
//
// accum_emit64_kernel (K1): one warp per task streams g and r once (acc = r + alpha * g in fp64,
//    R: training.py:250), writes acc back into r, ORs the non-finite flag (R: training.py:174),
//    and appends every entry with key(acc) >= the layer's predicted threshold to the task's
//    candidate list in ascending index order (warp ballot, no atomics).  Algorithmic traffic:
//    24 B/element (+8 with the fused zero_grad).
// select64_kernel: one CTA per layer.  When the candidate set provably holds the top-k (no task
//    overflow, count >= k): gather into shared memory, radix select on the 64-bit keys starting
//    below the candidates' common prefix, ordered compaction (ascending indices, residual
//    acc - acc at the selected entries), and the next threshold from the same passes.  Otherwise
//    (first call, failed prediction, forced exact) the dense exact path over r, which also yields
//    the prediction.  Both return exactly the reference's selection (R: sparsify.py:84-90).
#pragma once
#include "lags_fast.cuh"

namespace lags {

struct State64 {
  unsigned long long thr;  // candidate threshold key (0 = no prediction: dense exact path)
  uint32_t pf256;          // adaptive prediction rank factor x256 (0 = PRED_FACTOR)
  uint32_t fallbacks;      // dense-path executions after a prediction existed (diagnostic)
  uint32_t calls;
  uint32_t last_cands;     // candidates at the last call (0 = dense path)
  uint32_t path;           // 0 dense, 1 candidates
  uint32_t pad;
};

#ifndef LAGS_K1_64_UNROLL
#define LAGS_K1_64_UNROLL 4
#endif
constexpr int K1_64_UNROLL = LAGS_K1_64_UNROLL;  // doubles in flight per lane per operand

template <bool ZERO_G>
__global__ void __launch_bounds__(K1_WARPS * 32) accum_emit64_kernel(
    const Task* __restrict__ tasks, int ntasks, const lags_layer_t* __restrict__ layers,
    const State64* __restrict__ state, double* __restrict__ g, double* __restrict__ r, double alpha, int cap,
    int32_t* __restrict__ cand_idx, double* __restrict__ cand_val, int32_t* __restrict__ cand_cnt, uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * K1_WARPS + (threadIdx.x >> 5);
  griddep_wait();  // the previous kernel on the stream has completed
  griddep_launch_dependents();
  if (wid >= ntasks) return;
  const Task T = tasks[wid];
  const int64_t local0 = T.start - layers[T.layer].offset;
  const unsigned long long thr0 = state[T.layer].thr;
  const unsigned long long thr = thr0 ? thr0 : ~0ull;
  double* gt = g + T.start;
  double* rt = r + T.start;
  int32_t* cidx = cand_idx + static_cast<int64_t>(wid) * cap;
  double* cval = cand_val + static_cast<int64_t>(wid) * cap;
  const uint32_t below = (1u << lane) - 1u;
  uint32_t cnt = 0;
  bool bad = false;
  const int n = T.len;
  for (int q0 = 0; q0 < n; q0 += 32 * K1_64_UNROLL) {
    double gv[K1_64_UNROLL], rv[K1_64_UNROLL];
#pragma unroll
    for (int u = 0; u < K1_64_UNROLL; ++u) {
      const int i = q0 + u * 32 + lane;
      if (i < n) {
        gv[u] = __ldcs(gt + i);
        rv[u] = __ldcs(rt + i);
      }
    }
#pragma unroll
    for (int u = 0; u < K1_64_UNROLL; ++u) {
      const int i = q0 + u * 32 + lane;
      bool c = false;
      double a = 0.0;
      if (i < n) {
        if (ZERO_G) __stcs(gt + i, 0.0);
        bad |= nonfinite(gv[u]);
        a = accum(rv[u], gv[u], alpha);
        __stcs(rt + i, a);
        c = Key<double>::of(a) >= thr;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, c);
      if (bal) {  // lanes in index order: ascending within the task
        const uint32_t pos = cnt + __popc(bal & below);
        if (c && pos < static_cast<uint32_t>(cap)) {
          cidx[pos] = static_cast<int32_t>(local0 + i);
          cval[pos] = a;
        }
        cnt += __popc(bal);
      }
    }
  }
  if (lane == 0) cand_cnt[wid] = static_cast<int32_t>(cnt);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// Next threshold when fewer candidates than the prediction rank were seen: the threshold's
// magnitude scaled down (keys are monotone in |x|), at least 1.
__device__ __forceinline__ unsigned long long lower_threshold64(unsigned long long thr, uint32_t m, uint32_t k2) {
  const double x = __longlong_as_double(static_cast<long long>(thr));
  const double f = m == 0 ? 0.5 : fmax(0.5, fmin(0.95, static_cast<double>(m) / static_cast<double>(k2)));
  const unsigned long long next = Key<double>::of(x * f);
  return next >= thr ? (thr > 1ull ? thr - 1ull : 1ull) : (next ? next : 1ull);
}

__global__ void __launch_bounds__(SEL_NT) select64_kernel(const lags_layer_t* __restrict__ layers,
                                                          const int2* __restrict__ layer_tasks, State64* state,
                                                          const int32_t* __restrict__ cand_cnt,
                                                          const int32_t* __restrict__ cand_idx,
                                                          const double* __restrict__ cand_val, int cap, int32_t* gidx,
                                                          double* gval, double* r, int32_t* idx_out, double* val_out,
                                                          int32_t* count_out, int smem_words, int force_exact) {
  using K = unsigned long long;
  constexpr int RB = Key<double>::RB;
  extern __shared__ __align__(16) uint32_t dyn[];
  __shared__ RadixSmem<RB> sm;
  __shared__ uint32_t tpos[SEL_NT];
  griddep_wait();  // K1 has completed and its writes are visible
  const int j = blockIdx.x;
  const lags_layer_t L = layers[j];
  const int2 tr = layer_tasks[j];
  const State64 st = state[j];
  const uint32_t k = static_cast<uint32_t>(L.k);
  double* data = r + L.offset;
  int32_t* oidx = idx_out + L.slot;
  double* oval = val_out + L.slot;
  const float pf = st.pf256 ? st.pf256 / 256.0f : static_cast<float>(PRED_FACTOR);
  uint32_t local = 0, over = 0;
  for (int t = tr.x + threadIdx.x; t < tr.y; t += SEL_NT) {
    const uint32_t c = static_cast<uint32_t>(__ldcg(cand_cnt + t));
    over |= c > static_cast<uint32_t>(cap) ? 1u : 0u;
    local += min(c, static_cast<uint32_t>(cap));
  }
  const uint32_t m = block_sum(local, sm);
  const bool overflow = __syncthreads_or(over) != 0;
  const bool cand = !force_exact && st.thr != 0ull && !overflow && !(m < k && st.thr > 1ull);
  State64 ns = st;
  ns.calls += 1;
  uint32_t cnt = 0;
  if (cand) {
    const uint32_t k2 = max(k + 1u, static_cast<uint32_t>(fminf(pf * static_cast<float>(k), 4.0e9f)));
    K key2 = st.thr;
    if (m > 0) {
      const bool in_smem = 3ull * m + 2ull <= static_cast<uint64_t>(smem_words);
      const int64_t gbase = static_cast<int64_t>(tr.x) * cap;
      double* sv = in_smem ? reinterpret_cast<double*>(dyn) : gval + gbase;
      int32_t* si = in_smem ? reinterpret_cast<int32_t*>(dyn) + 2 * m : gidx + gbase;
      // gather: positions by a block scan over the task counts, one thread per entry (the owning
      // task by binary search), index order kept
      uint32_t carry = 0;
      for (int t0 = tr.x; t0 < tr.y; t0 += SEL_NT) {
        const int nt = min(SEL_NT, tr.y - t0);
        const uint32_t c = threadIdx.x < nt ? min(static_cast<uint32_t>(__ldcg(cand_cnt + t0 + threadIdx.x)),
                                                  static_cast<uint32_t>(cap))
                                            : 0u;
        uint32_t tot;
        tpos[threadIdx.x] = block_exclusive_scan<SEL_NT>(c, sm.warp_tot, &tot);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < tot; e += SEL_NT) {
          int lo = 0, hi = nt - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tpos[mid] <= e) lo = mid;
            else hi = mid - 1;
          }
          const int64_t src = static_cast<int64_t>(t0 + lo) * cap + (e - tpos[lo]);
          sv[carry + e] = __ldcg(cand_val + src);
          si[carry + e] = __ldcg(cand_idx + src);
        }
        carry += tot;
        __syncthreads();
      }
      auto key_at = [=](int64_t i) { return Key<double>::of(sv[i]); };
      const SelectThreshold<K> th = radix_select<K, Key<double>::BITS, RB>(key_at, m, k, sm, min(k2, m), &key2, true);
      auto load = [=](int64_t i, K* key, double* x, int64_t* ix) {
        *x = sv[i];
        *key = Key<double>::of(*x);
        *ix = si[i];
      };
      auto emit = [=](uint32_t pos, int64_t, int64_t ix, double x) {
        oidx[pos] = static_cast<int32_t>(ix);
        oval[pos] = x;
        data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
      };
      cnt = ordered_compact<K, double>(m, th, load, emit, sm);
    }
    ns.thr = m >= k2 ? max(key2, 1ull) : lower_threshold64(st.thr, m, k2);
    ns.last_cands = m;
    ns.path = 1u;
    if (m > 0) {  // steer the candidate count toward pred_target_count(k) (as the fp32 path)
      const float corrected = pf * pred_target_count(k) / static_cast<float>(m);
      ns.pf256 = pf_encode(sqrtf(pf * fmaxf(corrected, 0.25f)));
    }
  } else {
    // dense exact path over r (= acc): the k-th key and, in the same passes, the next prediction
    const bool predicted = st.thr != 0ull && !force_exact;
    const float pf_next = !predicted ? pf : (overflow ? 0.5f * pf : 2.0f * pf);
    const int64_t pk = static_cast<int64_t>(fmaxf(pf_next, 1.0f) * static_cast<float>(k));
    const uint32_t k2 = static_cast<uint32_t>(pk < L.dim ? (pk > k ? pk : k + 1) : L.dim);
    K key2 = 0ull;
    cnt = exact_topk_dense<double, double>(data, L.dim, k, oidx, oval, true, sm, k2, &key2);
    ns.thr = max(key2, 1ull);
    ns.fallbacks += predicted ? 1u : 0u;
    ns.last_cands = 0;
    ns.pf256 = pf_encode(pf_next);
    ns.path = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    count_out[j] = static_cast<int32_t>(cnt);
    state[j] = ns;
  }
}

}  // namespace lags
