// fp64 fast path (LAGS_F64, the reference's default LayeredVector dtype, R: layered.py:88-90):
// the same two-launch structure as the fp32 path on 64-bit keys.
//
// accum_emit64_kernel (K1): one warp per task streams g and r once (acc = r + alpha * g in fp64,
//    R: training.py:250), writes acc back into r, ORs the non-finite flag (R: training.py:174),
//    and appends every entry with key(acc) >= the layer's predicted threshold to the task's
//    candidate list in ascending index order (warp ballot, no atomics).  Algorithmic traffic:
//    24 B/element (+8 with the fused zero_grad).
//    LAGS_F32_ACC64 (fp32 storage, numpy-float64 alpha, R: training.py:250 under NEP 50) runs the
//    same kernel on float g / r: acc in fp64 into the bucket's acc64 (the selection's dense
//    fallback reads it) and fl32(acc) back into r -- 20 B/element.
// select64_kernel: one CTA per layer, the longest first.  When the candidate set provably holds
//    the top-k (no task overflow, count >= k): gather into shared memory (warp per task), radix
//    select on the 64-bit keys starting below the candidates' common prefix, ordered compaction
//    (ascending indices, residual acc - acc at the selected entries; fp32 for LAGS_F32_ACC64),
//    and the next threshold from the same passes.  Otherwise (first call, failed prediction,
//    forced exact, layers of <= TINY_LAYER entries) the dense exact path over acc, which also
//    yields the prediction.  Both return exactly the reference's selection (R: sparsify.py:84-90).
#pragma once
#include "lags_fast.cuh"

namespace lags {

struct State64 {
  unsigned long long thr;  // candidate threshold key (0 = no prediction: dense exact path)
  uint32_t pf256;          // adaptive prediction rank factor x256 (0 = PRED_FACTOR)
  uint32_t fallbacks;      // dense-path executions after a prediction existed (diagnostic)
  uint32_t calls;
  uint32_t last_cands;     // candidates at the last call (0 = dense path)
  uint32_t path;           // 0 small layer (always dense), 1 candidates, 2 dense (first call / fallback)
  uint32_t pad;
};

#ifndef LAGS_K1_64_UNROLL
#define LAGS_K1_64_UNROLL 4
#endif
constexpr int K1_64_UNROLL = LAGS_K1_64_UNROLL;  // doubles in flight per lane per operand

// TS: the storage type of g and r (double; float for LAGS_F32_ACC64, which also writes the fp64 acc
// into acc64).
template <bool ZERO_G, typename TS>
__global__ void __launch_bounds__(K1_WARPS * 32) accum_emit64_kernel(
    const Task* __restrict__ tasks, int ntasks, const lags_layer_t* __restrict__ layers,
    const State64* __restrict__ state, TS* __restrict__ g, TS* __restrict__ r, double* __restrict__ acc64,
    double alpha, int cap, int32_t* __restrict__ cand_idx, double* __restrict__ cand_val,
    int32_t* __restrict__ cand_cnt, uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * K1_WARPS + (threadIdx.x >> 5);
  griddep_wait();  // the previous kernel on the stream has completed
  griddep_launch_dependents();
  if (wid >= ntasks) return;
  const Task T = tasks[wid];
  const int64_t local0 = T.start - layers[T.layer].offset;
  const unsigned long long thr0 = state[T.layer].thr;
  const unsigned long long thr = thr0 ? thr0 : ~0ull;
  TS* gt = g + T.start;
  TS* rt = r + T.start;
  int32_t* cidx = cand_idx + static_cast<int64_t>(wid) * cap;
  double* cval = cand_val + static_cast<int64_t>(wid) * cap;
  const uint32_t below = (1u << lane) - 1u;
  uint32_t cnt = 0;
  bool bad = false;
  const int n = T.len;
  for (int q0 = 0; q0 < n; q0 += 32 * K1_64_UNROLL) {
    TS gv[K1_64_UNROLL], rv[K1_64_UNROLL];
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
        if (ZERO_G) __stcs(gt + i, TS(0));
        bad |= nonfinite(gv[u]);
        a = accum(static_cast<double>(rv[u]), static_cast<double>(gv[u]), alpha);
        __stcs(rt + i, static_cast<TS>(a));
        if (sizeof(TS) == 4) __stcs(acc64 + T.start + i, a);
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

// Ordered compaction of candidates staged in sv (doubles) / si (indices, 16-byte aligned; both
// in index order, readable 3 entries past m): 4 entries per thread per block scan, read as
// 16-byte vectors.  The rule is ordered_compact's: (key & pmask) > prefix, plus the first need_eq
// equal ones in index order.  The (index, value) pairs leave through shared memory as coalesced
// runs into oidx / oval; emit(ix, x) does the scattered residual write.  Returns the selected
// count (all threads).
template <typename Emit>
__device__ uint32_t compact64_staged(uint32_t m, const SelectThreshold<unsigned long long>& th, const double* sv,
                                     const int32_t* si, Emit emit, RadixSmem<Key<double>::RB>& sm, int32_t* oidx,
                                     double* oval) {
  constexpr int V = 4;
  static_assert(3 * SEL_NT * V <= RadixSmem<Key<double>::RB>::NB, "a chunk's output fits the staging arrays");
  int32_t* st_idx = reinterpret_cast<int32_t*>(sm.hist);  // free here: the threshold is known
  double* st_val = reinterpret_cast<double*>(sm.hist + SEL_NT * V);
  uint32_t carry_gt = 0, carry_eq = 0;
  for (uint32_t base = 0; base < m; base += SEL_NT * V) {
    const uint32_t out0 = carry_gt + min(carry_eq, th.need_eq);  // the chunk's first output slot
    const uint32_t i0 = base + threadIdx.x * V;
    double xs[V];
#pragma unroll
    for (int q = 0; q < V / 2; ++q) {
      double2 x2 = make_double2(0.0, 0.0);
      if (i0 + 2 * q < m) x2 = *reinterpret_cast<const double2*>(sv + i0 + 2 * q);
      xs[2 * q] = x2.x;
      xs[2 * q + 1] = x2.y;
    }
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const unsigned long long key = i0 + v < m ? Key<double>::of(xs[v]) : 0ull;
      const unsigned long long hk = key & th.pmask;
      if (key != 0ull) {
        if (hk > th.prefix) gtm |= 1u << v;
        else if (hk == th.prefix) eqm |= 1u << v;
      }
    }
    int4 ix4 = make_int4(0, 0, 0, 0);
    if (gtm | eqm) ix4 = *reinterpret_cast<const int4*>(si + i0);
    const int32_t ixs[V] = {ix4.x, ix4.y, ix4.z, ix4.w};
    const uint32_t packed = (static_cast<uint32_t>(__popc(eqm)) << 16) | static_cast<uint32_t>(__popc(gtm));
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<SEL_NT>(packed, sm.warp_tot, &tot);
    uint32_t gt_before = carry_gt + (ex & 0xffffu);
    uint32_t eq_before = carry_eq + (ex >> 16);
    if (gtm | eqm) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool g = (gtm >> v) & 1u, e = (eqm >> v) & 1u;
        if (g || (e && eq_before < th.need_eq)) {
          const uint32_t q = gt_before + min(eq_before, th.need_eq) - out0;
          st_idx[q] = ixs[v];
          st_val[q] = xs[v];
          emit(ixs[v], xs[v]);
        }
        gt_before += g;
        eq_before += e;
      }
    }
    carry_gt += tot & 0xffffu;
    carry_eq += tot >> 16;
    __syncthreads();  // the staged pairs are complete (and warp_tot is free for the next scan)
    const uint32_t n_out = carry_gt + min(carry_eq, th.need_eq) - out0;
    for (uint32_t q = threadIdx.x; q < n_out; q += SEL_NT) {
      oidx[out0 + q] = st_idx[q];
      oval[out0 + q] = st_val[q];
    }
  }
  __syncthreads();  // the staging arrays are read before any reuse
  return carry_gt + min(carry_eq, th.need_eq);
}

#ifdef LAGS_DBG_STAMPS
// Diagnostic builds only: per layer (j < 1024) clock64 after the wait / counts / gather / radix /
// compaction / end, and %globaltimer at the wait and the end.
__device__ unsigned long long lags_dbg_s64[1024][8];
#define LAGS_S64(i, v)                                            \
  do {                                                            \
    if (j < 1024 && threadIdx.x == 0) lags_dbg_s64[j][i] = (v);   \
  } while (0)
#else
#define LAGS_S64(i, v) \
  do {                 \
  } while (0)
#endif

__global__ void __launch_bounds__(SEL_NT) select64_kernel(const lags_layer_t* __restrict__ layers,
                                                          const int2* __restrict__ layer_tasks, State64* state,
                                                          const int32_t* __restrict__ cand_cnt,
                                                          const int32_t* __restrict__ cand_idx,
                                                          const double* __restrict__ cand_val, int cap, int32_t* gidx,
                                                          double* gval, double* r, int32_t* idx_out, double* val_out,
                                                          int32_t* count_out, int smem_words, int force_exact,
                                                          float* r32, const int32_t* __restrict__ order) {
  using K = unsigned long long;
  constexpr int RB = Key<double>::RB;
  extern __shared__ __align__(16) uint32_t dyn[];
  __shared__ RadixSmem<RB> sm;
  __shared__ uint32_t tpos[SEL_NT], tcnt[SEL_NT];
  griddep_wait();  // K1 has completed and its writes are visible
  const int j = order[blockIdx.x];  // the longest layers first: they must not wait for a second wave
  LAGS_S64(0, clock64());
  LAGS_S64(6, globaltimer_lo());
  const lags_layer_t L = layers[j];
  const int2 tr = layer_tasks[j];
  const State64 st = state[j];
  const uint32_t k = static_cast<uint32_t>(L.k);
  double* data = r + L.offset;
  int32_t* oidx = idx_out + L.slot;
  double* oval = val_out + L.slot;
  const float pf = st.pf256 ? st.pf256 / 256.0f : static_cast<float>(PRED_FACTOR);
  constexpr int NW = SEL_NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // speculative: entry `lane` of the warp's first GATHER_TASKS tasks, in flight with the counts
  // (reading past a short list stays inside its cap slots)
  double pre_v[GATHER_TASKS];
  int32_t pre_i[GATHER_TASKS];
  const bool spec = st.thr != 0ull && L.dim > TINY_LAYER && !force_exact;
#pragma unroll
  for (int u = 0; u < GATHER_TASKS; ++u) {
    const int tt = warp + u * NW;
    if (spec && tt < min(SEL_NT, tr.y - tr.x)) {
      const int64_t src = static_cast<int64_t>(tr.x + tt) * cap + lane;
      pre_v[u] = __ldcg(cand_val + src);
      pre_i[u] = __ldcg(cand_idx + src);
    }
  }
  uint32_t local = 0, over = 0, c_first = 0;  // c_first: this thread's task count in the first chunk
  for (int t = tr.x + threadIdx.x; t < tr.y; t += SEL_NT) {
    const uint32_t c = static_cast<uint32_t>(__ldcg(cand_cnt + t));
    over |= c > static_cast<uint32_t>(cap) ? 1u : 0u;
    local += min(c, static_cast<uint32_t>(cap));
    if (t == tr.x + static_cast<int>(threadIdx.x)) c_first = min(c, static_cast<uint32_t>(cap));
  }
  const uint32_t m = block_sum(local, sm);
  LAGS_S64(1, clock64());
  const bool overflow = __syncthreads_or(over) != 0;
  // layers of <= TINY_LAYER entries always take the dense path (no prediction: K1 emits nothing);
  // a k = 1 prediction over a few hundred entries missed every other step
  const bool tiny = L.dim <= TINY_LAYER;
  const bool cand = !tiny && !force_exact && st.thr != 0ull && !overflow && !(m < k && st.thr > 1ull);
  State64 ns = st;
  ns.calls += 1;
  uint32_t cnt = 0;
  if (cand) {
    const uint32_t k2 = max(k + 1u, static_cast<uint32_t>(fminf(pf * static_cast<float>(k), 4.0e9f)));
    K key2 = st.thr;
    if (m > 0) {
      // staging: doubles, then the indices at a 16-byte boundary (+4 words of vector over-read)
      const uint32_t si_off = (2u * m + 3u) & ~3u;
      const bool in_smem = static_cast<uint64_t>(si_off) + m + 4ull <= static_cast<uint64_t>(smem_words);
      const int64_t gbase = static_cast<int64_t>(tr.x) * cap;
      double* sv = in_smem ? reinterpret_cast<double*>(dyn) : gval + gbase;
      int32_t* si = in_smem ? reinterpret_cast<int32_t*>(dyn) + si_off : gidx + gbase;
      // gather: positions by a block scan over the task counts; one warp per task, lane = entry
      // (a task holds ~17 candidates of a 2.4 M-element layer at the margin), GATHER_TASKS tasks'
      // loads in flight per warp, entries past the first 32 in a loop; index order kept
      uint32_t carry = 0;
      for (int t0 = tr.x; t0 < tr.y; t0 += SEL_NT) {
        const int nt = min(SEL_NT, tr.y - t0);
        const uint32_t c = threadIdx.x >= nt ? 0u
                           : t0 == tr.x  ? c_first
                                         : min(static_cast<uint32_t>(__ldcg(cand_cnt + t0 + threadIdx.x)),
                                               static_cast<uint32_t>(cap));
        uint32_t tot;
        tpos[threadIdx.x] = carry + block_exclusive_scan<SEL_NT>(c, sm.warp_tot, &tot);
        tcnt[threadIdx.x] = c;
        __syncthreads();
        for (int tb = warp; tb < nt; tb += NW * GATHER_TASKS) {
          uint32_t cc[GATHER_TASKS], pp[GATHER_TASKS];
          double xv[GATHER_TASKS];
          int32_t xi[GATHER_TASKS];
          const bool first = t0 == tr.x && tb == warp;  // the speculative loads
#pragma unroll
          for (int u = 0; u < GATHER_TASKS; ++u) {
            const int tt = tb + u * NW;
            cc[u] = tt < nt ? tcnt[tt] : 0u;
            pp[u] = tt < nt ? tpos[tt] : 0u;
            if (static_cast<uint32_t>(lane) < cc[u]) {
              if (first) {
                xv[u] = pre_v[u];
                xi[u] = pre_i[u];
              } else {
                const int64_t src = static_cast<int64_t>(t0 + tt) * cap + lane;
                xv[u] = __ldcg(cand_val + src);
                xi[u] = __ldcg(cand_idx + src);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < GATHER_TASKS; ++u)
            if (static_cast<uint32_t>(lane) < cc[u]) {
              sv[pp[u] + lane] = xv[u];
              si[pp[u] + lane] = xi[u];
            }
#pragma unroll 1
          for (int u = 0; u < GATHER_TASKS; ++u) {  // lists longer than a warp
            const int64_t row = static_cast<int64_t>(t0 + tb + u * NW) * cap;
            for (uint32_t e = 32u + lane; e < cc[u]; e += 32u) {
              sv[pp[u] + e] = __ldcg(cand_val + row + e);
              si[pp[u] + e] = __ldcg(cand_idx + row + e);
            }
          }
        }
        carry += tot;
        __syncthreads();  // tpos / tcnt reuse; the staged candidates are visible
      }
      LAGS_S64(2, clock64());
      auto key_at = [=](int64_t i) { return Key<double>::of(sv[i]); };
      const SelectThreshold<K> th = radix_select<K, Key<double>::BITS, RB>(key_at, m, k, sm, min(k2, m), &key2, true);
      LAGS_S64(3, clock64());
      auto emit = [=](int32_t ix, double x) {
        if (r32) r32[L.offset + ix] = static_cast<float>(sent_residual(x));  // fl32(acc - acc)
        else data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
      };
      cnt = compact64_staged(m, th, sv, si, emit, sm, oidx, oval);
      LAGS_S64(4, clock64());
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
    if (r32) {  // the fp32 residual of the selected entries (the compaction's writes are visible)
      __syncthreads();
      for (uint32_t q = threadIdx.x; q < cnt; q += SEL_NT)
        r32[L.offset + oidx[q]] = static_cast<float>(sent_residual(oval[q]));
    }
    ns.thr = tiny ? 0ull : max(key2, 1ull);
    ns.fallbacks += predicted ? 1u : 0u;
    ns.last_cands = 0;
    ns.pf256 = pf_encode(pf_next);
    ns.path = tiny ? 0u : 2u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    count_out[j] = static_cast<int32_t>(cnt);
    state[j] = ns;
    LAGS_S64(5, clock64());
    LAGS_S64(7, globaltimer_lo());
  }
}

}  // namespace lags
