// fp32 fast path: one streaming pass over g and r that also emits index-ordered candidates above
// a per-layer predicted threshold, then a per-layer exact select over the (few) candidates.
//
// K1 (accum_emit_kernel): one warp per task (a <= TASK_ELEMS slice of one layer).  Reads g and r
//    once (16-byte vectors), writes acc back into r, ORs the non-finite flag, and appends every
//    entry with key(acc) >= thr[layer] to the task's candidate list in ascending index order
//    (warp ballot + shuffle scan, no atomics).  Algorithmic traffic: 12 B/element.
// K2 (select_fast_kernel): one CTA per layer.  If the layer's candidate set provably contains the
//    top-k (count >= k, no task overflow) the exact top-k is taken over the candidates only
//    (radix select in shared memory + ordered compaction), selected residual entries are zeroed
//    by scatter, and the next threshold is predicted from the candidates.  Otherwise (first
//    call, misprediction, overflow, small layer) it runs the dense exact path over r.
// Both paths give bit-identical results: the candidate set contains every top-k element.
#pragma once
#include "lags_select.cuh"

namespace lags {

constexpr int TASK_ELEMS = 8192;   // elements per K1 task (one warp)
constexpr int SMALL_LAYER = 16384; // layers up to this size always take the dense exact path
constexpr int K1_WARPS = 8;        // warps per K1 CTA
constexpr int K1_UNROLL = 4;       // float4 loads in flight per lane per operand
constexpr int PRED_FACTOR = 2;     // predicted threshold targets PRED_FACTOR * k candidates

struct Task {
  int64_t start;  // flat element offset
  int32_t len;
  int32_t layer;
};

struct FastState {
  uint32_t thr;         // candidate threshold key (0 = no prediction: dense exact path)
  uint32_t fallbacks;   // dense-path executions after a prediction existed (diagnostic)
  uint32_t last_cands;  // candidates at the last call
  uint32_t calls;
};

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Append this lane's candidate bits (ascending element order within the lane, lanes in index
// order) to the task list.  Warp-collective.
__device__ __forceinline__ void emit_candidates(uint32_t bits, const float* vals, int64_t local0, int lane,
                                                uint32_t& cnt, int32_t* cidx, float* cval, int cap) {
  if (__ballot_sync(0xffffffffu, bits != 0) == 0u) return;
  const uint32_t c = __popc(bits);
  const uint32_t inc = warp_inclusive_scan(c, lane);
  uint32_t pos = cnt + inc - c;
  while (bits) {
    const int b = __ffs(bits) - 1;
    if (pos < static_cast<uint32_t>(cap)) {
      cidx[pos] = static_cast<int32_t>(local0 + b);
      cval[pos] = vals[b];
    }
    ++pos;
    bits &= bits - 1;
  }
  cnt += __shfl_sync(0xffffffffu, inc, 31);
}

__global__ void __launch_bounds__(K1_WARPS * 32) accum_emit_kernel(
    const Task* __restrict__ tasks, int ntasks, const lags_layer_t* __restrict__ layers,
    const FastState* __restrict__ state, const float* __restrict__ g, float* __restrict__ r, float alpha, int cap,
    int32_t* __restrict__ cand_idx, float* __restrict__ cand_val, int32_t* __restrict__ cand_cnt,
    uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * K1_WARPS + (threadIdx.x >> 5);
  if (wid >= ntasks) return;
  const Task T = tasks[wid];
  const int64_t loff = layers[T.layer].offset;
  const uint32_t thr0 = state[T.layer].thr;
  const uint32_t thr = thr0 ? thr0 : 0xffffffffu;
  int32_t* cidx = cand_idx + static_cast<int64_t>(wid) * cap;
  float* cval = cand_val + static_cast<int64_t>(wid) * cap;
  uint32_t cnt = 0;
  bool bad = false;
  const int64_t s = T.start, e = T.start + T.len;
  // scalar head up to 16-byte alignment (flat buffers are 16-byte aligned)
  const int64_t h = min(static_cast<int64_t>((4 - (s & 3)) & 3), static_cast<int64_t>(T.len));
  {
    uint32_t bits = 0;
    float a = 0.f;
    if (lane < h) {
      const float gi = g[s + lane];
      bad |= nonfinite(gi);
      a = accum(r[s + lane], gi, alpha);
      r[s + lane] = a;
      bits = (Key<float>::of(a) >= thr) ? 1u : 0u;
    }
    emit_candidates(bits, &a, s + lane - loff, lane, cnt, cidx, cval, cap);
  }
  const int64_t vb = s + h;
  const int64_t n4 = (e - vb) >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(g + vb);
  float4* r4 = reinterpret_cast<float4*>(r + vb);
  for (int64_t q0 = 0; q0 < n4; q0 += 32 * K1_UNROLL) {
    float4 gv[K1_UNROLL], rv[K1_UNROLL];
#pragma unroll
    for (int u = 0; u < K1_UNROLL; ++u) {
      const int64_t q = q0 + u * 32 + lane;
      if (q < n4) {
        gv[u] = __ldcs(g4 + q);
        rv[u] = r4[q];
      }
    }
#pragma unroll
    for (int u = 0; u < K1_UNROLL; ++u) {
      const int64_t q = q0 + u * 32 + lane;
      uint32_t bits = 0;
      float a[4] = {0.f, 0.f, 0.f, 0.f};
      if (q < n4) {
        bad |= nonfinite(gv[u].x) | nonfinite(gv[u].y) | nonfinite(gv[u].z) | nonfinite(gv[u].w);
        a[0] = accum(rv[u].x, gv[u].x, alpha);
        a[1] = accum(rv[u].y, gv[u].y, alpha);
        a[2] = accum(rv[u].z, gv[u].z, alpha);
        a[3] = accum(rv[u].w, gv[u].w, alpha);
        r4[q] = make_float4(a[0], a[1], a[2], a[3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) bits |= (Key<float>::of(a[c]) >= thr ? 1u : 0u) << c;
      }
      if (q0 + u * 32 < n4) emit_candidates(bits, a, vb + 4 * q - loff, lane, cnt, cidx, cval, cap);
    }
  }
  // scalar tail
  {
    const int64_t t0 = vb + 4 * n4;
    uint32_t bits = 0;
    float a = 0.f;
    if (t0 + lane < e) {
      const float gi = g[t0 + lane];
      bad |= nonfinite(gi);
      a = accum(r[t0 + lane], gi, alpha);
      r[t0 + lane] = a;
      bits = (Key<float>::of(a) >= thr) ? 1u : 0u;
    }
    if (t0 < e) emit_candidates(bits, &a, t0 + lane - loff, lane, cnt, cidx, cval, cap);
  }
  if (lane == 0) cand_cnt[wid] = static_cast<int32_t>(cnt);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// Reduce (sum, or) over the block; all threads get the result.  Uses sm.warp_tot.
template <int RB>
__device__ __forceinline__ uint32_t block_sum(uint32_t v, RadixSmem<RB>& sm) {
  uint32_t tot;
  block_exclusive_scan<SEL_NT>(v, sm.warp_tot, &tot);
  __syncthreads();
  return tot;
}

__global__ void __launch_bounds__(SEL_NT) select_fast_kernel(
    const lags_layer_t* __restrict__ layers, const int2* __restrict__ layer_tasks, FastState* state,
    const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_val,
    int cap, int32_t* gidx, float* gval, float* r, int32_t* __restrict__ idx_out, float* __restrict__ val_out,
    int32_t* __restrict__ count_out, int smem_keys, int force_exact) {
  extern __shared__ uint32_t skeys[];
  __shared__ RadixSmem<Key<float>::RB> sm;
  const int j = blockIdx.x;
  const lags_layer_t L = layers[j];
  const int2 tr = layer_tasks[j];
  const FastState st = state[j];
  const uint32_t k = static_cast<uint32_t>(L.k);
  float* data = r + L.offset;
  int32_t* oidx = idx_out + L.slot;
  float* oval = val_out + L.slot;
  const bool big = L.dim > SMALL_LAYER;
  bool exact = force_exact || !big || st.thr == 0;
  uint32_t m = 0;
  if (!exact) {
    uint32_t local = 0, over = 0;
    for (int t = tr.x + threadIdx.x; t < tr.y; t += SEL_NT) {
      const uint32_t c = static_cast<uint32_t>(cand_cnt[t]);
      over |= c > static_cast<uint32_t>(cap) ? 1u : 0u;
      local += min(c, static_cast<uint32_t>(cap));
    }
    m = block_sum(local, sm);
    over = block_sum(over, sm);
    if (over || (m < k && st.thr > 1u)) exact = true;
  }
  uint32_t cnt;
  if (exact) {
    uint32_t pred = 0;
    cnt = exact_topk_dense<float, float>(data, L.dim, k, oidx, oval, true, sm, big ? PRED_FACTOR * k : 0u, &pred);
    if (threadIdx.x == 0) {
      FastState ns = st;
      ns.thr = big ? max(pred, 1u) : 0u;
      ns.fallbacks += (st.thr != 0 && !force_exact) ? 1u : 0u;
      ns.last_cands = 0;
      ns.calls += 1;
      state[j] = ns;
    }
  } else if (m == 0) {  // threshold <= 1 and no nonzero entry: nothing to send
    cnt = 0;
    if (threadIdx.x == 0) {
      FastState ns = st;
      ns.last_cands = 0;
      ns.calls += 1;
      state[j] = ns;
    }
  } else {
    // gather the layer's task lists in task order (= index order) into contiguous scratch
    const int64_t gbase = static_cast<int64_t>(tr.x) * cap;
    const bool in_smem = m <= static_cast<uint32_t>(smem_keys);
    uint32_t carry = 0;
    for (int t0 = tr.x; t0 < tr.y; t0 += SEL_NT) {
      const int t = t0 + threadIdx.x;
      const uint32_t c = t < tr.y ? static_cast<uint32_t>(cand_cnt[t]) : 0u;
      uint32_t tot;
      const uint32_t pos = carry + block_exclusive_scan<SEL_NT>(c, sm.warp_tot, &tot);
      for (uint32_t q = 0; q < c; ++q) {
        const int64_t src = static_cast<int64_t>(t) * cap + q;
        const float x = cand_val[src];
        gidx[gbase + pos + q] = cand_idx[src];
        gval[gbase + pos + q] = x;
        if (in_smem) skeys[pos + q] = Key<float>::of(x);
      }
      carry += tot;
      __syncthreads();
    }
    __threadfence_block();
    __syncthreads();
    const float* gv = gval + gbase;
    const int32_t* gi = gidx + gbase;
    const uint32_t* sk = skeys;
    auto key_at = [=](int64_t i) { return in_smem ? sk[i] : Key<float>::of(gv[i]); };
    const auto th = radix_select<uint32_t, 31, Key<float>::RB>(key_at, m, k, sm);
    auto load = [=](int64_t i, uint32_t* key, float* x, int64_t* ix) {
      *x = gv[i];
      *key = Key<float>::of(*x);
      *ix = gi[i];
    };
    auto emit = [=](uint32_t pos, int64_t, int64_t ix, float x) {
      oidx[pos] = static_cast<int32_t>(ix);
      oval[pos] = x;
      data[ix] = 0.0f;  // acc - acc == +0.0 (R: training.py:252)
    };
    cnt = ordered_compact<uint32_t, float>(m, th, load, emit, sm);
    // predict the next threshold: the (PRED_FACTOR*k)-th largest key of this call's candidates
    uint32_t pred;
    if (m >= PRED_FACTOR * k) {
      pred = radix_select<uint32_t, 31, Key<float>::RB>(key_at, m, PRED_FACTOR * k, sm).prefix;
    } else {
      const uint32_t T = th.prefix;  // >= st.thr
      const uint32_t step = max(2u * (T - min(T, st.thr)), 1u << 18);
      pred = st.thr > step ? st.thr - step : 1u;
    }
    if (threadIdx.x == 0) {
      FastState ns = st;
      ns.thr = max(pred, 1u);
      ns.last_cands = m;
      ns.calls += 1;
      state[j] = ns;
    }
  }
  if (threadIdx.x == 0) count_out[j] = static_cast<int32_t>(cnt);
}

}  // namespace lags
