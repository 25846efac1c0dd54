// fp32 fast path: one streaming pass over g and r that also emits index-ordered candidates above
// a per-layer predicted threshold, then a per-layer exact select over the candidates.
//
// K1 (accum_emit_kernel): one warp per task (a <= TASK_ELEMS slice of one layer).  Reads g and r
//    once (16-byte vectors), writes acc back into r, ORs the non-finite flag, and appends every
//    entry with key(acc) >= thr[layer] to the task's candidate list in ascending index order
//    (warp ballot + shuffle scan, no atomics).  Algorithmic traffic: 12 B/element.
// Selection (select_kernel, lags_cluster.cuh, one launch) per layer:
//  - tiny layers: warp_topk_layer, one warp, register top-k (no prediction needed);
//  - other layers with a prediction: candidate_select (or cluster_select_layer for the largest),
//    when the candidate set provably holds the top-k (count >= k, no task overflow): dual-rank
//    radix select in shared memory, ordered compaction, residual zeroing by scatter, and the
//    next threshold;
//  - otherwise the dense exact path in the same CTA (small_fallback_select staged in shared
//    memory, dense_fallback_select over r), which also yields the next prediction.
// Every path returns exactly the reference's selection: the candidate set contains every top-k
// element, and the dense paths scan all of r.  All launches are ordinary (not cooperative), so
// the selection can share the GPU with backprop kernels on other streams.
#pragma once
#include "lags_select.cuh"

namespace lags {

#ifndef LAGS_TASK_ELEMS
#define LAGS_TASK_ELEMS 8192
#endif
#ifndef LAGS_K1_UNROLL
#define LAGS_K1_UNROLL 4
#endif
constexpr int TASK_ELEMS = LAGS_TASK_ELEMS;  // elements per streaming task (one warp), large buckets
constexpr int MIN_TASK_ELEMS = 256;          // small buckets: down to this (bucket-dependent)
// layers up to SMALL_LAYER stage their dense exact path in shared memory (on a failed prediction);
// up to TINY_LAYER they always take it.  Measured: always-dense up to 16384 or 40960 elements
// (bigger staging, longer radix passes) made ResNet-50 78.9 / 95.4 us and ResNet-20 19.2 / 40.9 us
// per step, against 71.5 / 16.8 us with candidates above 4096.
constexpr int SMALL_LAYER = 16384;
constexpr int TINY_LAYER = 4096;
#ifndef LAGS_K1_WARPS
#define LAGS_K1_WARPS 8
#endif
#ifndef LAGS_K1_MINB
#define LAGS_K1_MINB 1
#endif
// K1's residual traffic (read + write of r, 8 B/element): for a residual much larger than L2 it
// streams through with evict-first priority like the gradient, so normal-priority lines (the
// candidate lists and histograms K1 writes, the weights, the selection kernel's own code) stay in
// L2 for the selection that follows (ResNet-50: 75.4 -> 71.4 us per step); a residual that fits in
// L2 keeps normal priority and is re-read from L2 by the next step (VGG-16: 53.7 -> 49.5 us).
template <bool RSTREAM>
__device__ __forceinline__ float4 r_load(const float4* p) {
  return RSTREAM ? __ldcs(p) : *p;
}
template <bool RSTREAM>
__device__ __forceinline__ void r_store(float4* p, float4 v) {
  if (RSTREAM) __stcs(p, v);
  else *p = v;
}
constexpr int K1_WARPS = LAGS_K1_WARPS;  // warps per K1 CTA
constexpr int K1_MINB = LAGS_K1_MINB;    // K1 CTAs per SM the register allocation must allow
constexpr int K1_UNROLL = LAGS_K1_UNROLL;        // float4 loads in flight per lane per operand (K1)
constexpr int PRED_FACTOR = 3;     // predicted threshold targets PRED_FACTOR * k candidates
constexpr int F32_BINS = 1 << Key<float>::RB;

struct Task {
  int64_t start;  // flat element offset
  int32_t len;
  int32_t layer;
};

struct FastState {
  uint32_t thr;         // candidate threshold key (0 = no prediction: dense exact path)
  uint32_t fallbacks;   // dense-path executions after a prediction existed (diagnostic)
  uint32_t last_cands;  // candidates at the last call (0 = dense path)
  uint32_t calls;
  uint32_t cycles;      // SM cycles the layer's selection took at the last call (diagnostic)
  uint32_t path;        // last path: 0 small / tiny dense, 1 candidates, 2 dense over r, 3 cluster
  uint32_t pf256;       // adaptive prediction rank factor x256 (0 = PRED_FACTOR)
  uint32_t reserved;    // candidate-path phase cycles (diagnostic)
  uint32_t t_start;     // %globaltimer (ns, low 32 bits) when the layer's CTA started / ended its
  uint32_t t_end;       //   selection work at the last call (diagnostic timeline)
  uint32_t t_launch;    // %globaltimer when the CTA entered the kernel (before griddepcontrol.wait)
  uint32_t cut;         // histogram-cut diagnostic: in_bin << 8 | code (0 resolved, see cut_code)
};

__device__ __forceinline__ uint32_t globaltimer_lo() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<uint32_t>(t);
}

constexpr float PRED_TARGET = 2.0f;  // wanted candidates per selected entry (m / k)
#ifndef LAGS_PRED_SIGMAS
#define LAGS_PRED_SIGMAS 3.0f
#endif
// Plus this many sqrt(m) of margin: at small k the candidate count's spread alone dropped it
// below k about once per 100 steps (k = 9 / 16 layers, tools/fallback_trace.py).
constexpr float PRED_SIGMAS = LAGS_PRED_SIGMAS;

// Wanted candidate count for a layer selecting k: PRED_TARGET * k plus a Poisson-style margin.
__device__ __forceinline__ float pred_target_count(uint32_t k) {
  const float m = PRED_TARGET * static_cast<float>(k);
  return m + PRED_SIGMAS * sqrtf(m);
}

__device__ __forceinline__ float pred_factor(const FastState& st) {
  return st.pf256 ? st.pf256 / 256.0f : static_cast<float>(PRED_FACTOR);
}

// Rank whose key becomes the next threshold: pf * k (at least k + 1).
__device__ __forceinline__ uint32_t pred_rank(const FastState& st, uint32_t k) {
  const float r = pred_factor(st) * static_cast<float>(k);
  return max(k + 1u, static_cast<uint32_t>(fminf(r, 4.0e9f)));
}

__device__ __forceinline__ uint32_t pf_encode(float pf) {
  return static_cast<uint32_t>(fminf(fmaxf(pf, 1.25f), 8.0f) * 256.0f);
}

// Per-call counter of the selection kernel (device memory of the bucket, reset by the next
// call's accum_emit_kernel): next position of the LPT layer list to hand out (persistent CTAs).
struct SelectCounters {
  uint32_t* work;
};

// Fused push: the selection writes each finished layer's count and (index, value) pairs into slot
// `rank` of every peer's receive area (csrc/lags_p2p.cu layout, parity of the coming epoch) right
// after its CTA produced them, so the NVLink transfer overlaps the remaining selection work; the
// last CTA to finish publishes the flags the peers' lags_p2p_wait acquires.  bases == nullptr: off.
struct PeerPush {
  const uint64_t* bases;  // device array: every rank's receive area (own included)
  int P, rank, G;         // G: flags per source rank (lags_p2p_wait checks P * G flags)
  uint64_t flags_bytes;
  int64_t msg_bytes, off_cnt, off_idx, off_val;
  const uint32_t* epoch;  // device epoch counter (advanced by the wait kernel)
  uint32_t* done;         // CTAs finished in this launch (reset by the last one)
};

__device__ __forceinline__ char* peer_slot(const PeerPush& pp, int p, uint32_t epoch) {
  return reinterpret_cast<char*>(pp.bases[p]) + pp.flags_bytes +
         static_cast<int64_t>(epoch & 1u) * pp.P * pp.msg_bytes + static_cast<int64_t>(pp.rank) * pp.msg_bytes;
}

// Threads tid (of nth) copy the layer's slots [lo, hi) (relative to its first slot) and, when
// cnt >= 0, its count to every peer.  The caller's writes of those slots are visible to it.
__device__ void peer_copy(const PeerPush& pp, uint32_t epoch, const int32_t* idx_out, const float* val_out, int64_t slot,
                          uint32_t lo, uint32_t hi, int j, int cnt, int tid, int nth) {
  for (int p = 0; p < pp.P; ++p) {
    char* d = peer_slot(pp, p, epoch);
    int32_t* di = reinterpret_cast<int32_t*>(d + pp.off_idx) + slot;
    float* dv = reinterpret_cast<float*>(d + pp.off_val) + slot;
    for (uint32_t i = lo + tid; i < hi; i += nth) {
      di[i] = idx_out[slot + i];
      dv[i] = val_out[slot + i];
    }
    if (cnt >= 0 && tid == 0) reinterpret_cast<int32_t*>(d + pp.off_cnt)[j] = cnt;
  }
}

// Every CTA of the selection, at its end: the last one to finish publishes epoch in its G flags
// of every peer (system-scope release; each CTA fenced its remote stores before counting itself).
__device__ void peer_publish(const PeerPush& pp, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(pp.done, 1u) == gridDim.x - 1) {
      *pp.done = 0u;
      __threadfence_system();
      for (int p = 0; p < pp.P; ++p)
        for (int gq = 0; gq < pp.G; ++gq) {
          uint32_t* flag = reinterpret_cast<uint32_t*>(pp.bases[p]) + pp.rank * pp.G + gq;
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
        }
    }
  }
}

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// K1's per-layer histogram of its candidate keys -- the selection's first cut without a pass over
// the candidates: HIST_BINS bins of 2^HIST_SHIFT consecutive keys, counted up from the layer's
// candidate threshold (32768 bins per octave of |x|, so the 4096 bins span keys up to 2^(1/8) =
// 1.09 times the threshold; larger keys share the top bin).  Error feedback piles the accumulated
// magnitudes up just below the threshold, so the bins must be fine there (at 1024 per octave the
// cut bin of a 2.4 M-element layer held 150-220 keys; at 8192 a 15 M-element LSTM layer's still
// held ~400, above BIN_LIST_MAX; at 16384 the 2.4 M-element layers' held 24-35, just above the
// one-key-per-lane warp resolve).  With the adaptive margin (m ~ 2k candidates) the k-th key sits
// a few percent above the threshold; a cut in the top bin takes the radix select.
// HIST_BINS equals the radix histogram size, so the radix find_bin2 resolves ranks on it.
#ifndef LAGS_HIST_SHIFT
#define LAGS_HIST_SHIFT 8
#endif
constexpr int HIST_SHIFT = LAGS_HIST_SHIFT;
constexpr int HIST_BINS = F32_BINS;
__device__ __forceinline__ uint32_t hist_bin(uint32_t key, uint32_t base) {
  return min((key >> HIST_SHIFT) - base, static_cast<uint32_t>(HIST_BINS - 1));
}

// Append this lane's candidate bits (ascending element order within the lane, lanes in index
// order) to the task list, and count each in the layer histogram hl (nullable; base = the
// threshold's bin).  Warp-collective.  The lane's (up to 4) values come by value: a dynamically
// indexed array would live in local memory.
__device__ __forceinline__ void emit_candidates(uint32_t bits, float4 vals, int64_t local0, int lane, uint32_t& cnt,
                                                int32_t* cidx, float* cval, int cap, uint32_t* hl, uint32_t base) {
  if (__ballot_sync(0xffffffffu, bits != 0) == 0u) return;
  const uint32_t c = __popc(bits);
  const uint32_t inc = warp_inclusive_scan(c, lane);
  uint32_t pos = cnt + inc - c;
  while (bits) {
    const int b = __ffs(bits) - 1;
    const float x = b == 0 ? vals.x : b == 1 ? vals.y : b == 2 ? vals.z : vals.w;
    if (pos < static_cast<uint32_t>(cap)) {
      cidx[pos] = static_cast<int32_t>(local0 + b);
      cval[pos] = x;
    }
    if (hl) atomicAdd(hl + hist_bin(Key<float>::of(x), base), 1u);
    ++pos;
    bits &= bits - 1;
  }
  cnt += __shfl_sync(0xffffffffu, inc, 31);
}

// One task of the streaming pass, by one warp (warp-collective): acc = r + alpha * g written back
// into r, the non-finite flag, and the task's candidate list (entries with key(acc) >= thr[layer],
// ascending index order) with its count in cand_cnt[tid].  gt / rt point at the task's first
// gradient / residual element (the gradient may live in its own per-layer tensor); 16-byte
// vectors when both share an alignment, scalar otherwise.
// ZERO_G: also clear the gradient after reading it (the optimizer's zero_grad fused into the pass;
// +4 B/element of writes instead of a separate memset pass).
template <bool ZERO_G, bool RSTREAM, int UNROLL>
__device__ __forceinline__ void stream_task(const Task& T, int tid, int lane, const lags_layer_t* __restrict__ layers,
                                            const FastState* state, float* __restrict__ gt, float* __restrict__ rt,
                                            float alpha, int cap, int32_t* __restrict__ cand_idx,
                                            float* __restrict__ cand_val, int32_t* __restrict__ cand_cnt,
                                            uint32_t* status, uint32_t* hist) {
  const int64_t local0 = T.start - layers[T.layer].offset;  // layer-local index of element 0
  const uint32_t thr0 = state[T.layer].thr;
  const uint32_t thr = thr0 ? thr0 : 0xffffffffu;
  uint32_t* hl = hist ? hist + static_cast<int64_t>(T.layer) * HIST_BINS : nullptr;
  const uint32_t hbase = thr0 >> HIST_SHIFT;
  int32_t* cidx = cand_idx + static_cast<int64_t>(tid) * cap;
  float* cval = cand_val + static_cast<int64_t>(tid) * cap;
  uint32_t cnt = 0;
  bool bad = false;
  const int n = T.len;
  const uintptr_t ra = reinterpret_cast<uintptr_t>(rt), ga = reinterpret_cast<uintptr_t>(gt);
  // scalar head up to 16-byte alignment of r; the whole task scalar if g is aligned differently
  const int h = ((ra ^ ga) & 15u) == 0 ? min(static_cast<int>(((16u - (ra & 15u)) & 15u) >> 2), n) : n;
  auto scalar = [&](int lo, int hi) {
    for (int q0 = lo; q0 < hi; q0 += 32) {  // warp-uniform trip count
      const int i = q0 + lane;
      uint32_t bits = 0;
      float a = 0.f;
      if (i < hi) {
        const float gi = gt[i];
        if (ZERO_G) gt[i] = 0.0f;
        bad |= nonfinite(gi);
        a = accum(rt[i], gi, alpha);
        rt[i] = a;
        bits = (Key<float>::of(a) >= thr) ? 1u : 0u;
      }
      emit_candidates(bits, make_float4(a, a, a, a), local0 + i, lane, cnt, cidx, cval, cap, hl, hbase);
    }
  };
  scalar(0, h);
  const int n4 = (n - h) >> 2;
  float4* g4 = reinterpret_cast<float4*>(gt + h);
  float4* r4 = reinterpret_cast<float4*>(rt + h);
  for (int q0 = 0; q0 < n4; q0 += 32 * UNROLL) {
    float4 gv[UNROLL], rv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int q = q0 + u * 32 + lane;
      if (q < n4) {
        gv[u] = __ldcs(g4 + q);
        rv[u] = r_load<RSTREAM>(r4 + q);
      }
    }
    if (ZERO_G) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int q = q0 + u * 32 + lane;
        if (q < n4) __stcs(g4 + q, make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int q = q0 + u * 32 + lane;
      uint32_t bits = 0;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < n4) {
        bad |= nonfinite(gv[u].x) | nonfinite(gv[u].y) | nonfinite(gv[u].z) | nonfinite(gv[u].w);
        a.x = accum(rv[u].x, gv[u].x, alpha);
        a.y = accum(rv[u].y, gv[u].y, alpha);
        a.z = accum(rv[u].z, gv[u].z, alpha);
        a.w = accum(rv[u].w, gv[u].w, alpha);
        r_store<RSTREAM>(r4 + q, a);
        bits = (Key<float>::of(a.x) >= thr ? 1u : 0u) | (Key<float>::of(a.y) >= thr ? 2u : 0u) |
               (Key<float>::of(a.z) >= thr ? 4u : 0u) | (Key<float>::of(a.w) >= thr ? 8u : 0u);
      }
      if (q0 + u * 32 < n4)
        emit_candidates(bits, a, local0 + h + 4 * static_cast<int64_t>(q), lane, cnt, cidx, cval, cap, hl, hbase);
    }
  }
  scalar(h + 4 * n4, n);  // scalar tail
  if (lane == 0) cand_cnt[tid] = static_cast<int32_t>(cnt);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, LAGS_STATUS_NONFINITE);
}

// K1, CTA form (large buckets): one CTA of K1C_NT threads per task of K1C_TASK elements, every
// thread's loads issued at once (no loop), so the hardware schedules thousands of short CTAs and
// the kernel ends within one CTA's lifetime of the last byte (a warp looping over a long task
// left a tail: 55 vs 47 us for the same 12 B/element in torch's elementwise kernel).  Thread t
// owns the float4 groups f = q * K1C_NT + t (q < 4): each load instruction of a warp reads 512
// contiguous bytes.  The task's candidates keep ascending index order = (q, t) order: one block
// scan of the four per-group counts packed into 16-bit fields.
constexpr int K1C_NT = 256;
constexpr int K1C_GROUPS = 4;
constexpr int K1C_TASK = K1C_NT * K1C_GROUPS * 4;  // 4096 elements

// Exclusive block scan of a packed 64-bit value (fields never carry: <= 4 * K1C_NT per field).
__device__ __forceinline__ unsigned long long k1c_scan(unsigned long long v, unsigned long long* wsum,
                                                       unsigned long long* total) {
  constexpr int NW = K1C_NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < NW ? wsum[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NW) wsum[lane] = wi - w;
    if (lane == NW - 1) wsum[NW] = wi;
  }
  __syncthreads();
  *total = wsum[NW];
  return wsum[warp] + x - v;
}

template <bool ZERO_G, bool RSTREAM>
__global__ void __launch_bounds__(K1C_NT) accum_emit_cta_kernel(
    const Task* __restrict__ tasks, int ntasks, const lags_layer_t* __restrict__ layers,
    const FastState* __restrict__ state, float* __restrict__ g, float* const* __restrict__ gtab,
    float* __restrict__ r, float alpha, int cap, int32_t* __restrict__ cand_idx, float* __restrict__ cand_val,
    int32_t* __restrict__ cand_cnt, uint32_t* status, uint32_t* work, uint32_t* hist) {
  __shared__ unsigned long long wsum[K1C_NT / 32 + 1];
  griddep_wait();  // the previous kernel on the stream (last call's select / decode) has completed
#ifndef LAGS_NO_EARLY_TRIGGER
  griddep_launch_dependents();
#endif
  const int tid = blockIdx.x;
  const int t = threadIdx.x;
  if (tid == 0 && t == 0) *work = 0u;  // the previous call's selection kernel has completed
  // the task descriptor is the only load the streaming loads depend on (flat g): the layer
  // offset and the threshold are read while they are in flight
  const Task T = tasks[tid];
  float* rt = r + T.start;
  int64_t local0 = 0;
  float* gt = g + T.start;
  if (gtab) {
    local0 = T.start - layers[T.layer].offset;
    gt = gtab[T.layer] + local0;
  }
  const int n = T.len;
  const bool vec = ((reinterpret_cast<uintptr_t>(rt) | reinterpret_cast<uintptr_t>(gt)) & 15u) == 0;
  float4 gv[K1C_GROUPS], rv[K1C_GROUPS];
#pragma unroll
  for (int q = 0; q < K1C_GROUPS; ++q) {
    const int e = 4 * (q * K1C_NT + t);
    gv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    rv[q] = gv[q];
    if (vec && e + 3 < n) {
      gv[q] = __ldcs(reinterpret_cast<const float4*>(gt + e));
      rv[q] = r_load<RSTREAM>(reinterpret_cast<const float4*>(rt + e));
    } else if (e < n) {  // unaligned task or the layer's last partial group
      float* gp = &gv[q].x;
      float* rp = &rv[q].x;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (e + c < n) {
          gp[c] = gt[e + c];
          rp[c] = rt[e + c];
        }
    }
  }
  if (!gtab) local0 = T.start - layers[T.layer].offset;
  const uint32_t thr0 = state[T.layer].thr;
  const uint32_t thr = thr0 ? thr0 : 0xffffffffu;
  uint32_t* hl = hist ? hist + static_cast<int64_t>(T.layer) * HIST_BINS : nullptr;
  const uint32_t hbase = thr0 >> HIST_SHIFT;
  bool bad = false;
  uint32_t masks = 0;  // 4 bits per group
  unsigned long long packed = 0ull;
  float4 av[K1C_GROUPS];
#pragma unroll
  for (int q = 0; q < K1C_GROUPS; ++q) {
    const int e = 4 * (q * K1C_NT + t);
    float4 a;
    a.x = accum(rv[q].x, gv[q].x, alpha);
    a.y = accum(rv[q].y, gv[q].y, alpha);
    a.z = accum(rv[q].z, gv[q].z, alpha);
    a.w = accum(rv[q].w, gv[q].w, alpha);
    av[q] = a;
    if (vec && e + 3 < n) {
      bad |= nonfinite(gv[q].x) | nonfinite(gv[q].y) | nonfinite(gv[q].z) | nonfinite(gv[q].w);
      if (ZERO_G) __stcs(reinterpret_cast<float4*>(gt + e), make_float4(0.f, 0.f, 0.f, 0.f));
      r_store<RSTREAM>(reinterpret_cast<float4*>(rt + e), a);
      const uint32_t m = (Key<float>::of(a.x) >= thr ? 1u : 0u) | (Key<float>::of(a.y) >= thr ? 2u : 0u) |
                         (Key<float>::of(a.z) >= thr ? 4u : 0u) | (Key<float>::of(a.w) >= thr ? 8u : 0u);
      masks |= m << (4 * q);
      packed |= static_cast<unsigned long long>(__popc(m)) << (16 * q);
    } else if (e < n) {
      const float* ap = &a.x;
      const float* gp = &gv[q].x;
      uint32_t m = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (e + c < n) {
          bad |= nonfinite(gp[c]);
          if (ZERO_G) gt[e + c] = 0.0f;
          rt[e + c] = ap[c];
          m |= (Key<float>::of(ap[c]) >= thr ? 1u : 0u) << c;
        }
      masks |= m << (4 * q);
      packed |= static_cast<unsigned long long>(__popc(m)) << (16 * q);
    }
  }
  unsigned long long tot;
  const unsigned long long ex = k1c_scan(packed, wsum, &tot);
  int32_t* cidx = cand_idx + static_cast<int64_t>(tid) * cap;
  float* cval = cand_val + static_cast<int64_t>(tid) * cap;
  uint32_t before = 0;  // candidates of the lower groups (all threads)
#pragma unroll
  for (int q = 0; q < K1C_GROUPS; ++q) {
    uint32_t pos = before + static_cast<uint32_t>((ex >> (16 * q)) & 0xffffu);
    uint32_t m = (masks >> (4 * q)) & 0xfu;
    while (m) {
      const int c = __ffs(m) - 1;
      const float x = c == 0 ? av[q].x : c == 1 ? av[q].y : c == 2 ? av[q].z : av[q].w;
      if (pos < static_cast<uint32_t>(cap)) {
        cidx[pos] = static_cast<int32_t>(local0 + 4 * (q * K1C_NT + t) + c);
        cval[pos] = x;
      }
      if (hl) atomicAdd(hl + hist_bin(Key<float>::of(x), hbase), 1u);
      ++pos;
      m &= m - 1;
    }
    before += static_cast<uint32_t>((tot >> (16 * q)) & 0xffffu);
  }
  if (t == 0) cand_cnt[tid] = static_cast<int32_t>(before);
  if (__any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(status, LAGS_STATUS_NONFINITE);  // no barrier
}

// K1: one warp per task.  gtab (nullable): per-layer gradient pointers replacing the flat g.
// UNROLL: float4 loads in flight per lane and operand -- K1_UNROLL (80 registers, 24 warps per SM)
// or 2 * K1_UNROLL (116 registers, 16 warps per SM); the bucket picks the one whose resident-warp
// waves are fuller (lags_bucket_create).
template <bool ZERO_G, bool RSTREAM, int UNROLL = K1_UNROLL>
__global__ void __launch_bounds__(K1_WARPS * 32, K1_MINB) accum_emit_kernel(
    const Task* __restrict__ tasks, int ntasks, const lags_layer_t* __restrict__ layers,
    const FastState* __restrict__ state, float* __restrict__ g, float* const* __restrict__ gtab,
    float* __restrict__ r, float alpha, int cap, int32_t* __restrict__ cand_idx, float* __restrict__ cand_val,
    int32_t* __restrict__ cand_cnt, uint32_t* status, uint32_t* work, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * K1_WARPS + (threadIdx.x >> 5);
  griddep_wait();  // the previous kernel on the stream (last call's select / decode) has completed
  // let the selection kernel (PDL) be scheduled: it is launched once the last K1 CTA has started,
  // so its CTAs take SMs as K1's last wave drains, and it waits for K1's completion itself
#ifndef LAGS_NO_EARLY_TRIGGER
  griddep_launch_dependents();
#endif
  if (wid == 0 && lane == 0) *work = 0u;  // the previous call's selection kernel has completed
  if (wid >= ntasks) return;
  const Task T = tasks[wid];
  float* gt = gtab ? gtab[T.layer] + (T.start - layers[T.layer].offset) : g + T.start;
  stream_task<ZERO_G, RSTREAM, UNROLL>(T, wid, lane, layers, state, gt, r + T.start, alpha, cap, cand_idx, cand_val,
                                 cand_cnt, status, hist);
}

// Block-wide sum; all threads get the result.  Uses sm.warp_tot.
template <int RB>
__device__ LAGS_SUM_ATTR uint32_t block_sum(uint32_t v, RadixSmem<RB>& sm) {
  uint32_t tot;
  block_exclusive_scan<SEL_NT>(v, sm.warp_tot, &tot);
  __syncthreads();
  return tot;
}

struct SelectSmem {
  RadixSmem<Key<float>::RB> sm;
  alignas(16) uint32_t hist2[F32_BINS];  // second histogram (prediction rank) of the cooperative dense path
  uint32_t tpos[SEL_NT];     // candidate gather: per-task output position / count
  uint32_t tcnt[SEL_NT];
  uint32_t tcache[2 * SEL_NT];  // the layer's task counts from the counting pass (speculative gathers:
                                // <= SEL_NT tasks per CTA, <= 2 * SEL_NT per cluster layer)
  uint32_t rpos[SEL_NT];     // speculative gather: positions of the tasks' remainders
};

// P = 1 update fused into the selection epilogue (no exchange, no separate decode): the decode of
// R: training.py:248,253-254 with one worker, v = fl32(fl64(v) - (0.0 + x) / 1).  Computed in fp32:
// the division by 1 is exact, 0.0 + x only maps -0 to +0, and rounding the exact difference of two
// floats to double (53 >= 2*24 + 2 bits) then to float gives the directly rounded float difference
// (innocuous double rounding), so the bits are the same.
__device__ __forceinline__ float single_rank_update(float v, float x) { return __fsub_rn(v, __fadd_rn(0.0f, x)); }

// Post-pass over a layer's selected (idx, val) just written by the compaction: batches of
// independent weight loads in flight per thread (the weights are HBM-resident and scattered).
__device__ __forceinline__ void apply_single_rank_updates(float* vl, const int32_t* oidx, const float* oval,
                                                          uint32_t cnt) {
  __syncthreads();  // the block's compaction writes are visible
  constexpr int B = UPDATE_B;
  for (uint32_t q0 = 0; q0 < cnt; q0 += SEL_NT * B) {
    int32_t ix[B];
    float x[B], w[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const uint32_t q = q0 + u * SEL_NT + threadIdx.x;
      ix[u] = q < cnt ? oidx[q] : -1;
      x[u] = q < cnt ? oval[q] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) w[u] = ix[u] >= 0 ? vl[ix[u]] : 0.0f;
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (ix[u] >= 0) vl[ix[u]] = single_rank_update(w[u], x[u]);
  }
}

// Two ranks in one set of radix passes over m keys (shared memory): the exact threshold of the
// k largest (select form) and a lower bound of the k2-th largest key (the next prediction).
// Passes start below the common prefix of all keys (candidates crowd just above the threshold).
// skip_prefix = false (dense data in global memory) starts at the top bit without the OR pass;
// diff_key0 = {OR of key ^ key0 over all keys, key0} (computed by the caller's gather) skips it.
// coarse_key2: the prediction is the lower edge of its first-pass bin (candidate sets, where a
// first-pass bin holds a few keys) instead of being refined in the later passes.
// Once the threshold's bin holds at most BIN_LIST_MAX keys, the remaining passes are replaced by
// one pass that lists the bin's keys and a direct rank count among them.
#ifndef LAGS_BIN_LIST_MAX
#define LAGS_BIN_LIST_MAX 256
#endif
constexpr uint32_t BIN_LIST_MAX = LAGS_BIN_LIST_MAX;

template <typename KeyAt>
__device__ void radix_select_dual(KeyAt key_at, int64_t m, uint32_t k, uint32_t k2, SelectSmem& cs,
                                  SelectThreshold<uint32_t>* th_out, uint32_t* key2_out, bool skip_prefix = true,
                                  const uint32_t* diff_key0 = nullptr, bool coarse_key2 = false) {
  constexpr int RB = Key<float>::RB;
  constexpr uint32_t FULL = 0x7fffffffu;
  RadixSmem<RB>& sm = cs.sm;
  uint32_t key0 = 0u, diff = FULL;
  if (diff_key0) {
    diff = diff_key0[0];
    key0 = diff_key0[1];
  } else if (skip_prefix) {
    key0 = key_at(0);
    diff = 0;
    for (int64_t i = threadIdx.x; i < m; i += SEL_NT) diff |= key_at(i) ^ key0;
    diff = block_or<uint32_t, RB>(diff, sm);
  }
  uint32_t prefix[2], pmask[2];
  uint32_t rank[2] = {static_cast<int64_t>(k) < m ? k : static_cast<uint32_t>(m),
                      static_cast<int64_t>(k2) < m ? k2 : static_cast<uint32_t>(m)};
  uint32_t n_gt0 = 0;
  bool done[2] = {false, false};
  int shift = 0, width = 0;
  if (diff == 0) {
    prefix[0] = prefix[1] = key0;
    pmask[0] = pmask[1] = FULL;
  } else {
    const int h = 31 - __clz(static_cast<int>(diff));
    const uint32_t pm = FULL & ~((1u << (h + 1)) - 1u);
    prefix[0] = prefix[1] = key0 & pm;
    pmask[0] = pmask[1] = pm;
    shift = h + 1 > RB ? h + 1 - RB : 0;
    width = h + 1 - shift;
  }
  while (width > 0 && !(done[0] && done[1])) {
    const bool same = !done[0] && !done[1] && prefix[0] == prefix[1] && pmask[0] == pmask[1];
    const bool second = !same && !done[1];
    for (int b = threadIdx.x; b < F32_BINS; b += SEL_NT) {
      sm.hist[b] = 0;
      if (second) cs.hist2[b] = 0;
    }
    if (threadIdx.x == 0) sm.list_n = 0;
    __syncthreads();
    const uint32_t dmask = (1u << width) - 1u;
    for (int64_t i = threadIdx.x; i < m; i += SEL_NT) {
      const uint32_t key = key_at(i);
      const uint32_t bin = (key >> shift) & dmask;
      if (!done[0] && (key & pmask[0]) == prefix[0]) atomicAdd(&sm.hist[bin], 1u);
      if (second && (key & pmask[1]) == prefix[1]) atomicAdd(&cs.hist2[bin], 1u);
    }
    __syncthreads();
    uint32_t bin[2], above[2], in_bin[2];
    if (same) {
      find_bin2<RB>(sm, sm.hist, rank[0], rank[1], bin, above, in_bin);
    } else {
      for (int q = 0; q < 2; ++q)
        if (!done[q]) find_bin<RB>(sm, rank[q], &bin[q], &above[q], &in_bin[q], q == 0 ? sm.hist : cs.hist2);
    }
    for (int q = 0; q < 2; ++q) {
      if (done[q]) continue;
      prefix[q] |= bin[q] << shift;
      pmask[q] |= dmask << shift;
      rank[q] -= above[q];
      if (q == 0) n_gt0 += above[q];
      if (shift == 0 || (in_bin[q] == rank[q] && prefix[q] != 0u)) done[q] = true;
    }
    if (coarse_key2) done[1] = true;
#ifdef LAGS_DBG_SELECT
    if (threadIdx.x == 0) {
      if (shift + width == (diff ? 32 - __clz(static_cast<int>(diff)) : 0))  // first pass
        sm.dbg = min(in_bin[0], 4095u) | (static_cast<uint32_t>(diff ? 31 - __clz(static_cast<int>(diff)) : 0) << 12);
      sm.dbg += 1u << 18;  // passes
    }
#endif
    const int ns = shift > RB ? shift - RB : 0;
    width = shift - ns;
    shift = ns;
    if (!done[0] && done[1] && in_bin[0] <= BIN_LIST_MAX) {
      // bin-list finish: the threshold bin's keys, then the rank[0]-th largest by direct count
      uint32_t* list = cs.hist2;
      for (int64_t i = threadIdx.x; i < m; i += SEL_NT) {
        const uint32_t key = key_at(i);
        if ((key & pmask[0]) == prefix[0]) list[atomicAdd(&sm.list_n, 1u)] = key;
      }
      __syncthreads();
      const uint32_t c = in_bin[0];
      if (threadIdx.x < c) {
        const uint32_t mine = list[threadIdx.x];
        uint32_t gt = 0, eq = 0;
        for (uint32_t q = 0; q < c; ++q) {
          const uint32_t x = list[q];
          gt += x > mine ? 1u : 0u;
          eq += x == mine ? 1u : 0u;
        }
        if (gt < rank[0] && rank[0] <= gt + eq) {  // equal keys write equal values
          sm.list_key = mine;
          sm.list_gt = gt;
        }
      }
      __syncthreads();
      prefix[0] = sm.list_key;
      pmask[0] = FULL;
      rank[0] -= sm.list_gt;
      n_gt0 += sm.list_gt;
      done[0] = true;
#ifdef LAGS_DBG_SELECT
      if (threadIdx.x == 0) sm.dbg |= 1u << 22;
#endif
      __syncthreads();  // list_key / list_gt / the list are read before any reuse
    }
  }
  if (static_cast<int64_t>(k) >= m) {  // every nonzero candidate is selected
    th_out->prefix = 0u;
    th_out->pmask = 0xffffffffu;
    th_out->n_gt = 0;
    th_out->need_eq = 0;
  } else {
    th_out->prefix = prefix[0];
    th_out->pmask = pmask[0];
    th_out->n_gt = n_gt0;
    th_out->need_eq = prefix[0] == 0u ? 0u : rank[0];
  }
  *key2_out = prefix[1];
}

// Next candidate threshold: the k2-th largest candidate key, or, when fewer candidates were seen,
// an extrapolation below the current threshold from the observed candidate density.
__device__ __forceinline__ uint32_t next_threshold(const FastState& st, uint32_t m, uint32_t k, uint32_t k2,
                                                   uint32_t th_prefix, uint32_t key2) {
  if (m >= k2) return key2;
  if (st.thr <= 1u) return st.thr;
  const uint32_t T = max(th_prefix, st.thr);
  const double density = (static_cast<double>(m - min(m, k)) + 1.0) / (static_cast<double>(T - st.thr) + 1.0);
  double step = (static_cast<double>(k2) - m) / density;
  step = fmin(fmax(step, 64.0), 4.0 * (static_cast<double>(T - st.thr) + (1 << 16)));
  return st.thr > step ? st.thr - static_cast<uint32_t>(step) : 1u;
}

// State after a candidate-path selection; the rank factor gets feedback: the threshold set last
// call (rank pf*k) produced m candidates now, steer the next toward pred_target_count(k)
// (geometric mean of the old and the corrected factor).
__device__ __forceinline__ FastState candidate_state(const FastState& st, uint32_t pred, uint32_t m, uint32_t k,
                                                     uint32_t phases) {
  FastState ns = st;
  ns.thr = max(pred, 1u);
  ns.last_cands = m;
  ns.calls += 1;
  ns.reserved = phases;
  if (m > 0) {
    const float pf = pred_factor(st);
    const float corrected = pf * pred_target_count(k) / static_cast<float>(m);
    ns.pf256 = pf_encode(sqrtf(pf * fmaxf(corrected, 0.25f)));
  }
  return ns;
}

// Histogram cut of a candidate set (K1's per-layer histogram, staged in cs.sm.hist): the bins
// holding the k-th and the k2-th largest candidate (k, k2 <= m).
struct HistCut {
  uint32_t bin, above, in_bin;  // rank k: its bin, the candidates in higher bins, the bin's count
  uint32_t bin2;                // rank k2 (the next prediction): its bin
};

// The layer's histogram in registers: thread t holds the 8 consecutive bins of chunk
// SEL_NT - 1 - t (two 16-byte loads), so the block scan over threads runs from the top bin down.
constexpr int HIST_PER_THREAD = HIST_BINS / SEL_NT;
static_assert(HIST_PER_THREAD == 8, "two uint4 of bins per thread");
struct HistRegs {
  uint4 lo, hi;  // bins c*8 + 0..3, c*8 + 4..7 of chunk c = SEL_NT - 1 - threadIdx.x
};
__device__ __forceinline__ void hist_load(const uint32_t* hl, HistRegs& h) {
  const uint4* src = reinterpret_cast<const uint4*>(hl) + 2 * (SEL_NT - 1 - static_cast<int>(threadIdx.x));
  h.lo = __ldcg(src);
  h.hi = __ldcg(src + 1);
}

// Clear the nonzero bins of this thread's chunk (its register copy) for the next call's K1: a
// few hundred bins of the 4096 are in use, so this writes ~50 KB instead of 16 KB per layer x 53.
__device__ __forceinline__ void clear_hist_chunk(const HistRegs& h, uint32_t* hl) {
  uint4* dst = reinterpret_cast<uint4*>(hl) + 2 * (SEL_NT - 1 - static_cast<int>(threadIdx.x));
  if (h.lo.x | h.lo.y | h.lo.z | h.lo.w) dst[0] = make_uint4(0u, 0u, 0u, 0u);
  if (h.hi.x | h.hi.y | h.hi.z | h.hi.w) dst[1] = make_uint4(0u, 0u, 0u, 0u);
}

// Clear bins [lo, hi) of a layer histogram for the next call's K1 (16-byte stores).
__device__ __forceinline__ void zero_hist(uint32_t* hl, int lo, int hi) {
  uint4* dst = reinterpret_cast<uint4*>(hl);
  for (int i = lo / 4 + threadIdx.x; i < hi / 4; i += SEL_NT) dst[i] = make_uint4(0u, 0u, 0u, 0u);
}

// The bins of ranks k and k2 (<= m) from the register histogram: one block scan, no staging.
// All threads.
__device__ __forceinline__ HistCut hist_cut(const HistRegs& h, SelectSmem& cs, uint32_t k, uint32_t k2, uint32_t m) {
  // descending: bin 7 of the chunk first
  const uint32_t hv[8] = {h.hi.w, h.hi.z, h.hi.y, h.hi.x, h.lo.w, h.lo.z, h.lo.y, h.lo.x};
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += hv[q];
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<SEL_NT>(s, cs.sm.warp_tot, &tot);
  const uint32_t top = (SEL_NT - threadIdx.x) * 8u - 1u;  // the chunk's highest bin
  const uint32_t rr[2] = {min(k, m), min(k2, m)};
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const uint32_t r = rr[w];
    if (ex < r && r <= ex + s) {
      uint32_t c = ex;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (r <= c + hv[q]) {
          cs.sm.count2[w] = hv[q];
          cs.sm.above2[w] = c;
          cs.sm.found2[w] = top - q;
          break;
        }
        c += hv[q];
      }
    }
  }
  __syncthreads();
  // (no trailing barrier: found2 / above2 / count2 are written again only by a later layer's cut,
  // many barriers later)
  return HistCut{cs.sm.found2[0], cs.sm.above2[0], cs.sm.count2[0], cs.sm.found2[1]};
}

// Warp-level resolution of the cut (every warp computes it redundantly: no block barrier).  The
// cut bin's c <= WARP_CUT_MAX keys, lane i holding keys i + 32 j (kk[j]) of owner ranks oo[j]
// (cluster rank; 0 single CTA): the r-th largest is the threshold T; returns {T, gt = keys > T,
// low_gt / low_eq = keys > / == T owned by ranks below `rank`}.
struct WarpCut {
  uint32_t key, gt, low_gt, low_eq;
};
constexpr int WARP_CUT_KEYS = 1;  // keys per lane: beyond 32 keys the histogram resolve is faster
constexpr uint32_t WARP_CUT_MAX = 32u * WARP_CUT_KEYS;
__device__ __forceinline__ WarpCut warp_resolve(const uint32_t (&kk)[WARP_CUT_KEYS],
                                                const uint32_t (&oo)[WARP_CUT_KEYS], uint32_t c, uint32_t r,
                                                uint32_t rank) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t gt[WARP_CUT_KEYS], eq[WARP_CUT_KEYS];
#pragma unroll
  for (int j = 0; j < WARP_CUT_KEYS; ++j) gt[j] = eq[j] = 0u;
#pragma unroll
  for (int jq = 0; jq < WARP_CUT_KEYS; ++jq) {  // source slot jq: keys 32 jq .. 32 jq + 31
    const uint32_t n = c > 32u * jq ? min(c - 32u * jq, 32u) : 0u;
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t x = __shfl_sync(0xffffffffu, kk[jq], q);
#pragma unroll
      for (int j = 0; j < WARP_CUT_KEYS; ++j) {
        gt[j] += x > kk[j] ? 1u : 0u;
        eq[j] += x == kk[j] ? 1u : 0u;
      }
    }
  }
  WarpCut wc{0u, 0u, 0u, 0u};
  bool found = false;
#pragma unroll
  for (int j = 0; j < WARP_CUT_KEYS; ++j) {  // equal keys give equal answers: any hit
    const unsigned hit = __ballot_sync(0xffffffffu, lane + 32u * j < c && gt[j] < r && r <= gt[j] + eq[j]);
    if (!found && hit) {
      const int src = __ffs(hit) - 1;
      wc.key = __shfl_sync(0xffffffffu, kk[j], src);
      wc.gt = __shfl_sync(0xffffffffu, gt[j], src);
      found = true;
    }
  }
#pragma unroll
  for (int j = 0; j < WARP_CUT_KEYS; ++j) {
    const bool low = lane + 32u * j < c && oo[j] < rank;
    wc.low_gt += __popc(__ballot_sync(0xffffffffu, low && kk[j] > wc.key));
    wc.low_eq += __popc(__ballot_sync(0xffffffffu, low && kk[j] == wc.key));
  }
  return wc;
}

// The exact threshold from the keys of the cut bin (list[0..c), any order, c <= BIN_LIST_MAX): the
// r-th largest of them (1 <= r <= c) is T; the selection is every key > T (n_gt = above + those in
// the list) plus the first need_eq entries equal to T in index order (R: sparsify.py:85-88, lowest
// index wins).  Every key's rank is counted against the list by all threads at once (key i, slice
// t / c of the others), the partial counts added in shared memory: two barriers.  The counters
// (cut_counters) must be zero on entry (the callers clear them before an earlier barrier).
constexpr int CUT_COUNTERS = 2 * BIN_LIST_MAX + 2;  // gt[c], eq[c], and two totals for the callers
__device__ __forceinline__ uint32_t* cut_counters(SelectSmem& cs) { return cs.sm.hist; }
__device__ __forceinline__ void clear_cut_counters(SelectSmem& cs) {
  for (int i = threadIdx.x; i < CUT_COUNTERS; i += SEL_NT) cs.sm.hist[i] = 0u;
}
__device__ __forceinline__ SelectThreshold<uint32_t> resolve_cut(const uint32_t* list, uint32_t c, uint32_t r,
                                                                 uint32_t above, SelectSmem& cs) {
  uint32_t* gtc = cut_counters(cs);
  uint32_t* eqc = gtc + BIN_LIST_MAX;
  const uint32_t slices = SEL_NT / c, per = (c + slices - 1) / slices;
  if (threadIdx.x < slices * c) {
    const uint32_t i = threadIdx.x % c, sl = threadIdx.x / c;
    const uint32_t mine = list[i];
    uint32_t gt = 0, eq = 0;
    for (uint32_t j = sl * per; j < min(c, (sl + 1) * per); ++j) {
      const uint32_t x = list[j];
      gt += x > mine ? 1u : 0u;
      eq += x == mine ? 1u : 0u;
    }
    if (gt) atomicAdd(&gtc[i], gt);
    if (eq) atomicAdd(&eqc[i], eq);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < c; i += SEL_NT) {
    if (gtc[i] < r && r <= gtc[i] + eqc[i]) {  // equal keys write equal values
      cs.sm.list_key = list[i];
      cs.sm.list_gt = gtc[i];
    }
  }
  __syncthreads();
  SelectThreshold<uint32_t> th;
  th.prefix = cs.sm.list_key;
  th.pmask = 0x7fffffffu;
  th.n_gt = above + cs.sm.list_gt;
  th.need_eq = r - cs.sm.list_gt;
  return th;
}

// Candidate gather of tasks [t_lo, t_hi) into sv / si (ascending index order): positions by a
// block scan over the task counts, then one warp per task copies the task's list (lane l takes
// entries l, l + 32, ...: coalesced), GATHER_TASKS tasks per warp in flight.  On the way, against
// the histogram cut (cut_bin, base; cut_bin == ~0u: no cut): the entries in higher bins are
// counted into *gtb (shared), the keys of the cut bin are appended to list (shared, *list_n), and
// the weights of possibly selected entries are prefetched into L2 (vpf, P = 1 update).  The keys'
// common-prefix OR against key0 goes to cs.sm.diff_acc (radix fallback).  tc (nullable): the task
// counts already in shared memory, tc[t - t_base] for every task of the range.  Returns the
// number gathered.  All threads.
#ifndef LAGS_GATHER_TASKS
#define LAGS_GATHER_TASKS 5
#endif
#ifndef LAGS_GATHER_ILP
#define LAGS_GATHER_ILP 4
#endif
constexpr int GATHER_ILP = LAGS_GATHER_ILP;  // leftover candidate loads in flight per thread
constexpr int GATHER_TASKS = LAGS_GATHER_TASKS;

__device__ uint32_t gather_candidates(int t_lo, int t_hi, const int32_t* __restrict__ cand_cnt,
                                      const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_val, int cap,
                                      float* sv, int32_t* si, SelectSmem& cs, uint32_t key0, uint32_t base,
                                      uint32_t cut_bin, uint32_t* gtb, uint32_t* list, uint32_t* list_n,
                                      const float* vpf, const uint32_t* tc, int t_base) {
  constexpr int NW = SEL_NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t carry = 0, my_gt = 0, dx = 0;
  if (threadIdx.x == 0) cs.sm.diff_acc = 0u;
  auto take = [&](float x, int32_t ix, uint32_t e) {
    const uint32_t key = Key<float>::of(x);
    sv[e] = x;
    si[e] = ix;
    dx |= key ^ key0;
    const uint32_t b = hist_bin(key, base);
    if (cut_bin == ~0u || b >= cut_bin) {
      if (vpf) asm volatile("prefetch.global.L2 [%0];" ::"l"(vpf + ix));  // P = 1 weight
      if (cut_bin != ~0u) {
        if (b > cut_bin) {
          ++my_gt;
        } else {
          const uint32_t at = atomicAdd(list_n, 1u);
          if (at < BIN_LIST_MAX) list[at] = key;
        }
      }
    }
  };
  for (int t0 = t_lo; t0 < t_hi; t0 += SEL_NT) {
    const int nt = min(SEL_NT, t_hi - t0);
    uint32_t c = 0u;
    if (threadIdx.x < nt) c = tc ? tc[t0 - t_base + threadIdx.x] : static_cast<uint32_t>(__ldcg(cand_cnt + t0 + threadIdx.x));
    c = min(c, static_cast<uint32_t>(cap));
    uint32_t tot;
    const uint32_t pos = block_exclusive_scan<SEL_NT>(c, cs.sm.warp_tot, &tot);
    cs.tpos[threadIdx.x] = carry + pos;
    cs.tcnt[threadIdx.x] = c;
    __syncthreads();
    for (int tb = warp; tb < nt; tb += NW * GATHER_TASKS) {
      uint32_t cc[GATHER_TASKS], pp[GATHER_TASKS];
      float xv[GATHER_TASKS];
      int32_t xi[GATHER_TASKS];
#pragma unroll
      for (int u = 0; u < GATHER_TASKS; ++u) {
        const int tt = tb + u * NW;
        cc[u] = tt < nt ? cs.tcnt[tt] : 0u;
        pp[u] = tt < nt ? cs.tpos[tt] : 0u;
        if (static_cast<uint32_t>(lane) < cc[u]) {
          const int64_t src = static_cast<int64_t>(t0 + tt) * cap + lane;
          xv[u] = __ldcg(cand_val + src);
          xi[u] = __ldcg(cand_idx + src);
        }
      }
#pragma unroll
      for (int u = 0; u < GATHER_TASKS; ++u)
        if (static_cast<uint32_t>(lane) < cc[u]) take(xv[u], xi[u], pp[u] + lane);
#pragma unroll 1
      for (int u = 0; u < GATHER_TASKS; ++u) {  // lists longer than a warp (rare)
        const int64_t row = static_cast<int64_t>(t0 + tb + u * NW) * cap;
        for (uint32_t e = 32u + lane; e < cc[u]; e += 32u) take(__ldcg(cand_val + row + e), __ldcg(cand_idx + row + e), pp[u] + e);
      }
    }
    carry += tot;
    __syncthreads();  // tpos / tcnt reuse
  }
  dx = __reduce_or_sync(0xffffffffu, dx);
  if (lane == 0 && dx) atomicOr(&cs.sm.diff_acc, dx);
  my_gt = __reduce_add_sync(0xffffffffu, my_gt);
  if (gtb && lane == 0 && my_gt) atomicAdd(gtb, my_gt);
  return carry;
}

// Speculative candidate gather: counts, histogram and candidates in ONE round trip.  Before the
// counts are known, warp w loads entry `lane` of its tasks t_lo + w + NW * u (u < GATHER_TASKS),
// i.e. each task's first 32 candidates (usually all of them; reading past a short list stays
// inside its cap slots).  After the counts' scan, spec_place puts them at their positions,
// classifies them against the histogram cut and prefetches the possibly selected entries' weights
// (P = 1 update) into L2 for the compaction.  Leftovers (tasks beyond NW * GATHER_TASKS, lists
// longer than 32) follow with one thread per entry.  nt <= SEL_NT.
#ifndef LAGS_SPEC_LANES
#define LAGS_SPEC_LANES 16
#endif
// lanes per task in the speculative loads (SPEC_TPW tasks per warp load instruction): a
// 4096-element task of K1's CTA form holds ~8 candidates at the margin
constexpr int SPEC_LANES = LAGS_SPEC_LANES;
constexpr int SPEC_TPW = 32 / SPEC_LANES;
#ifdef LAGS_DBG_STAMPS
__device__ unsigned long long lags_dbg_sp[8];  // spec_place phases of block 0 (diagnostic builds)
#define LAGS_SPSTAMP(i)                                                          \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0) lags_dbg_sp[i] = clock64();         \
  } while (0)
#else
#define LAGS_SPSTAMP(i) \
  do {                  \
  } while (0)
#endif
struct SpecGather {
  float xv[GATHER_TASKS];
  int32_t xi[GATHER_TASKS];
};

__device__ __forceinline__ void spec_load(SpecGather& g, int t_lo, int nt, const int32_t* __restrict__ cand_idx,
                                          const float* __restrict__ cand_val, int cap) {
  constexpr int NW = SEL_NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < GATHER_TASKS; ++u) {
    const int tt = (warp + NW * u) * SPEC_TPW + lane / SPEC_LANES;
    if (tt < nt) {
      const int64_t src = static_cast<int64_t>(t_lo + tt) * cap + lane % SPEC_LANES;
      g.xv[u] = __ldcg(cand_val + src);
      g.xi[u] = __ldcg(cand_idx + src);
    }
  }
}

// All threads.  tc[0..nt): the range's task counts (shared).  vl (nullable): the layer's weights
// (P = 1 update), prefetched for the possibly selected.  Classification as gather_candidates.
__device__ uint32_t spec_place(SpecGather& g, int t_lo, int nt, const uint32_t* tc, const int32_t* __restrict__ cand_idx,
                               const float* __restrict__ cand_val, int cap, float* sv, int32_t* si,
                               const float* vl, SelectSmem& cs, uint32_t key0, uint32_t base, uint32_t cut_bin,
                               uint32_t* gtb, uint32_t* list, uint32_t* list_n, uint32_t m_own) {
  constexpr int NW = SEL_NT / 32;
  // tasks whose first SPEC_LANES entries are loaded speculatively; a covered task of up to
  // 2 * SPEC_LANES entries has its rest taken by its own lanes, everything else is a leftover
  constexpr int COVERED = NW * GATHER_TASKS * SPEC_TPW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  LAGS_SPSTAMP(0);
  const uint32_t c = threadIdx.x < nt ? min(tc[threadIdx.x], static_cast<uint32_t>(cap)) : 0u;
  const bool covered = static_cast<int>(threadIdx.x) < COVERED;
  const uint32_t skip = !covered ? 0u : (c <= 2u * SPEC_LANES ? c : static_cast<uint32_t>(SPEC_LANES));
  const uint32_t rem = c > skip ? c - skip : 0u;
  // positions of the tasks and of their leftovers: one scan of both counts packed into 16-bit
  // halves when the range's total fits (m_own: the caller's sum of the range's counts)
  uint32_t tot, pos, rtot = 0, rp = 0;
  if (m_own < 65536u) {
    uint32_t t2;
    const uint32_t ex = block_exclusive_scan<SEL_NT>(c | (rem << 16), cs.sm.warp_tot, &t2);
    pos = ex & 0xffffu;
    rp = ex >> 16;
    tot = t2 & 0xffffu;
    rtot = t2 >> 16;
  } else {
    pos = block_exclusive_scan<SEL_NT>(c, cs.sm.warp_tot, &tot);
    if (__syncthreads_or(rem != 0u)) rp = block_exclusive_scan<SEL_NT>(rem, cs.sm.warp_tot, &rtot);
  }
  cs.tpos[threadIdx.x] = pos;
  cs.tcnt[threadIdx.x] = c;
  if (rtot) cs.rpos[threadIdx.x] = rp;
  __syncthreads();
  LAGS_SPSTAMP(1);
  uint32_t my_gt = 0, dx = 0;
  // returns whether the entry may be selected (its weight is wanted)
  auto take = [&](float x, int32_t ix, uint32_t e) -> bool {
    const uint32_t key = Key<float>::of(x);
    sv[e] = x;
    si[e] = ix;
    dx |= key ^ key0;
    const uint32_t b = hist_bin(key, base);
    if (cut_bin != ~0u) {
      if (b < cut_bin) return false;
      if (b > cut_bin) {
        ++my_gt;
      } else {
        const uint32_t at = atomicAdd(list_n, 1u);
        if (at < BIN_LIST_MAX) list[at] = key;
      }
    }
    return true;
  };
#pragma unroll
  for (int u = 0; u < GATHER_TASKS; ++u) {
    const int tt = (warp + NW * u) * SPEC_TPW + lane / SPEC_LANES;
    const uint32_t en = static_cast<uint32_t>(lane % SPEC_LANES);
    if (tt < nt) {
      const uint32_t ct = cs.tcnt[tt];
      if (en < ct && take(g.xv[u], g.xi[u], cs.tpos[tt] + en) && vl)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(vl + g.xi[u]));  // P = 1 weight
      if (ct > SPEC_LANES && ct <= 2 * SPEC_LANES && en + SPEC_LANES < ct) {  // the rest, by the same lanes
        const int64_t src = static_cast<int64_t>(t_lo + tt) * cap + en + SPEC_LANES;
        const int32_t ix = __ldcg(cand_idx + src);
        if (take(__ldcg(cand_val + src), ix, cs.tpos[tt] + en + SPEC_LANES) && vl)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(vl + ix));  // P = 1 weight
      }
    }
  }
  LAGS_SPSTAMP(2);
  // leftovers (tasks beyond the covered ones, lists longer than 2 * SPEC_LANES): one thread per
  // entry over the scan of the remainders, GATHER_ILP loads in flight per thread (large k: a
  // 2.4 M-element layer at rho = 0.01 has ~80 candidates per task)
  LAGS_SPSTAMP(3);
  if (rtot) {
    for (uint32_t e0 = 0; e0 < rtot; e0 += SEL_NT * GATHER_ILP) {
      int tk[GATHER_ILP];
      uint32_t off[GATHER_ILP];
      float x[GATHER_ILP];
      int32_t ix[GATHER_ILP];
#pragma unroll
      for (int u = 0; u < GATHER_ILP; ++u) {
        const uint32_t e = e0 + u * SEL_NT + threadIdx.x;
        tk[u] = -1;
        if (e < rtot) {
          // the last task whose remainder starts at or before e; fixed steps, so the
          // GATHER_ILP searches interleave
          int lo = 0;
#pragma unroll
          for (int step = SEL_NT / 2; step > 0; step >>= 1)
            if (lo + step < nt && cs.rpos[lo + step] <= e) lo += step;
          tk[u] = lo;
          off[u] = (lo < COVERED ? static_cast<uint32_t>(SPEC_LANES) : 0u) + (e - cs.rpos[lo]);
          const int64_t src = static_cast<int64_t>(t_lo + lo) * cap + off[u];
          x[u] = __ldcg(cand_val + src);
          ix[u] = __ldcg(cand_idx + src);
        }
      }
#pragma unroll
      for (int u = 0; u < GATHER_ILP; ++u)
        if (tk[u] >= 0 && take(x[u], ix[u], cs.tpos[tk[u]] + off[u]) && vl)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(vl + ix[u]));  // P = 1 weight
    }
  }
  LAGS_SPSTAMP(4);
  dx = __reduce_or_sync(0xffffffffu, dx);
  if (lane == 0 && dx) atomicOr(&cs.sm.diff_acc, dx);
  my_gt = __reduce_add_sync(0xffffffffu, my_gt);
  if (gtb && lane == 0 && my_gt) atomicAdd(gtb, my_gt);
  return tot;
}

// compact_staged with V entries per thread (see below).
template <int V, typename Emit>
__device__ uint32_t compact_staged_v(uint32_t m, const SelectThreshold<uint32_t>& th, const float* sv,
                                     const int32_t* si, const float* vl, Emit emit, SelectSmem& cs,
                                     uint32_t carry_gt, uint32_t carry_eq, int32_t* oidx, float* oval) {
  static_assert(V % 4 == 0, "whole 16-byte vectors per plane and thread");
  static_assert(SEL_NT * V <= F32_BINS, "a chunk's output fits the staging arrays");
  RadixSmem<Key<float>::RB>& sm = cs.sm;
  int32_t* st_idx = reinterpret_cast<int32_t*>(sm.hist);  // free here: the threshold is known
  float* st_val = reinterpret_cast<float*>(cs.hist2);
  for (uint32_t base = 0; base < m; base += SEL_NT * V) {
    const uint32_t out0 = carry_gt + min(carry_eq, th.need_eq);  // the chunk's first output slot
    const uint32_t i0 = base + threadIdx.x * V;
    float xs[V];
#pragma unroll
    for (int q = 0; q < V / 4; ++q) {
      float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + 4 * q < m) x4 = *reinterpret_cast<const float4*>(sv + i0 + 4 * q);
      xs[4 * q] = x4.x;
      xs[4 * q + 1] = x4.y;
      xs[4 * q + 2] = x4.z;
      xs[4 * q + 3] = x4.w;
    }
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t key = i0 + v < m ? Key<float>::of(xs[v]) : 0u;
      const uint32_t hk = key & th.pmask;
      if (key != 0u) {
        if (hk > th.prefix) gtm |= 1u << v;
        else if (hk == th.prefix) eqm |= 1u << v;
      }
    }
    int32_t ixs[V];
    float ws[V];
#pragma unroll
    for (int q = 0; q < V / 4; ++q) {
      int4 ix4 = make_int4(0, 0, 0, 0);
      if (!si) ix4 = make_int4(i0 + 4 * q, i0 + 4 * q + 1, i0 + 4 * q + 2, i0 + 4 * q + 3);  // a whole layer
      else if (((gtm | eqm) >> (4 * q)) & 0xfu) ix4 = *reinterpret_cast<const int4*>(si + i0 + 4 * q);
      ixs[4 * q] = ix4.x;
      ixs[4 * q + 1] = ix4.y;
      ixs[4 * q + 2] = ix4.z;
      ixs[4 * q + 3] = ix4.w;
    }
    // the weights of the entries at or above the threshold (P = 1 update; L2-prefetched by the
    // gather), in flight across the block scan
#pragma unroll
    for (int v = 0; v < V; ++v) ws[v] = vl && (((gtm | eqm) >> v) & 1u) ? vl[ixs[v]] : 0.0f;
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
          emit(ixs[v], xs[v], ws[v]);
        }
        gt_before += g;
        eq_before += e;
      }
    }
    carry_gt += tot & 0xffffu;
    carry_eq += tot >> 16;
    __syncthreads();  // the staged pairs are complete (and warp_tot is free for the next scan)
    // the chunk's (index, value) pairs leave as coalesced runs (the per-thread emits are scattered)
    const uint32_t n_out = carry_gt + min(carry_eq, th.need_eq) - out0;
    for (uint32_t q = threadIdx.x; q < n_out; q += SEL_NT) {
      oidx[out0 + q] = st_idx[q];
      oval[out0 + q] = st_val[q];
    }
  }
  __syncthreads();  // the staging arrays are read before the callers reuse them
  return carry_gt + min(carry_eq, th.need_eq);
}

// Ordered compaction of candidates staged in shared memory (sv / si: 16-byte aligned planes in
// index order; si == nullptr: sv is a whole layer, the index is the position), 4 (8 for large
// sets: half the block scans) entries per thread read as 16-byte
// vectors per plane; vl (nullable): the layer's weights for the fused P = 1 update.  The rule and
// the result are ordered_compact_pf's: (key & pmask) > prefix, plus the first need_eq equal ones
// in index order; carry_gt / carry_eq count the lower ranks' entries.  The (index, value) pairs
// leave through shared memory as coalesced runs into oidx / oval; emit(ix, x, w) does the
// scattered residual / weight writes.  Returns the selected count (all threads).
template <typename Emit>
__device__ uint32_t compact_staged(uint32_t m, const SelectThreshold<uint32_t>& th, const float* sv, const int32_t* si,
                                   const float* vl, Emit emit, SelectSmem& cs, uint32_t carry_gt, uint32_t carry_eq,
                                   int32_t* oidx, float* oval) {
  if (m > 2u * SEL_NT * 4u) return compact_staged_v<8>(m, th, sv, si, vl, emit, cs, carry_gt, carry_eq, oidx, oval);
  return compact_staged_v<4>(m, th, sv, si, vl, emit, cs, carry_gt, carry_eq, oidx, oval);
}

// Candidate path of one layer inside one CTA.  Returns 0 on success, or why the candidate set
// cannot be proven to hold the top-k (FB_TOO_FEW / FB_OVERFLOW); the caller then runs a dense
// exact path in the same CTA.  Candidates are gathered once into shared memory (value + index,
// ascending index order) when they fit (2*m words <= smem_words), else into global scratch.
// The threshold: K1's histogram locates the bin of the k-th largest candidate and the gather lists
// that bin's keys (a handful), so one count among them resolves it exactly; a cut in the top
// (open-ended) bin or a crowded bin (ties) takes the radix select over the gathered keys instead.
constexpr int FB_TOO_FEW = 1, FB_OVERFLOW = 2;

#ifdef LAGS_DBG_STAMPS
#ifndef LAGS_DBG_J
#define LAGS_DBG_J 78
#endif
__device__ unsigned long long lags_dbg_cstamps[16];
#define LAGS_CSTAMP(i)                                           \
  do {                                                           \
    if (j == LAGS_DBG_J && threadIdx.x == 0) lags_dbg_cstamps[i] = clock64(); \
  } while (0)
#else
#define LAGS_CSTAMP(i) \
  do {                 \
  } while (0)
#endif

// The radix select over gathered candidates sv[0..m) (a cut in the open top bin, a crowded bin, or
// k >= m): out of line, the histogram cut resolves the common case.
__device__ LAGS_COLD void candidate_radix(const float* sv, uint32_t m, uint32_t k, uint32_t k2, uint32_t diff,
                                          uint32_t key0, SelectSmem& cs, SelectThreshold<uint32_t>* th,
                                          uint32_t* key2) {
  auto key_at = [=](int64_t i) { return Key<float>::of(sv[i]); };
  const uint32_t dk[2] = {diff, key0};
  radix_select_dual(key_at, m, k, k2, cs, th, key2, true, dk, true);
}

__device__ int candidate_select(int j, const lags_layer_t& L, int2 tr, FastState st, const int32_t* cand_cnt,
                                const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_val, int cap,
                                int32_t* gidx, float* gval, float* r, int32_t* idx_out, float* val_out,
                                int32_t* count_out, FastState* state, uint32_t* dyn, int smem_words, SelectSmem& cs,
                                float* vupd, const uint32_t* hl) {
  RadixSmem<Key<float>::RB>& sm = cs.sm;
  const uint32_t k = static_cast<uint32_t>(L.k);
  const int T = tr.y - tr.x;
  const bool spec = T <= SEL_NT;  // counts cached in shared memory, candidates loaded speculatively
  float* vl = vupd ? vupd + L.offset : nullptr;
  LAGS_CSTAMP(0);
  // 1. one round trip: the candidates (speculative), the histogram and the task counts
  SpecGather g;
  if (spec) spec_load(g, tr.x, T, cand_idx, cand_val, cap);
  HistRegs hr;
  if (hl) hist_load(hl, hr);
  uint32_t local = 0, over = 0;
  for (int t = tr.x + threadIdx.x; t < tr.y; t += SEL_NT) {
    const uint32_t c = static_cast<uint32_t>(__ldcg(cand_cnt + t));
    over |= c > static_cast<uint32_t>(cap) ? 1u : 0u;
    local += min(c, static_cast<uint32_t>(cap));
    if (spec) cs.tcache[t - tr.x] = c;
  }
  LAGS_CSTAMP(1);
  if (threadIdx.x == 0) {  // the gather's counters (published by the barriers below)
    sm.list_n = 0u;
    sm.gtb = 0u;  // entries above the cut bin, counted by the gather
    sm.diff_acc = 0u;
  }
  const uint32_t m = block_sum(local, sm);
  if (__syncthreads_or(over)) {
    if (hl) clear_hist_chunk(hr, const_cast<uint32_t*>(hl));
    return FB_OVERFLOW;
  }
  LAGS_CSTAMP(2);
  if (m < k && st.thr > 1u) {
    if (hl) clear_hist_chunk(hr, const_cast<uint32_t*>(hl));
    return FB_TOO_FEW;
  }
  float* data = r + L.offset;
  uint32_t cnt = 0;
  uint32_t pred = st.thr;
  const uint32_t k2 = pred_rank(st, k);
  uint32_t phases = 0;  // diagnostic: gather / select / compact cycles (units of 64, 11 bits each)
  uint32_t cut_diag = 0u;  // diagnostic (FastState.cut): 0 resolved by the cut, 2 not; bits 8.. the bin's count
  if (m > 0) {
    const long long c0 = clock64();
    const uint32_t m4 = (m + 3u) & ~3u;  // 16-byte aligned planes (the staged compaction reads vectors)
    const bool in_smem = 2u * m4 <= static_cast<uint32_t>(smem_words);
    const int64_t gbase = static_cast<int64_t>(tr.x) * cap;
    float* sv = in_smem ? reinterpret_cast<float*>(dyn) : gval + gbase;
    int32_t* si = in_smem ? reinterpret_cast<int32_t*>(dyn) + m4 : gidx + gbase;
    const uint32_t base = st.thr >> HIST_SHIFT;
    // the histogram cut (uniform): usable when the k-th candidate is in a closed bin with few keys
    HistCut hc{~0u, 0u, 0u, 0u};
    bool cut = hl != nullptr && k < m;
    if (cut) {
      hc = hist_cut(hr, cs, k, k2, m);
      cut = hc.bin < HIST_BINS - 1u && hc.in_bin <= BIN_LIST_MAX;
    }
    uint32_t* list = cs.hist2;
    if (spec) {
      spec_place(g, tr.x, T, cs.tcache, cand_idx, cand_val, cap, sv, si, vl, cs, st.thr, base, cut ? hc.bin : ~0u,
                 &sm.gtb, list, &sm.list_n, m);
    } else {
      gather_candidates(tr.x, tr.y, cand_cnt, cand_idx, cand_val, cap, sv, si, cs, st.thr, base, cut ? hc.bin : ~0u,
                        &sm.gtb, list, &sm.list_n, vl, nullptr, tr.x);
    }
    clear_cut_counters(cs);
    __syncthreads();  // the gather's counts (gtb, list_n) are complete: one uniform decision below
    const long long c1 = clock64();
    LAGS_CSTAMP(3);
    SelectThreshold<uint32_t> th;
    uint32_t key2 = 0u;
    if (cut && sm.list_n == hc.in_bin && sm.gtb == hc.above) {
      const uint32_t c = hc.in_bin, r = k - hc.above;
      if (c <= WARP_CUT_MAX) {  // every warp resolves it from the list, no barrier
        const uint32_t lane = threadIdx.x & 31;
        uint32_t kk[WARP_CUT_KEYS], oo[WARP_CUT_KEYS];
#pragma unroll
        for (int jj = 0; jj < WARP_CUT_KEYS; ++jj) {
          kk[jj] = lane + 32u * jj < c ? list[lane + 32u * jj] : 0u;
          oo[jj] = 0u;
        }
        const WarpCut wc = warp_resolve(kk, oo, c, r, 0u);
        th.prefix = wc.key;
        th.pmask = 0x7fffffffu;
        th.n_gt = hc.above + wc.gt;
        th.need_eq = r - wc.gt;
      } else {
        th = resolve_cut(list, c, r, hc.above, cs);
      }
      key2 = (base + hc.bin2) << HIST_SHIFT;  // lower edge of the k2-th candidate's bin
    } else {
      candidate_radix(sv, m, k, k2, sm.diff_acc, st.thr, cs, &th, &key2);
      cut_diag = 2u;
    }
    if (hl && k < m) cut_diag |= min(hc.in_bin, 0xffffffu) << 8;
    const long long c2 = clock64();
    auto load = [=](int64_t i, uint32_t* key, float* x, int64_t* ix) {
      *x = sv[i];
      *key = Key<float>::of(*x);
      *ix = si[i];
    };
    int32_t* oidx = idx_out + L.slot;
    float* oval = val_out + L.slot;
    LAGS_CSTAMP(4);
    if (in_smem) {  // staged: vector reads of the planes
      auto emit = [=](int32_t ix, float x, float w) {
        data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
        if (vl) vl[ix] = single_rank_update(w, x);
      };
      cnt = compact_staged(m, th, sv, si, vl, emit, cs, 0u, 0u, oidx, oval);
    } else if (vl) {  // fused P = 1 update: the weights are loaded before the compaction's scan
      auto emit = [=](uint32_t pos, int64_t, int64_t ix, float x, float w) {
        oidx[pos] = static_cast<int32_t>(ix);
        oval[pos] = x;
        data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
        vl[ix] = single_rank_update(w, x);
      };
      cnt = ordered_compact_pf<uint32_t, float>(m, th, load, emit, sm, 0u, 0u,
                                                [=](int64_t, int64_t ix) { return vl[ix]; });
    } else {
      auto emit = [=](uint32_t pos, int64_t, int64_t ix, float x) {
        oidx[pos] = static_cast<int32_t>(ix);
        oval[pos] = x;
        data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
      };
      cnt = ordered_compact<uint32_t, float>(m, th, load, emit, sm);
    }
    LAGS_CSTAMP(5);
    LAGS_CSTAMP(6);
    const long long c3 = clock64();
    auto q = [](long long c) { return static_cast<uint32_t>(min(c >> 6, 2047ll)); };
    phases = q(c1 - c0) | (q(c2 - c1) << 11) | (q(c3 - c2) << 22);
#ifdef LAGS_DBG_SELECT
    phases = sm.dbg;
#endif
    pred = next_threshold(st, m, k, k2, th.prefix, key2);
  }
  if (hl) clear_hist_chunk(hr, const_cast<uint32_t*>(hl));  // the cut is consumed (every thread read its own)
  if (threadIdx.x == 0) {
    FastState ns = candidate_state(st, pred, m, k, phases);
    ns.cut = cut_diag;
    state[j] = ns;
    count_out[j] = static_cast<int32_t>(cnt);
  }
  __syncthreads();
  LAGS_CSTAMP(7);
  return 0;
}

// Dense exact path of one big layer inside one CTA (first call of a layer, failed prediction or
// forced exact mode): radix select of the k-th key and, in the same passes, of the next
// prediction rank over r, then an ordered compaction that zeroes the selected residuals.
__device__ LAGS_COLD void dense_fallback_select(int j, const lags_layer_t& L, FastState st, float* r, int32_t* idx_out,
                                      float* val_out, int32_t* count_out, FastState* state, bool force_exact,
                                      int why, SelectSmem& cs, float* vupd) {
  float* data = r + L.offset;
  const int64_t d = L.dim;
  const uint32_t k = static_cast<uint32_t>(L.k);
  // a failed prediction widens the candidate margin (too few) or narrows it (task overflow)
  const bool predicted = st.thr != 0u && !force_exact;
  const float pf_next = !predicted ? pred_factor(st)
                                   : (why == FB_OVERFLOW ? 0.5f * pred_factor(st) : 2.0f * pred_factor(st));
  const int64_t pk = static_cast<int64_t>(fmaxf(pf_next, 1.0f) * static_cast<float>(k));
  const uint32_t k2 = static_cast<uint32_t>(pk < d ? (pk > k ? pk : k + 1) : d);
  auto key_at = [=](int64_t i) { return Key<float>::of(__ldcg(data + i)); };
  SelectThreshold<uint32_t> th;
  uint32_t key2;
  radix_select_dual(key_at, d, k, k2, cs, &th, &key2, false);
  auto load = [=](int64_t i, uint32_t* key, float* x, int64_t* ix) {
    *x = __ldcg(data + i);
    *key = Key<float>::of(*x);
    *ix = i;
  };
  int32_t* oidx = idx_out + L.slot;
  float* oval = val_out + L.slot;
  float* vl = vupd ? vupd + L.offset : nullptr;
  auto emit = [=](uint32_t pos, int64_t i, int64_t, float x) {
    oidx[pos] = static_cast<int32_t>(i);
    oval[pos] = x;
    data[i] = sent_residual(x);  // acc - acc (R: training.py:252)
  };
  const uint32_t cnt = ordered_compact<uint32_t, float>(d, th, load, emit, cs.sm);
  if (vl) apply_single_rank_updates(vl, oidx, oval, cnt);
  if (threadIdx.x == 0) {
    count_out[j] = static_cast<int32_t>(cnt);
    FastState ns = st;
    ns.thr = max(key2, 1u);
    ns.fallbacks += predicted ? 1u : 0u;
    ns.last_cands = 0;
    ns.calls += 1;
    ns.pf256 = pf_encode(pf_next);
    state[j] = ns;
  }
}

// Exact threshold of the k largest keys of a tiny layer staged in shared memory (d <= TINY_LAYER,
// small k, no prediction wanted): rounds of a block-wide (largest key below the bound, its count)
// from registers -- one barrier per round, at most k rounds, ~640 cycles each -- instead of three
// 4096-bin radix passes (a 4096-element layer's radix select took ~9.5 k cycles).  Ties are left to the
// compaction (the first need_eq equal keys in index order).  All threads.
constexpr uint32_t SMALL_K_ROUNDS = 16;  // k up to this takes the rounds
__device__ SelectThreshold<uint32_t> small_k_threshold(const float* sv, uint32_t d, uint32_t k, SelectSmem& cs) {
  constexpr int NW = SEL_NT / 32, PT = (TINY_LAYER + SEL_NT - 1) / SEL_NT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t keys[PT];
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    const uint32_t i = threadIdx.x + q * SEL_NT;
    keys[q] = i < d ? Key<float>::of(sv[i]) : 0u;
  }
  uint32_t* red = cs.sm.hist;  // (max, count) per warp, double-buffered by round parity
  SelectThreshold<uint32_t> th;
  th.pmask = 0x7fffffffu;
  uint32_t bound = 0xffffffffu, taken = 0;
  for (uint32_t round = 0;; ++round) {
    uint32_t open[PT], mx = 0u, c = 0u;
#pragma unroll
    for (int q = 0; q < PT; ++q) {
      open[q] = keys[q] < bound ? keys[q] : 0u;
      mx = max(mx, open[q]);
    }
#pragma unroll
    for (int q = 0; q < PT; ++q) c += open[q] == mx ? 1u : 0u;
    const uint32_t wmx = __reduce_max_sync(0xffffffffu, mx);
    const uint32_t wc = __reduce_add_sync(0xffffffffu, mx == wmx ? c : 0u);
    uint32_t* buf = red + (round & 1u) * 2 * NW;
    if (lane == 0) {
      buf[warp] = wmx;
      buf[NW + warp] = wc;
    }
    __syncthreads();
    // the warps' pairs, one per lane
    const uint32_t v = lane < NW ? buf[lane] : 0u, n = lane < NW ? buf[NW + lane] : 0u;
    const uint32_t bmx = __reduce_max_sync(0xffffffffu, v);
    const uint32_t bc = __reduce_add_sync(0xffffffffu, v == bmx ? n : 0u);
    if (bmx == 0u) {  // fewer than k nonzero keys: every nonzero one (zeros never selected)
      th.prefix = 0u;
      th.n_gt = taken;
      th.need_eq = 0u;
      return th;
    }
    if (taken + bc >= k) {
      th.prefix = bmx;
      th.n_gt = taken;
      th.need_eq = k - taken;
      return th;
    }
    taken += bc;
    bound = bmx;
  }
}

// Dense exact path of a small layer (d <= SMALL_LAYER): staged once in shared memory, so the
// radix passes and the compaction read shared memory; the same dual-rank select predicts the
// next candidate threshold (small layers then take the candidate path like the big ones).
__device__ LAGS_COLD void small_fallback_select(int j, const lags_layer_t& L, FastState st, float* r, int32_t* idx_out,
                                      float* val_out, int32_t* count_out, FastState* state, bool force_exact, int why,
                                      SelectSmem& cs, float* vupd, float* sv, bool predict) {
  float* data = r + L.offset;
  const int64_t d = L.dim;
  const uint32_t k = static_cast<uint32_t>(L.k);
  const long long c0 = clock64();
  if ((reinterpret_cast<uintptr_t>(data) & 15u) == 0u) {
    const float4* d4 = reinterpret_cast<const float4*>(data);
    float4* s4 = reinterpret_cast<float4*>(sv);
    const int64_t n4 = d >> 2;
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < n4; i += SEL_NT) s4[i] = __ldcg(d4 + i);
    for (int64_t i = 4 * n4 + threadIdx.x; i < d; i += SEL_NT) sv[i] = __ldcg(data + i);
  } else {
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < d; i += SEL_NT) sv[i] = __ldcg(data + i);
  }
  __syncthreads();
  const bool predicted = st.thr != 0u && !force_exact;
  const float pf_next = !predicted ? pred_factor(st)
                                   : (why == FB_OVERFLOW ? 0.5f * pred_factor(st) : 2.0f * pred_factor(st));
  const int64_t pk = static_cast<int64_t>(fmaxf(pf_next, 1.0f) * static_cast<float>(k));
  const uint32_t k2 = static_cast<uint32_t>(pk < d ? (pk > k ? pk : k + 1) : d);
  auto key_at = [=](int64_t i) { return Key<float>::of(sv[i]); };
  SelectThreshold<uint32_t> th;
  uint32_t key2;
  const long long c1 = clock64();
  if (!predict && d <= TINY_LAYER && k <= SMALL_K_ROUNDS) {
    th = small_k_threshold(sv, static_cast<uint32_t>(d), k, cs);
    key2 = 0u;  // no prediction: the layer stays on this path
  } else {
    radix_select_dual(key_at, d, k, k2, cs, &th, &key2, true);
  }
  const long long c2 = clock64();
  int32_t* oidx = idx_out + L.slot;
  float* oval = val_out + L.slot;
  float* vl = vupd ? vupd + L.offset : nullptr;
  auto emit = [=](int32_t i, float x, float w) {
    data[i] = sent_residual(x);  // acc - acc (R: training.py:252)
    if (vl) vl[i] = single_rank_update(w, x);
  };
  // staged compaction over the whole layer (positions are the indices), weights loaded per chunk
  const uint32_t cnt = compact_staged(static_cast<uint32_t>(d), th, sv, nullptr, vl, emit, cs, 0u, 0u, oidx, oval);
  if (threadIdx.x == 0) {
    count_out[j] = static_cast<int32_t>(cnt);
    FastState ns = st;
    ns.thr = predict ? max(key2, 1u) : 0u;  // 1: every nonzero entry is a candidate (layer mostly zeros)
    ns.fallbacks += predicted ? 1u : 0u;
    ns.last_cands = 0;
    ns.calls += 1;
    ns.pf256 = pf_encode(pf_next);
    auto q64 = [](long long c) { return static_cast<uint32_t>(min(c >> 6, 2047ll)); };
    ns.reserved = q64(c1 - c0) | (q64(c2 - c1) << 11) | (q64(clock64() - c2) << 22);  // load, select, compact
    state[j] = ns;
  }
}

// Exact top-k of a tiny layer (d <= TINY_LAYER, k <= WARP_TOPK) by ONE warp, no barriers: every
// lane keeps its WARP_TOPK largest (|x| key, index) of a lane-strided scan in registers (an
// insertion chain; on equal keys the earlier = lower index stays ahead), then k rounds of a warp
// argmax over the lanes' heads (key, then lower index) take the layer's top-k; zero keys are
// never selected (R: sparsify.py:84-90).  Output in ascending index order, residual zeroed, the
// optional fused P = 1 update applied.
#ifndef LAGS_WARP_B
#define LAGS_WARP_B 2  // small unrolls: the code footprint (instruction cache) dominates this path
#endif
#ifndef LAGS_WARP_TOPK
#define LAGS_WARP_TOPK 8
#endif
constexpr int WARP_TOPK = LAGS_WARP_TOPK;
#ifndef LAGS_WARP_MAX_DIM
#define LAGS_WARP_MAX_DIM 2048
#endif
constexpr int WARP_MAX_DIM = LAGS_WARP_MAX_DIM;  // larger tiny layers: a whole CTA (persistent role)

__device__ void warp_topk_layer(int j, const lags_layer_t& L, FastState* state, float* r, int32_t* idx_out,
                                float* val_out, int32_t* count_out, float* vupd, uint32_t t_launch) {
  const int lane = threadIdx.x & 31;
  const uint32_t t_start = globaltimer_lo();
  const long long c0 = clock64();
  float* data = r + L.offset;
  float val[WARP_TOPK];
  int32_t ix[WARP_TOPK];
#pragma unroll
  for (int q = 0; q < WARP_TOPK; ++q) {
    val[q] = 0.0f;
    ix[q] = 0x7fffffff;
  }
  const int d = static_cast<int>(L.dim);
  const uint32_t k = static_cast<uint32_t>(L.k);
  const bool vec = (reinterpret_cast<uintptr_t>(data) & 15u) == 0u;
  const float4* d4 = reinterpret_cast<const float4*>(data);
  const int n4 = vec ? d >> 2 : 0;
  // every lane visits its elements in ascending index order (the tie rule needs it); the loads
  // of a batch are issued together (LAGS_WARP_B x 16 B per lane in flight)
  constexpr int B = LAGS_WARP_B;
  auto scan = [&](auto&& visit) {
    for (int q0 = lane; q0 < n4; q0 += 32 * B) {
      float4 x[B];
#pragma unroll
      for (int u = 0; u < B; ++u) x[u] = q0 + 32 * u < n4 ? __ldcg(d4 + q0 + 32 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int e = 4 * (q0 + 32 * u);
        visit(x[u].x, e);
        visit(x[u].y, e + 1);
        visit(x[u].z, e + 2);
        visit(x[u].w, e + 3);
      }
    }
    for (int i0 = 4 * n4 + lane; i0 < d; i0 += 32 * B) {
      float x[B];
#pragma unroll
      for (int u = 0; u < B; ++u) x[u] = i0 + 32 * u < d ? __ldcg(data + i0 + 32 * u) : 0.0f;
#pragma unroll
      for (int u = 0; u < B; ++u) visit(x[u], i0 + 32 * u);
    }
  };
  // pass 1: a warp-wide lower bound of the k-th largest key -- the k-th largest of the 32 lane
  // maxima (at least k elements reach it); zero keys are never selected
  uint32_t lmax = 0;
  scan([&](float x, int) { lmax = max(lmax, Key<float>::of(x)); });
  uint32_t bound = 0, m = lmax;
  for (uint32_t q = 0; q < k && q < 32u; ++q) {
    bound = __reduce_max_sync(0xffffffffu, m);
    const unsigned who = __ballot_sync(0xffffffffu, m == bound);
    if (lane == __ffs(who) - 1) m = 0;
  }
  bound = max(bound, 1u);
  // pass 2: each lane keeps its WARP_TOPK largest entries at or above the bound (rarely more
  // than a few), an insertion chain where equal keys keep the earlier = lower index ahead
  scan([&](float cv, int ci) {
    if (Key<float>::of(cv) >= bound && Key<float>::of(cv) > Key<float>::of(val[WARP_TOPK - 1])) {
#pragma unroll
      for (int q = 0; q < WARP_TOPK; ++q) {
        if (Key<float>::of(cv) > Key<float>::of(val[q])) {
          const float tv = val[q];
          const int32_t ti = ix[q];
          val[q] = cv;
          ix[q] = ci;
          cv = tv;
          ci = ti;
        }
      }
    }
  });
  const long long c1 = clock64();
  // merge: round q's winner is kept by lane q
  float my_val = 0.0f;
  int32_t my_ix = 0x7fffffff;
  uint32_t cnt = 0;
  for (uint32_t q = 0; q < k; ++q) {
    const uint32_t key = Key<float>::of(val[0]);
    unsigned long long best = (static_cast<unsigned long long>(key) << 32) | static_cast<uint32_t>(~ix[0]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if ((best >> 32) == 0ull) break;  // no nonzero key left
    const int32_t wi = static_cast<int32_t>(~static_cast<uint32_t>(best));
    const bool mine = key == static_cast<uint32_t>(best >> 32) && ix[0] == wi;
    const unsigned wl = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    const float wv = __shfl_sync(0xffffffffu, val[0], wl);
    if (lane == static_cast<int>(q)) {
      my_val = wv;
      my_ix = wi;
    }
    if (mine) {  // pop the head
#pragma unroll
      for (int t = 0; t + 1 < WARP_TOPK; ++t) {
        val[t] = val[t + 1];
        ix[t] = ix[t + 1];
      }
      val[WARP_TOPK - 1] = 0.0f;
      ix[WARP_TOPK - 1] = 0x7fffffff;
    }
    ++cnt;
  }
  const long long c2 = clock64();
  // ascending index order: a winner's position = winners with a smaller index
  uint32_t pos = 0;
  for (uint32_t q = 0; q < cnt; ++q) pos += __shfl_sync(0xffffffffu, my_ix, q) < my_ix ? 1u : 0u;
  if (static_cast<uint32_t>(lane) < cnt) {
    idx_out[L.slot + pos] = my_ix;
    val_out[L.slot + pos] = my_val;
    data[my_ix] = sent_residual(my_val);  // acc - acc (R: training.py:252)
    if (vupd) vupd[L.offset + my_ix] = single_rank_update(vupd[L.offset + my_ix], my_val);
  }
  if (lane == 0) {
    const long long c3 = clock64();
    auto q64 = [](long long c) { return static_cast<uint32_t>(min(c >> 6, 2047ll)); };
    count_out[j] = static_cast<int32_t>(cnt);
    FastState ns = state[j];
    ns.thr = 0u;
    ns.last_cands = 0u;
    ns.calls += 1;
    ns.path = 0u;
    ns.cycles = static_cast<uint32_t>(c3 - c0);
    ns.reserved = q64(c1 - c0) | (q64(c2 - c1) << 11) | (q64(c3 - c2) << 22);
    ns.t_start = t_start;
    ns.t_end = globaltimer_lo();
    ns.t_launch = t_launch;
    state[j] = ns;
  }
}

// Selection of layer j by the whole CTA (all paths), with its diagnostic timeline entry.
__device__ void select_layer(int j, const lags_layer_t* __restrict__ layers, const int2* __restrict__ layer_tasks,
                             FastState* state, const int32_t* cand_cnt, const int32_t* cand_idx, const float* cand_val,
                             int cap, int32_t* gidx, float* gval, float* r, int32_t* idx_out, float* val_out,
                             int32_t* count_out, uint32_t* skeys, int smem_keys, int force_exact, SelectSmem& cs,
                             float* vupd, uint32_t t_launch, uint32_t* hist) {
  const uint32_t t_start = globaltimer_lo();
  LAGS_CSTAMP(8);
  const lags_layer_t L = layers[j];
  const FastState st = state[j];
  const long long t_begin = clock64();
  const bool tiny = L.dim <= TINY_LAYER;
  // K1 counted this layer's candidates into its histogram iff it had a threshold
  uint32_t* hl = hist && st.thr != 0u ? hist + static_cast<int64_t>(j) * HIST_BINS : nullptr;
  const int why = (force_exact || st.thr == 0u || tiny)
                      ? FB_TOO_FEW
                      : candidate_select(j, L, layer_tasks[j], st, cand_cnt, cand_idx, cand_val, cap, gidx, gval, r,
                                         idx_out, val_out, count_out, state, skeys, smem_keys, cs, vupd, hl);
  // the candidate set cannot be proven to hold the top-k: dense exact path, same CTA (small
  // layers staged in shared memory; SMALL_LAYER <= the staging capacity)
  if (why && L.dim <= SMALL_LAYER)
    small_fallback_select(j, L, st, r, idx_out, val_out, count_out, state, force_exact != 0, why, cs, vupd,
                          reinterpret_cast<float*>(skeys), !tiny);
  else if (why)
    dense_fallback_select(j, L, st, r, idx_out, val_out, count_out, state, force_exact != 0, why, cs, vupd);
  const uint32_t path = why ? (L.dim <= SMALL_LAYER ? 0u : 2u) : 1u;
  __syncthreads();
  // candidate_select clears the histogram it read; a forced exact call never read it
  if (hl && force_exact) zero_hist(hl, 0, HIST_BINS);
  if (threadIdx.x == 0) {
    state[j].cycles = static_cast<uint32_t>(clock64() - t_begin);
    state[j].path = path;
    state[j].t_start = t_start;
    state[j].t_end = globaltimer_lo();
    state[j].t_launch = t_launch;
  }
}

}  // namespace lags
