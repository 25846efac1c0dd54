// Selection of the largest layers by a thread-block cluster (CLUSTER CTAs, distributed shared
// memory).  One CTA per layer made the handful of ~2 M-element ResNet-50 layers the critical path
// of the selection; here the CTAs of a cluster each own a contiguous quarter of the layer's K1
// task lists (= a contiguous index range):
//   1. every CTA reads ALL of the layer's task counts and derives the candidate total m, every
//      rank's share and its own offset (no exchange);
//   2. every CTA reads K1's histogram of the layer's candidate keys and locates the bin of the k-th
//      largest (the same cut everywhere), then gathers its candidates (value, index) into its own
//      shared memory, counting those above the cut bin and listing the cut bin's keys (a handful);
//      it pushes that count and list into every CTA (DSMEM); one cluster barrier;
//   3. every CTA resolves the exact threshold from the listed keys and the lower ranks' carried
//      counts itself -- nothing crosses CTAs after the barrier.  A cut in the open top bin or a
//      crowded bin (ties) takes the distributed radix select instead: per-pass histograms summed
//      by rank 0 over DSMEM, threshold and counts exchanged;
//   4. every CTA compacts its own range in order with the carried counts (global output
//      positions), zeroes the selected residuals and applies the optional fused P = 1 update.
// Results are identical to the single-CTA candidate path (same keys, same order, same rule).
#pragma once
#include <cooperative_groups.h>

#include "lags_fast.cuh"

namespace lags {

#ifndef LAGS_CLUSTER
#define LAGS_CLUSTER 4
#endif
#ifndef LAGS_CLUSTER_MIN_K
#define LAGS_CLUSTER_MIN_K 512
#endif
constexpr int CLUSTER = LAGS_CLUSTER;              // CTAs per cluster layer
constexpr int CLUSTER_MIN_K = LAGS_CLUSTER_MIN_K;  // layers with at least this k (and > SMALL_LAYER) use clusters

// Execution-only cluster barrier: no release/acquire (cluster.sync()'s arrive is a release, which
// waits for every earlier global store of the thread to drain).  For the barriers that only keep a
// CTA resident while its peers finish reading its shared memory -- reads whose values the peers
// have already consumed before arriving.
__device__ __forceinline__ void cluster_sync_exec() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// -DLAGS_DBG_STAMPS: clock64 / globaltimer at the phase boundaries of the first cluster layer,
// per rank (read back by lags_dbg_stamps_read; diagnostic builds only).
#ifdef LAGS_DBG_STAMPS
__device__ unsigned long long lags_dbg_stamps[CLUSTER][2][24];
#define LAGS_STAMP(i)                                                   \
  do {                                                                  \
    if (blockIdx.x < CLUSTER && threadIdx.x == 0) {                     \
      lags_dbg_stamps[blockIdx.x][0][i] = clock64();                    \
      unsigned long long g_;                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));            \
      lags_dbg_stamps[blockIdx.x][1][i] = g_;                           \
    }                                                                   \
  } while (0)
#else
#define LAGS_STAMP(i) \
  do {                \
  } while (0)
#endif

struct ClusterShared {
  uint32_t gt, eq;           // distributed mode: this CTA's compaction counts
  uint32_t prefix, pmask, n_gt, need_eq, key2;  // distributed mode, rank 0: the threshold
  uint32_t qsum[CLUSTER];    // the ranks' candidate counts (every CTA computes all of them)
  uint32_t gtb[CLUSTER];     // histogram cut: every rank's count above the cut bin (pushed)
  uint32_t lc[CLUSTER];      //   and its keys in the cut bin (pushed)
  uint32_t lists[CLUSTER][BIN_LIST_MAX];
};

// Dual-rank radix select over a cluster's candidates when every CTA holds only its own keys
// (sv[0..mr)): per pass every CTA histograms its keys, rank 0 adds the CLUSTER histograms over
// DSMEM and resolves the bins of both ranks (radix_select_dual's rule), every CTA reads the
// digits back -- two cluster barriers per pass, no key moves between CTAs.  Same result as
// radix_select_dual over all m keys.  Called by every thread of every CTA of the cluster.
struct ClusterRadix {
  uint32_t bin[2], above[2], in_bin[2];
  uint32_t diff;
};

__device__ LAGS_COLD void cluster_radix_select_dual(cooperative_groups::cluster_group& cluster, int rank, const float* sv,
                                          uint32_t mr, uint32_t m, uint32_t key0, uint32_t k, uint32_t k2,
                                          SelectSmem& cs, ClusterRadix& cr, SelectThreshold<uint32_t>* th_out,
                                          uint32_t* key2_out) {
  constexpr int RB = Key<float>::RB;
  constexpr uint32_t FULL = 0x7fffffffu;
  RadixSmem<RB>& sm = cs.sm;
  uint32_t diff = 0;
  for (uint32_t i = threadIdx.x; i < mr; i += SEL_NT) diff |= Key<float>::of(sv[i]) ^ key0;
  diff = block_or<uint32_t, RB>(diff, sm);
  if (threadIdx.x == 0) cr.diff = diff;
  cluster.sync();
  diff = 0;
  for (int q = 0; q < CLUSTER; ++q) diff |= cluster.map_shared_rank(&cr, q)->diff;
  uint32_t prefix[2], pmask[2];
  uint32_t rank_[2] = {k < m ? k : m, k2 < m ? k2 : m};
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
      cs.hist2[b] = 0;
    }
    __syncthreads();
    const uint32_t dmask = (1u << width) - 1u;
    for (uint32_t i = threadIdx.x; i < mr; i += SEL_NT) {
      const uint32_t key = Key<float>::of(sv[i]);
      const uint32_t bin = (key >> shift) & dmask;
      if (!done[0] && (key & pmask[0]) == prefix[0]) atomicAdd(&sm.hist[bin], 1u);
      if (second && (key & pmask[1]) == prefix[1]) atomicAdd(&cs.hist2[bin], 1u);
    }
    __syncthreads();
    cluster.sync();  // every CTA's histograms are complete
    if (rank == 0) {
      const uint32_t* rh[CLUSTER];
      const uint32_t* rh2[CLUSTER];
      for (int q = 1; q < CLUSTER; ++q) {
        rh[q] = cluster.map_shared_rank(sm.hist, q);
        rh2[q] = cluster.map_shared_rank(cs.hist2, q);
      }
      for (int b = threadIdx.x; b < F32_BINS; b += SEL_NT) {
        uint32_t h = sm.hist[b], h2 = second ? cs.hist2[b] : 0u;
#pragma unroll
        for (int q = 1; q < CLUSTER; ++q) {
          h += rh[q][b];
          if (second) h2 += rh2[q][b];
        }
        sm.hist[b] = h;
        if (second) cs.hist2[b] = h2;
      }
      __syncthreads();
      for (int q = 0; q < 2; ++q) {
        if (done[q]) continue;
        uint32_t bin, above, in_bin;
        find_bin<RB>(sm, rank_[q], &bin, &above, &in_bin, (q == 0 || same) ? sm.hist : cs.hist2);
        if (threadIdx.x == 0) {
          cr.bin[q] = bin;
          cr.above[q] = above;
          cr.in_bin[q] = in_bin;
        }
      }
    }
    cluster.sync();  // rank 0's digits are visible; the histograms are no longer read remotely
    const ClusterRadix* r0 = cluster.map_shared_rank(&cr, 0);
    for (int q = 0; q < 2; ++q) {
      if (done[q]) continue;
      const uint32_t bin = r0->bin[q], above = r0->above[q], in_bin = r0->in_bin[q];
      prefix[q] |= bin << shift;
      pmask[q] |= dmask << shift;
      rank_[q] -= above;
      if (q == 0) n_gt0 += above;
      if (shift == 0 || (in_bin == rank_[q] && prefix[q] != 0u)) done[q] = true;
    }
    const int ns = shift > RB ? shift - RB : 0;
    width = shift - ns;
    shift = ns;
  }
  if (k >= m) {  // every nonzero key is selected
    th_out->prefix = 0u;
    th_out->pmask = 0xffffffffu;
    th_out->n_gt = 0;
    th_out->need_eq = 0;
  } else {
    th_out->prefix = prefix[0];
    th_out->pmask = pmask[0];
    th_out->n_gt = n_gt0;
    th_out->need_eq = prefix[0] == 0u ? 0u : rank_[0];
  }
  *key2_out = prefix[1];
}

// One layer by the CTA's cluster (all CLUSTER CTAs call this with the same j).
__device__ void cluster_select_layer(int j, const lags_layer_t* __restrict__ layers,
                                     const int2* __restrict__ layer_tasks, FastState* state,
                                     const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_idx,
                                     const float* __restrict__ cand_val, int cap, int32_t* gidx, float* gval, float* r,
                                     int32_t* idx_out, float* val_out, int32_t* count_out, int smem_words,
                                     int force_exact, float* vupd, uint32_t* dyn, SelectSmem& cs, ClusterShared& csh,
                                     ClusterRadix& cr, uint32_t t_launch, uint32_t* hist, bool dry = false,
                                     const PeerPush* pp = nullptr, uint32_t epoch = 0u) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t t_start = globaltimer_lo();
  const long long t_begin = clock64();
  const int rank = static_cast<int>(cluster.block_rank());
  const lags_layer_t L = layers[j];
  const int2 tr = layer_tasks[j];
  const FastState st = state[j];
  const uint32_t k = static_cast<uint32_t>(L.k);
  const int T = tr.y - tr.x;
  const int t_lo = tr.x + static_cast<int>((static_cast<int64_t>(T) * rank) / CLUSTER);
  const int t_hi = tr.x + static_cast<int>((static_cast<int64_t>(T) * (rank + 1)) / CLUSTER);
  // K1 counted this layer's candidates into its histogram iff it had a threshold
  uint32_t* hl = hist && st.thr != 0u ? hist + static_cast<int64_t>(j) * HIST_BINS : nullptr;
  // every CTA of the cluster must be running before any remote shared-memory access: arrive now,
  // wait just before the first remote store (the loads below overlap the barrier)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  LAGS_STAMP(0);
  // 1. one round trip: the own tasks' candidates (speculative, see spec_load), the histogram (every
  // CTA its own copy) and ALL of the layer's task counts (one load per thread for layers up to
  // SEL_NT tasks), from which every CTA derives m, the ranks' sums and its own offset
  const int nt_own = t_hi - t_lo;
  // counts cached in shared memory, candidates loaded speculatively (a 2.36 M-element layer has
  // 576 tasks of K1's CTA form)
  const bool spec = T <= 2 * SEL_NT && nt_own <= SEL_NT;
  SpecGather g;
  if (spec) spec_load(g, t_lo, nt_own, cand_idx, cand_val, cap);
  HistRegs hr;
  if (hl) hist_load(hl, hr);  // every CTA its own copy
  int bnd[CLUSTER + 1];
#pragma unroll
  for (int q = 0; q <= CLUSTER; ++q) bnd[q] = tr.x + static_cast<int>((static_cast<int64_t>(T) * q) / CLUSTER);
  if (threadIdx.x < CLUSTER) csh.qsum[threadIdx.x] = 0u;
  uint32_t qs[CLUSTER];
#pragma unroll
  for (int q = 0; q < CLUSTER; ++q) qs[q] = 0u;
  uint32_t over = 0;
  for (int t = tr.x + threadIdx.x; t < tr.y; t += SEL_NT) {
    const uint32_t c = static_cast<uint32_t>(__ldcg(cand_cnt + t));
    over |= c > static_cast<uint32_t>(cap) ? 1u : 0u;
    if (spec) cs.tcache[t - tr.x] = c;
    const uint32_t cc = min(c, static_cast<uint32_t>(cap));
#pragma unroll
    for (int q = 0; q < CLUSTER; ++q) qs[q] += (t >= bnd[q] && t < bnd[q + 1]) ? cc : 0u;
  }
  LAGS_STAMP(1);
  __syncthreads();  // qsum zeroed
#pragma unroll
  for (int q = 0; q < CLUSTER; ++q) {
    const uint32_t w = __reduce_add_sync(0xffffffffu, qs[q]);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(&csh.qsum[q], w);
  }
  if (threadIdx.x == 0) {  // the gather's counters (published by the barrier below)
    cs.sm.list_n = 0u;
    cs.sm.gtb = 0u;
    cs.sm.diff_acc = 0u;
  }
  const uint32_t over_any = __syncthreads_or(over) ? 1u : 0u;
  LAGS_STAMP(2);
  uint32_t m = 0, pre = 0, m_max = 0;
  uint32_t rpre[CLUSTER + 1];  // prefix of the ranks' candidate counts
  rpre[0] = 0;
#pragma unroll
  for (int q = 0; q < CLUSTER; ++q) {
    const uint32_t mq = csh.qsum[q];
    if (q < rank) pre += mq;
    m += mq;
    m_max = max(m_max, mq);
    rpre[q + 1] = rpre[q] + mq;
  }
  const uint32_t mr = csh.qsum[rank];
  // own values + indices
  const uint32_t mx4 = (m_max + 3u) & ~3u;  // 16-byte aligned planes (the staged compaction reads vectors)
  const bool fits = 2ull * mx4 <= static_cast<uint64_t>(smem_words);
  int why = 0;
  if (force_exact || st.thr == 0u) why = FB_TOO_FEW;
  else if (over_any) why = FB_OVERFLOW;
  else if (m < k && st.thr > 1u) why = FB_TOO_FEW;
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // all CTAs of the cluster are running
  LAGS_STAMP(3);
  if (why || !fits || m == 0) {  // uniform across the cluster; rank 0 finishes the layer alone
    if (rank == 0) {  // (no shared memory of another CTA was touched: the others just leave)
      if (why) {
        dense_fallback_select(j, L, st, r, idx_out, val_out, count_out, state, force_exact != 0, why, cs, vupd);
      } else {  // too many candidates for the cluster's shared memory, or none: one-CTA path
        candidate_select(j, L, tr, st, cand_cnt, cand_idx, cand_val, cap, gidx, gval, r, idx_out, val_out, count_out,
                         state, dyn, smem_words, cs, vupd, hl);
      }
      __syncthreads();
      if (pp) {  // the whole layer: this CTA wrote it
        const int c = count_out[j];
        peer_copy(*pp, epoch, idx_out, val_out, L.slot, 0u, static_cast<uint32_t>(c), j, c, threadIdx.x, SEL_NT);
      }
      if (hl) zero_hist(hl, 0, HIST_BINS);
      if (threadIdx.x == 0) {
        state[j].cycles = static_cast<uint32_t>(clock64() - t_begin);
        state[j].path = why ? 2u : 1u;
        state[j].t_start = t_start;
        state[j].t_end = globaltimer_lo();
        state[j].t_launch = t_launch;
      }
    }
    return;
  }
  // 2. the histogram cut (every CTA the same, from its own copy), then the gather of the own
  // quarter: values at [0, mr), indices at [m_max, m_max + mr) of dyn; entries above the cut bin
  // are counted and the cut bin's keys listed on the way
  const long long c0 = clock64();
  const uint32_t k2 = pred_rank(st, k);
  const uint32_t base = st.thr >> HIST_SHIFT;
  HistCut hc{~0u, 0u, 0u, 0u};
  bool cut = hl != nullptr && k < m;
  if (cut) {
    hc = hist_cut(hr, cs, k, k2, m);
    cut = hc.bin < HIST_BINS - 1u && hc.in_bin <= BIN_LIST_MAX;
  }
  LAGS_STAMP(4);
  float* sv = reinterpret_cast<float*>(dyn);
  int32_t* si = reinterpret_cast<int32_t*>(dyn + mx4);
  if (spec) {
    spec_place(g, t_lo, nt_own, cs.tcache + (t_lo - tr.x), cand_idx, cand_val, cap, sv, si,
               vupd ? vupd + L.offset : nullptr, cs, st.thr, base, cut ? hc.bin : ~0u, &cs.sm.gtb, cs.hist2,
               &cs.sm.list_n, mr);
  } else {
    gather_candidates(t_lo, t_hi, cand_cnt, cand_idx, cand_val, cap, sv, si, cs, st.thr, base, cut ? hc.bin : ~0u,
                      &cs.sm.gtb, cs.hist2, &cs.sm.list_n, vupd ? vupd + L.offset : nullptr, nullptr, tr.x);
  }
  __syncthreads();
  LAGS_STAMP(5);
  if (cut) {  // push the own count above the cut and the cut bin's keys into every CTA
    const uint32_t lc = min(cs.sm.list_n, BIN_LIST_MAX), per = lc + 1;
    for (uint32_t e = threadIdx.x; e < CLUSTER * per; e += SEL_NT) {
      ClusterShared* o = cluster.map_shared_rank(&csh, static_cast<int>(e / per));
      const uint32_t i = e % per;
      if (i < lc) {
        o->lists[rank][i] = cs.hist2[i];
      } else {
        o->gtb[rank] = cs.sm.gtb;
        o->lc[rank] = cs.sm.list_n;
      }
    }
  }
  LAGS_STAMP(6);
  cluster.sync();  // the pushed counts and lists are visible (the histogram copies are consumed)
  LAGS_STAMP(7);
  const long long c1 = clock64();
  SelectThreshold<uint32_t> th;
  uint32_t key2 = 0u;
  uint32_t cg0 = 0, ce0 = 0;
  bool resolved = false;
  if (k >= m) {  // every candidate (all nonzero: keys >= the threshold >= 1) is selected
    th.prefix = 0u;
    th.pmask = 0xffffffffu;
    th.n_gt = 0u;
    th.need_eq = 0u;
    cg0 = pre;
    resolved = true;
  } else if (cut) {
    uint32_t off[CLUSTER + 1], gsum = 0;
    off[0] = 0;
#pragma unroll
    for (int q = 0; q < CLUSTER; ++q) {
      off[q + 1] = off[q] + csh.lc[q];
      gsum += csh.gtb[q];
    }
    if (off[CLUSTER] == hc.in_bin && gsum == hc.above) {  // uniform: the same pushed data everywhere
      const uint32_t c = off[CLUSTER], r = k - hc.above;
      uint32_t low_gt, low_eq, gt_in;
      if (c <= WARP_CUT_MAX) {  // every warp resolves it from the pushed lists, no barrier
        const uint32_t lane = threadIdx.x & 31;
        uint32_t kk[WARP_CUT_KEYS], oo[WARP_CUT_KEYS];  // list entries lane + 32 j, their owner ranks
#pragma unroll
        for (int jj = 0; jj < WARP_CUT_KEYS; ++jj) {
          const uint32_t i = lane + 32u * jj;
          uint32_t q = 0, o = 0;
#pragma unroll
          for (int p = 1; p < CLUSTER; ++p) {
            if (i >= off[p]) {
              q = static_cast<uint32_t>(p);
              o = off[p];
            }
          }
          kk[jj] = i < c ? csh.lists[q][i - o] : 0u;
          oo[jj] = q;
        }
        const WarpCut wc = warp_resolve(kk, oo, c, r, static_cast<uint32_t>(rank));
        th.prefix = wc.key;
        gt_in = wc.gt;
        low_gt = wc.low_gt;
        low_eq = wc.low_eq;
      } else {
        uint32_t* list = cs.hist2;  // the cut bin's keys of all ranks, contiguous
        for (uint32_t i = threadIdx.x; i < c; i += SEL_NT) {
          int q = 0;
          while (i >= off[q + 1]) ++q;
          list[i] = csh.lists[q][i - off[q]];
        }
        clear_cut_counters(cs);
        __syncthreads();
        const SelectThreshold<uint32_t> t2 = resolve_cut(list, c, r, hc.above, cs);
        th.prefix = t2.prefix;
        gt_in = t2.n_gt - hc.above;
        // the lower ranks' listed keys above / equal to the threshold (the rank prefix of the list)
        uint32_t* tot = cut_counters(cs) + 2 * BIN_LIST_MAX;
        if (threadIdx.x < c && threadIdx.x < off[rank]) {
          const uint32_t x = list[threadIdx.x];
          if (x > th.prefix) atomicAdd(&tot[0], 1u);
          else if (x == th.prefix) atomicAdd(&tot[1], 1u);
        }
        __syncthreads();
        low_gt = tot[0];
        low_eq = tot[1];
      }
      th.pmask = 0x7fffffffu;
      th.n_gt = hc.above + gt_in;
      th.need_eq = r - gt_in;
      for (int q = 0; q < rank; ++q) cg0 += csh.gtb[q];
      cg0 += low_gt;
      ce0 = low_eq;
      key2 = (base + hc.bin2) << HIST_SHIFT;  // lower edge of the k2-th candidate's bin
      resolved = true;
      LAGS_STAMP(8);
      LAGS_STAMP(9);
      LAGS_STAMP(10);
    }
  }
  const bool hard = !resolved;  // uniform
  // diagnostic: 0 resolved by the cut, 1 no histogram, 2 top bin or crowded, 4 counts mismatch;
  // bits 8.. the cut bin's count
  uint32_t cut_diag = !hard ? 0u : (!hl ? 1u : (!cut ? 2u : 4u));
  if (hl && k < m) cut_diag |= min(hc.in_bin, 0xffffffu) << 8;
  if (hard) {  // top (open) bin or a crowded one: the distributed radix select over every CTA's keys
    int q0 = 0;
    while (rpre[q0 + 1] == rpre[q0]) ++q0;  // the first rank with candidates (m > 0)
    const uint32_t dkey0 = Key<float>::of(cluster.map_shared_rank(reinterpret_cast<const float*>(dyn), q0)[0]);
    cluster_radix_select_dual(cluster, rank, sv, mr, m, dkey0, k, k2, cs, cr, &th, &key2);
    if (rank == 0 && threadIdx.x == 0) {
      csh.prefix = th.prefix;
      csh.pmask = th.pmask;
      csh.n_gt = th.n_gt;
      csh.need_eq = th.need_eq;
      csh.key2 = key2;
    }
    cluster.sync();
    {
      const ClusterShared* o = cluster.map_shared_rank(&csh, 0);
      th.prefix = o->prefix;
      th.pmask = o->pmask;
      th.n_gt = o->n_gt;
      th.need_eq = o->need_eq;
      key2 = o->key2;
    }
    uint32_t lge = 0;  // gt count | eq count << 16 (mr < 65536: it fits the shared memory)
    for (uint32_t i = threadIdx.x; i < mr; i += SEL_NT) {
      const uint32_t key = Key<float>::of(sv[i]);
      const uint32_t hk = key & th.pmask;
      if (key != 0u) lge += hk > th.prefix ? 1u : (hk == th.prefix ? 0x10000u : 0u);
    }
    lge = block_sum(lge, cs.sm);
    if (threadIdx.x == 0) {
      csh.gt = lge & 0xffffu;
      csh.eq = lge >> 16;
    }
    cluster.sync();
    for (int q = 0; q < rank; ++q) {
      const ClusterShared* o = cluster.map_shared_rank(&csh, q);
      cg0 += o->gt;
      ce0 += o->eq;
    }
  }
  const long long c2 = clock64();
  // 3. ordered compaction of the own range with the carried counts of the lower ranks
  float* data = r + L.offset;
  int32_t* oidx = idx_out + L.slot;
  float* oval = val_out + L.slot;
  uint32_t end;
  {  // staged: vector reads of the planes; the P = 1 weights loaded before each chunk's scan
    float* vl = vupd ? vupd + L.offset : nullptr;
    auto emit = [=](int32_t ix, float x, float w) {
      data[ix] = sent_residual(x);  // acc - acc (R: training.py:252)
      if (vl) vl[ix] = single_rank_update(w, x);
    };
    end = compact_staged(mr, th, sv, si, vl, emit, cs, cg0, ce0, oidx, oval);
  }
  if (pp && !dry)  // this CTA's range of the layer's slots (compact_staged ends with a barrier)
    peer_copy(*pp, epoch, idx_out, val_out, L.slot, cg0 + min(ce0, th.need_eq), end, j,
              rank == CLUSTER - 1 ? static_cast<int>(end) : -1, threadIdx.x, SEL_NT);
  LAGS_STAMP(11);
  // the nonzero bins of the own quarter of the chunks (every CTA read its own register copy)
  if (hl && !dry && (SEL_NT - 1 - static_cast<int>(threadIdx.x)) / (SEL_NT / CLUSTER) == rank) clear_hist_chunk(hr, hl);
  LAGS_STAMP(12);
  const long long c3 = clock64();
  if (rank == CLUSTER - 1 && threadIdx.x == 0) count_out[j] = static_cast<int32_t>(end);
  if (rank == 0 && threadIdx.x == 0) {
    auto q = [](long long c) { return static_cast<uint32_t>(min(c >> 6, 2047ll)); };
#ifdef LAGS_DBG_SELECT
    const uint32_t ph = cs.sm.dbg;
#else
    const uint32_t ph = q(c1 - c0) | (q(c2 - c1) << 11) | (q(c3 - c2) << 22);
#endif
    FastState ns = candidate_state(st, next_threshold(st, m, k, k2, th.prefix, key2), m, k, ph);
    ns.cycles = static_cast<uint32_t>(clock64() - t_begin);
    ns.path = hard ? 4u : 3u;
    ns.cut = cut_diag;
    ns.t_start = t_start;
    ns.t_end = globaltimer_lo();
    ns.t_launch = t_launch;
    if (!dry) state[j] = ns;
  }
  // the distributed select reads other CTAs' shared memory up to its last barrier: no CTA leaves
  // before every CTA is past it (the cut path reads only its own after the gather barrier)
  if (hard) cluster_sync_exec();
  LAGS_STAMP(13);
}

// The whole selection of an fp32 compress in ONE launch (thread-block clusters of CLUSTER CTAs):
// the first CLUSTER * n_cl CTAs select the largest layers, one cluster per layer; the next CTAs
// select the tiny layers, one warp per layer (warp_topk_layer); the remaining CTAs walk the
// other layers persistently (largest estimated work first, first layer by block
// index, then an atomic counter).  One launch, so no CTA ever waits on another kernel while
// holding an SM -- this matters when the compress runs beside backprop on a side stream.
__global__ void __launch_bounds__(SEL_NT, SEL_MINB) select_kernel(
    const lags_layer_t* __restrict__ layers, const int2* __restrict__ layer_tasks, const int32_t* __restrict__ cl_layers,
    int n_cl, const int32_t* __restrict__ tiny_layers, int n_tiny, const int32_t* __restrict__ order, int nl,
    FastState* state, const int32_t* __restrict__ cand_cnt,
    const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_val, int cap, int32_t* gidx, float* gval,
    float* r, int32_t* idx_out, float* val_out, int32_t* count_out, int smem_words, int force_exact, SelectCounters sc,
    float* vupd, uint32_t* hist, PeerPush pp) {
  extern __shared__ __align__(16) uint32_t dyn[];
  __shared__ SelectSmem cs;
  __shared__ ClusterShared csh;
  __shared__ ClusterRadix cr;
  __shared__ int next_pos;
  const uint32_t t_launch = globaltimer_lo();
  const int cl_ctas = n_cl * CLUSTER;
  constexpr int NW = SEL_NT / 32;
  const int tiny_ctas = (n_tiny + NW - 1) / NW;
  LAGS_STAMP(14);
  griddep_wait();  // K1 has completed and its writes are visible (programmatic dependent launch)
  LAGS_STAMP(15);
  const PeerPush* ppp = pp.bases ? &pp : nullptr;
  const uint32_t epoch = ppp ? *reinterpret_cast<const volatile uint32_t*>(pp.epoch) + 1u : 0u;
  if (static_cast<int>(blockIdx.x) < cl_ctas) {
#ifdef LAGS_DBG_TWICE  // diagnostic: the layer twice, the first run without side effects on state / histogram
    {
      unsigned long long t0 = clock64();
      cluster_select_layer(cl_layers[blockIdx.x / CLUSTER], layers, layer_tasks, state, cand_cnt, cand_idx, cand_val,
                           cap, gidx, gval, r, idx_out, val_out, count_out, smem_words, force_exact, vupd, dyn, cs, csh,
                           cr, t_launch, hist, true);
      cluster_sync_exec();
      if (blockIdx.x < CLUSTER && threadIdx.x == 0) lags_dbg_stamps[blockIdx.x][0][16] = clock64() - t0;
    }
#endif
    cluster_select_layer(cl_layers[blockIdx.x / CLUSTER], layers, layer_tasks, state, cand_cnt, cand_idx, cand_val, cap,
                         gidx, gval, r, idx_out, val_out, count_out, smem_words, force_exact, vupd, dyn, cs, csh, cr,
                         t_launch, hist, false, ppp, epoch);
  } else if (static_cast<int>(blockIdx.x) < cl_ctas + tiny_ctas) {
    // tiny layers: one warp each, in the CTAs right after the clusters (all in the first wave)
    const int t = (static_cast<int>(blockIdx.x) - cl_ctas) * NW + static_cast<int>(threadIdx.x >> 5);
    if (t < n_tiny) {
      const int j = tiny_layers[t];
      warp_topk_layer(j, layers[j], state, r, idx_out, val_out, count_out, vupd, t_launch);
      if (ppp) {
        __syncwarp();
        const int c = count_out[j];
        peer_copy(pp, epoch, idx_out, val_out, layers[j].slot, 0u, static_cast<uint32_t>(c), j, c,
                  static_cast<int>(threadIdx.x & 31), 32);
      }
    }
  } else {
    const int base = cl_ctas + tiny_ctas;
    const int grid = static_cast<int>(gridDim.x) - base;
    for (int pos = static_cast<int>(blockIdx.x) - base; pos < nl;) {
      if (threadIdx.x == 0) next_pos = static_cast<int>(atomicAdd(sc.work, 1u)) + grid;
      const int j = order[pos];
      select_layer(j, layers, layer_tasks, state, cand_cnt, cand_idx, cand_val, cap, gidx, gval, r, idx_out, val_out,
                   count_out, dyn, smem_words, force_exact, cs, vupd, t_launch, hist);
      if (ppp) {  // select_layer ends with a barrier after the layer's writes
        const int c = count_out[j];
        peer_copy(pp, epoch, idx_out, val_out, layers[j].slot, 0u, static_cast<uint32_t>(c), j, c,
                  static_cast<int>(threadIdx.x), SEL_NT);
      }
      pos = next_pos;
      __syncthreads();  // every thread has read next_pos before thread 0 overwrites it
    }
  }
  if (ppp) peer_publish(pp, epoch);
}

}  // namespace lags
