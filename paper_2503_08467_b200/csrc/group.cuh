// group.cuh - device pieces of Step 2 groupPerExpert and the
// Sec. 3.3 per-expert concatenation shared by the grouping
// kernels of permute.cu: a CTA-wide exclusive scan, the per-forward segment
// tables and the stable in-block rank of a token.
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace moeshard {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan over the CTA (kThreads <= 1024, one value per thread); total in `total`.
// Every thread of the CTA must call it (it synchronises).
template <int kThreads>
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < kWarps ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += o;
    }
    if (lane < kWarps) s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const int res = s_warp[warp] + incl - v;
  total = s_warp[32];
  __syncthreads();
  return res;
}

// Offsets of every expert segment from the per-expert totals (thread e < E
// holds expert e; E <= kThreads): s_base[e] = public (compact) start +
// pre, s_bpad[e] = internal padded start + pre, where pre = tokens of e in
// earlier hist-blocks. If `publish`, also writes the tables the grouped
// GEMMs read (counts, offsets, chunking, padded starts, done = 0, stats).
template <int kThreads>
__device__ __forceinline__ void segment_tables(int E, const int* s_tot, const int* s_pre,
                                               int* s_base, int* s_bpad, int* s_warp, bool publish,
                                               Tables tb, int n_mt_up_tc, int n_mt_down_tc) {
  const int e = threadIdx.x;
  int cnt = 0, nc = 0, cs = 0, rows = 0, sc = 0;
  if (e < E) {
    cnt = s_tot[e];
    tc_chunking(cnt, &nc, &cs);
    rows = nc > 0 ? (cnt / cs) * cs + round_up(cnt % cs, 32) : 0;
    sc = ceil_div(cnt, kSimtTokTile);
  }
  int tot_cnt, tot_pad;
  const int off = block_excl_scan<kThreads>(cnt, s_warp, tot_cnt);
  const int pos = block_excl_scan<kThreads>(round_up(cnt, kSegAlign), s_warp, tot_pad);
  if (e < E) {
    s_base[e] = off + s_pre[e];
    s_bpad[e] = pos + s_pre[e];
  }
  if (publish) {
    int tot_tc, tot_sc, tot_rows;
    const int tcp = block_excl_scan<kThreads>(nc, s_warp, tot_tc);
    const int smp = block_excl_scan<kThreads>(sc, s_warp, tot_sc);
    block_excl_scan<kThreads>(rows, s_warp, tot_rows);
    for (int i = threadIdx.x; i < tot_tc; i += kThreads) tb.done[i] = 0;   // per token chunk
    if (e < E) {
      tb.pos[e] = pos;
      tb.counts[e] = cnt;
      tb.tc_chunk_size[e] = cs;
      tb.offsets[e] = off;
      tb.tc_chunk_pref[e] = tcp;
      tb.simt_chunk_pref[e] = smp;
    }
    if (threadIdx.x == 0) {
      tb.next_unit[0] = 0;
      tb.pos[E] = tot_pad;
      tb.offsets[E] = tot_cnt;
      tb.tc_chunk_pref[E] = tot_tc;
      tb.simt_chunk_pref[E] = tot_sc;
      tb.stats[0] = tot_tc * n_mt_up_tc;
      tb.stats[1] = tot_tc * n_mt_down_tc;
      tb.stats[2] = tot_rows * n_mt_up_tc;
    }
  }
}

}  // namespace moeshard
