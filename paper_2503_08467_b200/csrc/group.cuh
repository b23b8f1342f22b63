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
// The five exclusive prefixes (count, padded count, tcgen05 chunks, SIMT chunks, tcgen05
// rows) are computed in ONE pass: warp-level scans of all five, one exchange of the warp
// totals through s_warp (>= 5 * kThreads / 32 + 5 ints), two CTA barriers in total (the
// grouping CTAs sit on this before their row copies; five separate CTA-wide scans cost
// 1-2.6 us of the pre-FFN critical path).
// kNP = 5: all five prefixes (the publishing CTA); kNP = 2: only the compact and padded
// offsets every other grouping CTA needs for its own rows.
template <int kThreads, int kNP = 5>
__device__ __forceinline__ void segment_tables(int E, const int* s_tot, const int* s_pre,
                                               int* s_base, int* s_bpad, int* s_warp, bool publish,
                                               Tables tb, int n_mt_up_tc, int n_mt_down_tc) {
  static_assert(kNP == 2 || kNP == 5, "prefixes");
  constexpr int kWarps = kThreads / 32;
  const int e = threadIdx.x, lane = e & 31, w = e >> 5;
  int v[5] = {0, 0, 0, 0, 0};   // count, padded count, tc chunks, simt chunks, tc rows
  int cs = 0;
  if (e < E) {
    const int cnt = s_tot[e];
    int nc;
    tc_chunking(cnt, &nc, &cs);
    v[0] = cnt;
    v[1] = round_up(cnt, kSegAlign);
    v[2] = nc;
    v[3] = ceil_div(cnt, kSimtTokTile);
    v[4] = nc > 0 ? (cnt / cs) * cs + round_up(cnt % cs, 32) : 0;
  }
  int inc[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < kNP; ++i) {
    inc[i] = v[i];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, inc[i], off);
      if (lane >= off) inc[i] += o;
    }
  }
  __syncthreads();   // s_warp may still be read by an earlier scan
  if (lane == 31) {
#pragma unroll
    for (int i = 0; i < kNP; ++i) s_warp[i * kWarps + w] = inc[i];
  }
  __syncthreads();
  int ex[5] = {0, 0, 0, 0, 0}, tot[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < kNP; ++i) {
    int before = 0, all = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const int ws = s_warp[i * kWarps + q];
      before += q < w ? ws : 0;
      all += ws;
    }
    ex[i] = before + inc[i] - v[i];
    tot[i] = all;
  }
  if (e < E) {
    s_base[e] = ex[0] + s_pre[e];
    s_bpad[e] = ex[1] + s_pre[e];
  }
  if (kNP == 5 && publish) {
    for (int i = threadIdx.x; i < tot[2]; i += kThreads) tb.done[i] = 0;   // per token chunk
    if (e < E) {
      tb.pos[e] = ex[1];
      tb.counts[e] = v[0];
      tb.tc_chunk_size[e] = cs;
      tb.offsets[e] = ex[0];
      tb.tc_chunk_pref[e] = ex[2];
      tb.simt_chunk_pref[e] = ex[3];
    }
    if (threadIdx.x == 0) {
      tb.next_unit[0] = 0;
      tb.pos[E] = tot[1];
      tb.offsets[E] = tot[0];
      tb.tc_chunk_pref[E] = tot[2];
      tb.simt_chunk_pref[E] = tot[3];
      tb.stats[0] = tot[2] * n_mt_up_tc;
      tb.stats[1] = tot[2] * n_mt_down_tc;
      tb.stats[2] = tot[4] * n_mt_up_tc;
    }
  }
}

}  // namespace moeshard
