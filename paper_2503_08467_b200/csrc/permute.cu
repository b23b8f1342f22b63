// permute.cu - Step 2 groupPerExpert / countPerExpert and
// the Sec. 3.3 "concatenate the tokens for the same expert from all GPUs"
// fusion: all N gathered tokens are laid out
// expert-contiguously, ascending global token id inside each expert
// (stable).
//
//   K1 group_hist     per-1024-token block histogram, warp-aggregated atomics
//                     (__match_any_sync -> one shared atomic per distinct expert)
//   K2 group_scan     one CTA: per-(block, expert) bases, counts, offsets
//                     (exclusive scan), tcgen05/SIMT tile tables, work counters
//   K3 group_scatter  stable rank inside the block (per-warp histograms +
//                     match_any ranks), writes perm[j] = global token id
//   K4 gather_rows    X_perm[j] = X_all[perm[j]], 16-B vector copies
// Also: a batched transpose used once at load time to repack expert shards
// K-major (loadShard).
#include "common.cuh"

namespace moeshard {
namespace {

constexpr int kGroupThreads = 256;
constexpr int kTokPerThread = kHistChunk / kGroupThreads;  // 4

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(kGroupThreads) group_hist(const RouteRec* __restrict__ route,
                                                            int N, int E,
                                                            int32_t* __restrict__ block_hist) {
  __shared__ int32_t hist[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = blockIdx.x * kHistChunk;
#pragma unroll
  for (int r = 0; r < kTokPerThread; ++r) {
    const int t = base + r * kGroupThreads + threadIdx.x;
    const int e = (t < N) ? route[t].expert : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    if (e >= 0 && lane == leader) atomicAdd(&hist[e], __popc(peers));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) block_hist[blockIdx.x * E + e] = hist[e];
}

// One CTA of 1024 threads. E <= kMaxExperts.
__global__ void __launch_bounds__(1024) group_scan(const int32_t* __restrict__ block_hist,
                                                   int n_blocks, int E,
                                                   int32_t* __restrict__ block_base, Tables tb,
                                                   int n_mt_up_tc, int n_mt_down_tc) {
  __shared__ int32_t s_cnt[kMaxExperts];
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_tc[kMaxExperts];
  __shared__ int32_t s_simt[kMaxExperts];
  __shared__ int32_t s_rows[kMaxExperts];
  const int tid = threadIdx.x;
  // per-expert totals and per-(block, expert) running bases (relative)
  for (int e = tid; e < E; e += blockDim.x) {
    int run = 0;
    for (int b = 0; b < n_blocks; ++b) {
      const int v = block_hist[b * E + e];
      block_base[b * E + e] = run;
      run += v;
    }
    s_cnt[e] = run;
    int nc, cs;
    tc_chunking(run, &nc, &cs);
    s_tc[e] = nc;
    s_rows[e] = nc > 0 ? (run / cs) * cs + round_up(run % cs, 32) : 0;  // sum of MMA N over chunks
    s_simt[e] = ceil_div(run, kSimtTokTile);
    tb.counts[e] = run;
    tb.tc_chunk_size[e] = cs;
  }
  __syncthreads();
  // exclusive scans over experts (E <= 1024: one element per thread)
  const int lane = tid & 31, warp = tid >> 5;
  auto block_scan = [&](int v) -> int {  // returns exclusive prefix, total in s_warp[31]
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = s_warp[lane];
      int wi = w;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, wi, off);
        if (lane >= off) wi += o;
      }
      s_warp[lane] = wi - w;  // exclusive per-warp base
    }
    __syncthreads();
    const int res = s_warp[warp] + incl - v;
    __syncthreads();
    return res;
  };
  const int v_cnt = tid < E ? s_cnt[tid] : 0;
  const int v_tc = tid < E ? s_tc[tid] : 0;
  const int v_simt = tid < E ? s_simt[tid] : 0;
  const int v_rows = tid < E ? s_rows[tid] : 0;
  const int off = block_scan(v_cnt);
  const int tcp = block_scan(v_tc);
  const int smp = block_scan(v_simt);
  const int rwp = block_scan(v_rows);
  if (tid < E) {
    tb.offsets[tid] = off;
    tb.tc_chunk_pref[tid] = tcp;
    tb.simt_chunk_pref[tid] = smp;
  }
  if (tid == E - 1) {
    tb.offsets[E] = off + v_cnt;
    tb.tc_chunk_pref[E] = tcp + v_tc;
    tb.simt_chunk_pref[E] = smp + v_simt;
    tb.stats[0] = (tcp + v_tc) * n_mt_up_tc;
    tb.stats[1] = (tcp + v_tc) * n_mt_down_tc;
    tb.stats[2] = (rwp + v_rows) * n_mt_up_tc;
  }
  if (tid < E) s_cnt[tid] = off;
  __syncthreads();
  for (int i = tid; i < n_blocks * E; i += blockDim.x) block_base[i] += s_cnt[i % E];
}

// 8 warps x 128 consecutive tokens (4 rounds of 32) per block.
__global__ void __launch_bounds__(kGroupThreads) group_scatter(const RouteRec* __restrict__ route,
                                                               int N, int E,
                                                               const int32_t* __restrict__ block_base,
                                                               int32_t* __restrict__ perm) {
  constexpr int kWarps = kGroupThreads / 32;
  constexpr int kTokPerWarp = kHistChunk / kWarps;  // 128
  __shared__ int32_t whist[kWarps][kMaxExperts];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * E; i += blockDim.x) whist[i / E][i % E] = 0;
  __syncthreads();
  const int wbase = blockIdx.x * kHistChunk + warp * kTokPerWarp;
  int es[kTokPerWarp / 32];
#pragma unroll
  for (int r = 0; r < kTokPerWarp / 32; ++r) {
    const int t = wbase + r * 32 + lane;
    es[r] = (t < N) ? route[t].expert : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, es[r]);
    if (es[r] >= 0 && lane == __ffs(peers) - 1) whist[warp][es[r]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = block_base[blockIdx.x * E + e];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int v = whist[w][e];
      whist[w][e] = run;
      run += v;
    }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kTokPerWarp / 32; ++r) {
    const int t = wbase + r * 32 + lane;
    const int e = es[r];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0) {
      const int j = whist[warp][e] + __popc(peers & lt);
      perm[j] = t;
    }
    __syncwarp();
    if (e >= 0 && lane == __ffs(peers) - 1) whist[warp][e] += __popc(peers);
    __syncwarp();
  }
}

// 16-B vectors, 4 in flight per thread.
__global__ void __launch_bounds__(256) gather_rows_kernel(const uint4* __restrict__ src,
                                                          const int32_t* __restrict__ perm, int N,
                                                          int row_vecs, uint4* __restrict__ dst) {
  const long long total = (long long)N * row_vecs;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 4 * stride) {
    uint4 v[4];
    long long di[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      di[u] = -1;
      if (i < total) {
        const int j = (int)(i / row_vecs);
        const int c = (int)(i - (long long)j * row_vecs);
        const int t = __ldg(perm + j);
        v[u] = __ldg(src + (long long)t * row_vecs + c);
        di[u] = i;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (di[u] >= 0) dst[di[u]] = v[u];
  }
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ src, T* __restrict__ dst, int rows,
                                 int cols) {
  __shared__ T tile[32][33];
  const size_t b = blockIdx.z;
  const T* s = src + b * rows * (size_t)cols;
  T* d = dst + b * rows * (size_t)cols;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = s[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) d[(size_t)c * rows + r] = tile[threadIdx.x][i];
  }
}


// Single-CTA fused grouping (N <= kFusedMaxTokens): the three phases of
// hist / scan / scatter in one launch. 32 warps; warp w owns the contiguous
// token range [w*span, (w+1)*span) so the stable order is warp-major.
constexpr int kFusedMaxTokens = 65536;

__device__ __forceinline__ int block_excl_scan_1024(int v, int* s_warp, int& total) {
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
    const int w = s_warp[lane];
    int wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += o;
    }
    s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const int res = s_warp[warp] + incl - v;
  total = s_warp[32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(1024, 1) group_fused(const RouteRec* __restrict__ route, int N,
                                                       int E, Tables tb, int n_mt_up_tc,
                                                       int n_mt_down_tc, int32_t* __restrict__ perm) {
  __shared__ int32_t whist[32][kMaxExperts];
  __shared__ int32_t s_warp[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * E; i += 1024) whist[i / E][i % E] = 0;
  __syncthreads();
  const int span = ceil_div(ceil_div(N, 32), 32) * 32;   // multiple of 32 tokens per warp
  const int t_begin = warp * span, t_end = min(N, t_begin + span);
  constexpr int U = 8;  // rounds of 32 tokens loaded together (memory-level parallelism)
  // phase 1: per-warp histograms (warp-aggregated: one update per distinct expert per round)
  for (int t0 = t_begin; t0 < t_end; t0 += 32 * U) {
    int es[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * 32 + lane;
      es[u] = t < t_end ? __ldg(&route[t].expert) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned peers = __match_any_sync(0xffffffffu, es[u]);
      if (es[u] >= 0 && lane == __ffs(peers) - 1) whist[warp][es[u]] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  // phase 2: totals, tile tables, offsets, per-warp bases
  const int e = threadIdx.x;
  int cnt = 0, nc = 0, cs = 0, rows = 0, sc = 0;
  if (e < E) {
    for (int w = 0; w < 32; ++w) cnt += whist[w][e];
    tc_chunking(cnt, &nc, &cs);
    rows = nc > 0 ? (cnt / cs) * cs + round_up(cnt % cs, 32) : 0;
    sc = ceil_div(cnt, kSimtTokTile);
    tb.counts[e] = cnt;
    tb.tc_chunk_size[e] = cs;
  }
  int tot_cnt, tot_tc, tot_sc, tot_rows;
  const int off = block_excl_scan_1024(cnt, s_warp, tot_cnt);
  const int tcp = block_excl_scan_1024(nc, s_warp, tot_tc);
  const int smp = block_excl_scan_1024(sc, s_warp, tot_sc);
  block_excl_scan_1024(rows, s_warp, tot_rows);
  if (e < E) {
    tb.offsets[e] = off;
    tb.tc_chunk_pref[e] = tcp;
    tb.simt_chunk_pref[e] = smp;
    int run = off;
    for (int w = 0; w < 32; ++w) {
      const int v = whist[w][e];
      whist[w][e] = run;
      run += v;
    }
  }
  if (threadIdx.x == 0) {
    tb.offsets[E] = tot_cnt;
    tb.tc_chunk_pref[E] = tot_tc;
    tb.simt_chunk_pref[E] = tot_sc;
    tb.stats[0] = tot_tc * n_mt_up_tc;
    tb.stats[1] = tot_tc * n_mt_down_tc;
    tb.stats[2] = tot_rows * n_mt_up_tc;
  }
  __syncthreads();
  // phase 3: stable ranks -> perm
  const unsigned lt = lanemask_lt();
  for (int t0 = t_begin; t0 < t_end; t0 += 32 * U) {
    int es[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * 32 + lane;
      es[u] = t < t_end ? __ldg(&route[t].expert) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ee = es[u];
      const unsigned peers = __match_any_sync(0xffffffffu, ee);
      if (ee >= 0) perm[whist[warp][ee] + __popc(peers & lt)] = t0 + u * 32 + lane;
      __syncwarp();
      if (ee >= 0 && lane == __ffs(peers) - 1) whist[warp][ee] += __popc(peers);
      __syncwarp();
    }
  }
}

// One warp per destination row, rows_per_warp rows in flight per iteration.
template <int VPL>  // 16-B vectors per lane per row
__global__ void __launch_bounds__(256) gather_rows_warp(const uint4* __restrict__ src,
                                                        const int32_t* __restrict__ perm, int N,
                                                        int row_vecs, uint4* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int j0 = gw * 2; j0 < N; j0 += nw * 2) {
    uint4 v[2][VPL];
    int rows[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = j0 + r;
      rows[r] = j < N ? __ldg(perm + j) : -1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (rows[r] >= 0 && c < row_vecs) v[r][i] = __ldg(src + (size_t)rows[r] * row_vecs + c);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (rows[r] >= 0 && c < row_vecs) dst[(size_t)(j0 + r) * row_vecs + c] = v[r][i];
      }
  }
}
}  // namespace

void launch_group(const RouteRec* route, int N, int E, int32_t* block_hist, int32_t* block_base,
                  Tables tb, int n_mt_up_tc, int n_mt_down_tc, int32_t* perm, cudaStream_t s) {
  if (N <= kFusedMaxTokens) {
    group_fused<<<1, 1024, 0, s>>>(route, N, E, tb, n_mt_up_tc, n_mt_down_tc, perm);
    return;
  }
  const int nb = ceil_div(N, kHistChunk);
  if (nb > 0) group_hist<<<nb, kGroupThreads, 0, s>>>(route, N, E, block_hist);
  group_scan<<<1, 1024, 0, s>>>(block_hist, nb, E, block_base, tb, n_mt_up_tc, n_mt_down_tc);
  if (nb > 0) group_scatter<<<nb, kGroupThreads, 0, s>>>(route, N, E, block_base, perm);
}

void launch_gather_rows(const void* x_all, const int32_t* perm, int N, int row_bytes, void* x_perm,
                        cudaStream_t s) {
  if (N <= 0) return;
  const int row_vecs = row_bytes / 16;
  if (row_vecs <= 32 * 8) {
    const int vpl = ceil_div(row_vecs, 32);
    int grid = ceil_div(ceil_div(N, 2), 8);            // 8 warps per block, 2 rows per warp
    if (grid > 148 * 8) grid = 148 * 8;
    auto* sp = static_cast<const uint4*>(x_all);
    auto* dp = static_cast<uint4*>(x_perm);
    switch (vpl) {
      case 1: gather_rows_warp<1><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
      case 2: gather_rows_warp<2><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
      case 3: gather_rows_warp<3><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
      case 4: gather_rows_warp<4><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
      case 5: case 6: gather_rows_warp<6><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
      default: gather_rows_warp<8><<<grid, 256, 0, s>>>(sp, perm, N, row_vecs, dp); return;
    }
  }
  const long long total = (long long)N * row_vecs;
  int grid = (int)((total + 4LL * 256 - 1) / (4LL * 256));
  if (grid > 148 * 16) grid = 148 * 16;
  gather_rows_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(x_all), perm, N, row_vecs,
                                          static_cast<uint4*>(x_perm));
}

void launch_transpose(int dtype, const void* src, void* dst, int batch, int rows, int cols,
                      cudaStream_t s) {
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32), batch), block(32, 8);
  if (dtype == 0)
    transpose_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(
        static_cast<const __nv_bfloat16*>(src), static_cast<__nv_bfloat16*>(dst), rows, cols);
  else
    transpose_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(src),
                                                   static_cast<float*>(dst), rows, cols);
}

}  // namespace moeshard
