// permute.cu - Step 2 groupPerExpert / countPerExpert and
// the Sec. 3.3 "concatenate the tokens for the same expert from all GPUs"
// fusion: all N gathered tokens are laid out
// expert-contiguously, ascending global token id inside each expert
// (stable).
//
//   (router kernels)  per-hist-block expert histograms (countPerExpert)
//   group_scatter_gather  one CTA per hist-block: reduce the histograms to
//                     offsets (CTA 0 also publishes the tile tables), stable
//                     rank inside the block (match_any), perm[j] = global token
//                     id, and the row copy X_perm[j] = X_all[t] (16-B vectors)
// Also: a batched transpose used once at load time to repack expert shards
// K-major (loadShard).
#include <algorithm>

#include "common.cuh"
#include "group.cuh"
#include "ptx.cuh"
#include "timeline.cuh"

namespace moeshard {
namespace {


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


// ===========================================================================
// Step 2 from per-block histograms (the product path).
// The router CTAs write hist[b][e] = tokens of hist-block b (HB consecutive
// local tokens) routed to expert e: the paper's countPerExpert / m_sizes
// at block granularity; with G > 1 the blocks of all
// ranks arrive by AllGather in rank order, so block b covers global tokens
// [r*n + i*HB, min(r*n + (i+1)*HB, (r+1)*n)) with r = b / nbr, i = b % nbr.
// ===========================================================================

// One CTA per expert: exclusive prefix of hist[.][e] over the NB blocks ->
// base[b][e] (tokens of expert e in blocks before b) and tot[e]. O(NB*E)
// in total, so the grouping CTAs read only 2*E values each.
__global__ void __launch_bounds__(128) group_block_scan(const int32_t* __restrict__ hist, int NB,
                                                        int E, int32_t* __restrict__ base,
                                                        int32_t* __restrict__ tot) {
  ptx::griddep_wait();                 // hist comes from the router (or the AllGather)
  ptx::griddep_launch_dependents();
  if (threadIdx.x == 0) { TL_MIN(0); TL_MAX(0); }
  __shared__ int32_t s_warp[33];
  const int e = blockIdx.x;
  const int q = ceil_div(NB, 128);
  const int b0 = threadIdx.x * q, b1 = min(NB, b0 + q);
  int sum = 0;
  for (int b = b0; b < b1; ++b) sum += __ldg(hist + (size_t)b * E + e);
  int total;
  int run = block_excl_scan<128>(sum, s_warp, total);
  for (int b = b0; b < b1; ++b) {
    base[(size_t)b * E + e] = run;
    run += __ldg(hist + (size_t)b * E + e);
  }
  if (threadIdx.x == 0) tot[e] = total;
}

// One CTA group per hist-block (HB <= 128 tokens), the rest of Step 2:
//  1. totals and earlier-block counts come from group_block_scan; offsets =
//     exclusive scan of the totals; CTA 0 also publishes counts / offsets /
//     tile tables / work counters;
//  2. warps 0-3 give each token its stable rank inside the block
//     (match_any) -> j = offsets[e] + earlier[e] + rank, perm[j] = t;
//  3. the block's rows are copied to X_perm[j] (16-B vectors, 4 rows per warp
//     with every load of the first VPL*32 vectors in flight before the stores;
//     wider rows continue in column blocks of VPL*32 vectors).
// kSplit CTAs share one hist-block: all compute its ranks, each copies
// 128/kSplit of its rows (spreads the row traffic over more SMs).
template <int VPL, int kSplit, int K>
__global__ void __launch_bounds__(1024 / kSplit) group_scatter_gather(
    const int32_t* __restrict__ bbase, const int32_t* __restrict__ btot, int E, Tables tb,
    int n_mt_up_tc, int n_mt_down_tc, const RouteRec* __restrict__ route,
    const uint4* __restrict__ x_all, int n, int nbr, int HB, int32_t* __restrict__ perm,
    int row_vecs, uint4* __restrict__ x_perm, int NB) {
  // K = top_k: a block of HB tokens holds HB K (token, expert) assignments a = K t + j
  // (route records, histograms and the expert-ordered rows are per assignment)
  if (threadIdx.x == 0) TL_MIN(1);
  constexpr int kThreads = 1024 / kSplit;
  constexpr int kRowsPerWarp = 4;                 // rows copied per warp
  constexpr int kColBlock = VPL * 32;             // 16-B vectors per column block
  static_assert(kThreads >= 256, "ranks need 128 K threads (K <= 2)");
  static_assert(kRowsPerWarp * (kThreads / 32) == 128 / kSplit, "one row group = 128 / kSplit rows");
  __shared__ int32_t s_tot[kMaxExperts];
  __shared__ int32_t s_pre[kMaxExperts];
  __shared__ int32_t s_base[kMaxExperts];   // compact (public perm) position of this block's first e
  __shared__ int32_t s_bpad[kMaxExperts];   // padded internal position
  __shared__ int32_t whist[4 * K][kMaxExperts];
  __shared__ int32_t s_j[128 * K];
  __shared__ int32_t s_warp[5 * (kThreads / 32)];   // segment_tables' warp totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x / kSplit, part = blockIdx.x % kSplit;
  const int r = b / nbr, i = b - r * nbr;
  const int t0 = r * n + i * HB;
  const int t1 = min(t0 + HB, (r + 1) * n);
  const int a0 = t0 * K, na = (t1 - t0) * K;     // the block's assignments
  const int row_base = part * (128 * K / kSplit); // this CTA's assignment rows of the block
  // Everything that needs only the routing runs before the wait for the block scan: this
  // grid is launched once the scan has passed its own wait, so the route records and token
  // rows (router, AllGather or peer pushes, all before the scan) are complete. The stable
  // ranks inside the block (match_any) and the row loads overlap the scan; only the
  // segment starts need it.
  const bool has_block = b < NB;
  // issue this CTA's row loads first: the sources are known, only the
  // destinations depend on the scan
  uint4 v[kRowsPerWarp][VPL];
#pragma unroll
  for (int u = 0; u < kRowsPerWarp; ++u) {
    const int q = row_base + warp * kRowsPerWarp + u;   // assignment row of the block
    const int tt = has_block && q < na ? t0 + q / K : t1;
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const int col = lane + 32 * c;
      if (tt < t1 && col < row_vecs) v[u][c] = __ldg(x_all + (size_t)tt * row_vecs + col);
    }
  }
  constexpr int rank_warps = 4 * K;               // warps holding one assignment per thread
  int e = -1, rank_w = 0, a = 0;
  float gate = 0.f;
  if (warp < rank_warps && has_block) {
    a = a0 + threadIdx.x;
    if (threadIdx.x < na) {
      const RouteRec rec = route[a];
      e = rec.expert;
      gate = rec.gate;
    }
  }
  for (int k = threadIdx.x; k < rank_warps * E; k += kThreads) whist[k / E][k % E] = 0;
  __syncthreads();
  // 2. stable ranks inside the block (assignment order)
  if (warp < rank_warps) {
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    rank_w = __popc(peers & lanemask_lt());
    if (e >= 0 && rank_w == 0) whist[warp][e] = __popc(peers);
  }
  __syncthreads();
  if (warp < rank_warps && e >= 0)
    for (int w = 0; w < warp; ++w) rank_w += whist[w][e];   // rank inside the block
  ptx::griddep_wait();            // the block scan (base, tot)
  ptx::griddep_launch_dependents();   // the FFN's prologue may start now
  if (threadIdx.x == 0) { TL_MIN(3); TL_MAX(3); }
  for (int k = threadIdx.x; k < E; k += kThreads) {
    s_tot[k] = __ldg(btot + k);                        // tokens of expert k overall
    s_pre[k] = __ldg(bbase + (size_t)b * E + k);       // ... in blocks before this one
  }
  __syncthreads();
  if (threadIdx.x == 0) { TL_MIN(4); TL_MAX(4); }
#ifndef MOESHARD_TABLES_2P
#define MOESHARD_TABLES_2P 1
#endif
  if (!MOESHARD_TABLES_2P || blockIdx.x == 0)
    segment_tables<kThreads, 5>(E, s_tot, s_pre, s_base, s_bpad, s_warp, blockIdx.x == 0, tb,
                                n_mt_up_tc, n_mt_down_tc);
  else   // only the two offsets this CTA's rows need
    segment_tables<kThreads, 2>(E, s_tot, s_pre, s_base, s_bpad, s_warp, false, tb,
                                n_mt_up_tc, n_mt_down_tc);
  if (threadIdx.x == 0) { TL_MIN(5); TL_MAX(5); }
  __syncthreads();   // s_base / s_bpad of every expert
  if (blockIdx.x == 0) {   // the tables are out: the FFN's weight stream may start (early_tables)
    if (threadIdx.x == 0) ptx::st_release_gpu(tb.stats + 6, 1);
    if (threadIdx.x == 0) { TL_MIN(2); TL_MAX(2); }
  }
  if (warp < rank_warps) {
    if (e >= 0) {
      const int j = s_base[e] + rank_w;         // public, compact
      const int jp = s_bpad[e] + rank_w;        // internal, padded segments
      if (part == 0) {
        perm[j] = a;                            // global token id (K = 1) / assignment id
        tb.perm_pad[jp] = a;
        tb.gate_pad[jp] = gate;   // the down epilogue reads row and gate without an indirection
      }
      s_j[threadIdx.x] = jp;
    } else {
      s_j[threadIdx.x] = -1;
    }
  }
  __syncthreads();
  // 3. row stores (first column block loaded at the top)
  if (threadIdx.x == 0) { TL_MIN(6); TL_MAX(6); }
  if (x_perm == nullptr || !has_block) return;
#pragma unroll
  for (int g = 0; g < K; ++g) {   // groups of 32 assignment rows (kRowsPerWarp x 8 warps)
  const int gbase = row_base + g * kRowsPerWarp * (kThreads / 32);
  if (g > 0) {
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      const int q = gbase + warp * kRowsPerWarp + u;
      const int tt = q < na ? t0 + q / K : t1;
#pragma unroll
      for (int c = 0; c < VPL; ++c) {
        const int col = lane + 32 * c;
        if (tt < t1 && col < row_vecs) v[u][c] = __ldg(x_all + (size_t)tt * row_vecs + col);
      }
    }
  }
  int jj[kRowsPerWarp];
#pragma unroll
  for (int u = 0; u < kRowsPerWarp; ++u) {
    const int q = gbase + warp * kRowsPerWarp + u;
    jj[u] = q < na ? s_j[q] : -1;
  }
#pragma unroll
  for (int u = 0; u < kRowsPerWarp; ++u)
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const int col = lane + 32 * c;
      if (jj[u] >= 0 && col < row_vecs) x_perm[(size_t)jj[u] * row_vecs + col] = v[u][c];
    }
  for (int c0 = kColBlock; c0 < row_vecs; c0 += kColBlock) {   // rows wider than one block
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      const int tt = t0 + (gbase + warp * kRowsPerWarp + u) / K;
#pragma unroll
      for (int c = 0; c < VPL; ++c) {
        const int col = c0 + lane + 32 * c;
        if (jj[u] >= 0 && col < row_vecs) v[u][c] = __ldg(x_all + (size_t)tt * row_vecs + col);
      }
    }
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u)
#pragma unroll
      for (int c = 0; c < VPL; ++c) {
        const int col = c0 + lane + 32 * c;
        if (jj[u] >= 0 && col < row_vecs) x_perm[(size_t)jj[u] * row_vecs + col] = v[u][c];
      }
  }
  }   // groups
  if (threadIdx.x == 0) TL_MAX(1);
}

}  // namespace

TL_EXPORT(moeshard_tl_group)

void launch_group_blocks(const int32_t* hist, int NB, int E, int32_t* base, int32_t* tot,
                         Tables tb, int n_mt_up_tc, int n_mt_down_tc, const RouteRec* route,
                         const void* x_all, int n, int nbr, int HB, int row_bytes, int32_t* perm,
                         void* x_perm, cudaStream_t s, int K) {
  if (NB <= 0) return;
  launch_pdl(group_block_scan, dim3(E), dim3(128), 0, s, hist, NB, E, base, tot);
  const int row_vecs = row_bytes / 16;
  const int vpl = ceil_div(row_vecs, 32);
  auto* xs = static_cast<const uint4*>(x_all);
  auto* xd = static_cast<uint4*>(x_perm);
  // each hist-block's rows are copied by kSplit = 4 CTAs of 256 threads; rows wider
  // than 8 * 32 vectors (4 KB) are copied in column blocks of 4 KB
#ifndef MOESHARD_GROUP_SPLIT
#define MOESHARD_GROUP_SPLIT 4
#endif
  constexpr int kSp = MOESHARD_GROUP_SPLIT;
#define SG(V)                                                                                  \
  (K == 2 ? launch_pdl(group_scatter_gather<V, kSp, 2>, dim3(NB * kSp), dim3(1024 / kSp), 0, s,    \
                       base, tot, E, tb, n_mt_up_tc, n_mt_down_tc, route, xs, n, nbr, HB, perm,     \
                       row_vecs, xd, NB)                                                           \
          : launch_pdl(group_scatter_gather<V, kSp, 1>, dim3(NB * kSp), dim3(1024 / kSp), 0, s,    \
                       base, tot, E, tb, n_mt_up_tc, n_mt_down_tc, route, xs, n, nbr, HB, perm,     \
                       row_vecs, xd, NB))
  switch (vpl) {
    case 1: SG(1); break;
    case 2: SG(2); break;
    case 3: SG(3); break;
    case 4: SG(4); break;
    case 5: case 6: SG(6); break;
    default: SG(8); break;
  }
#undef SG
}

namespace {
// top_k > 1: the token's output is the sum of its K assignments' gate-scaled expert rows
// (R21), y[t] = sum_j y_assign[K t + j], fp32 sum, one bf16 rounding; 8 features per thread.
__global__ void __launch_bounds__(256) combine_assignments(const uint4* __restrict__ ya,
                                                           uint4* __restrict__ y, int n_tok,
                                                           int vecs, int K) {
  ptx::griddep_wait();   // the FFN's down epilogue wrote ya
  ptx::griddep_launch_dependents();
  const long long total = static_cast<long long>(n_tok) * vecs;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = q / vecs, c = q - t * vecs;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < K; ++j) {
      const uint4 v = __ldcg(ya + (t * K + j) * vecs + c);
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(p[i]);
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) po[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    y[t * vecs + c] = o;
  }
}
}  // namespace

void launch_combine_assignments(const void* y_assign, void* y, int n_tok, int row_bytes, int K,
                                int num_sms, cudaStream_t s) {
  if (n_tok <= 0) return;
  const int vecs = row_bytes / 16;
  const long long total = static_cast<long long>(n_tok) * vecs;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 4LL * num_sms));
  launch_pdl(combine_assignments, dim3(grid), dim3(256), 0, s, static_cast<const uint4*>(y_assign),
             static_cast<uint4*>(y), n_tok, vecs, K);
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
