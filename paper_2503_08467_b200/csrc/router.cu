// router.cu - Step 1 token routing (Alg. 1 line "m_expert <- router(x)",
// PAPER.md:187-188, 261-263): logits = x W_r (fp32 accumulation), softmax,
// top-1 argmax with lowest-index tie-break (R4), gate = softmax
// probability of the chosen expert (R2). Optional forced expert ids (the
// paper's replaced router).
//
// Two implementations:
//  * router_tc_kernel (bf16, the product path; bottom of this file): tcgen05
//    logits on the tensor cores, token on the TMEM lane axis;
//  * router_kernel (fp32 validation mode, and bf16 with MOESHARD_FLAG_SIMT_GEMM):
//    FFMA on CUDA cores, described next.
//
// Layout: x [n][h] row-major (bf16 or fp32), W_r [h][E] row-major.
// One CTA = 64 tokens x all E experts. 256 threads = 16 token groups (ty) x
// 16 expert lanes (tx); thread (ty, tx) owns tokens ty*4+i and experts
// tx + 16*j (j < EPT). The per-token max / sum-exp reductions over the 16
// expert lanes are xor warp shuffles (the 16 lanes sit in one half-warp).
#include "common.cuh"

namespace moeshard {
namespace {

constexpr int RT_TOK = 64;
constexpr int RT_KC = 32;

template <typename T> struct Load8;
template <> struct Load8<__nv_bfloat16> {
  __device__ static void run(const __nv_bfloat16* p, float* v) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(b[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
};
template <> struct Load8<float> {
  __device__ static void run(const float* p, float* v) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

template <typename T, int EPT>
__global__ void __launch_bounds__(256) router_kernel(const T* __restrict__ x, int n, int h,
                                                     const T* __restrict__ w_r, int E,
                                                     const int32_t* __restrict__ forced,
                                                     RouteRec* __restrict__ out,
                                                     int32_t* __restrict__ hist_out,
                                                     int32_t* __restrict__ err_flag) {
  constexpr int EP = EPT * 16;                 // padded expert count handled by this instantiation
  __shared__ __align__(16) float xs[RT_KC][RT_TOK + 4];
  __shared__ __align__(16) float ws[RT_KC][EP];
  __shared__ int32_t s_hist[kMaxExperts];

  const int tid = threadIdx.x;
  for (int e = tid; e < E; e += 256) s_hist[e] = 0;
  const int tx = tid & 15, ty = tid >> 4;
  const int tok0 = blockIdx.x * RT_TOK;

  float acc[4][EPT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < EPT; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < h; k0 += RT_KC) {
    // x tile: 64 tokens x 32 k -> 2048 elements, 8 per thread (one 16/32-B vector)
    {
      const int r = tid >> 2, c = (tid & 3) * 8;
      float v[8];
      if (tok0 + r < n) {
        Load8<T>::run(x + (size_t)(tok0 + r) * h + k0 + c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) xs[c + i][r] = v[i];
    }
    // W_r chunk: 32 rows x E (pad to EP with zeros)
    for (int idx = tid; idx < RT_KC * EP; idx += 256) {
      const int kk = idx / EP, e = idx - kk * EP;
      ws[kk][e] = (e < E) ? to_f32(w_r[(size_t)(k0 + kk) * E + e]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < RT_KC; ++kk) {
      const float4 xv = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
      const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const float w = ws[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(xa[i], w, acc[i][j]);
      }
    }
    __syncthreads();
  }

  // softmax + top-1 per token; reductions over the 16 expert lanes
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = tok0 + ty * 4 + i;
    float best = -INFINITY;
    int best_e = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tx + 16 * j;
      if (e < E && (acc[i][j] > best || (acc[i][j] == best && e < best_e))) {
        best = acc[i][j];
        best_e = e;
      }
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oe = __shfl_xor_sync(0xffffffffu, best_e, off);
      if (ob > best || (ob == best && oe < best_e)) {
        best = ob;
        best_e = oe;
      }
    }
    int sel = best_e;
    bool bad = false;
    if (forced != nullptr && t < n) {
      sel = forced[t];
      if (sel < 0 || sel >= E) {
        bad = true;
        sel = sel < 0 ? 0 : E - 1;
      }
    }
    float sum = 0.f, lsel = 0.f;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tx + 16 * j;
      if (e < E) sum += expf(acc[i][j] - best);
      if (e == sel) lsel = acc[i][j];
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, off);
      lsel += __shfl_xor_sync(0xffffffffu, lsel, off);
    }
    if (tx == 0 && t < n) {
      RouteRec r;
      r.expert = sel;
      r.gate = expf(lsel - best) / sum;
      out[t] = r;
      atomicAdd(&s_hist[sel], 1);
      if (bad) atomicOr(err_flag, 1);
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += 256) hist_out[(size_t)blockIdx.x * E + e] = s_hist[e];
}

template <typename T>
void launch_router_t(const T* x, int n, int h, const T* w_r, int E, const int32_t* forced,
                     RouteRec* out, int32_t* hist, int32_t* err, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid(ceil_div(n, RT_TOK));
  if (E <= 16) router_kernel<T, 1><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, hist, err);
  else if (E <= 32) router_kernel<T, 2><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, hist, err);
  else if (E <= 64) router_kernel<T, 4><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, hist, err);
  else if (E <= 128) router_kernel<T, 8><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, hist, err);
  else router_kernel<T, 16><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, hist, err);
}

}  // namespace

void launch_router(int dtype, const void* x, int n, int h, const void* w_r, int E,
                   const int32_t* forced, RouteRec* out, int32_t* hist_out, int32_t* err_flag,
                   cudaStream_t s) {
  if (dtype == 0)
    launch_router_t(static_cast<const __nv_bfloat16*>(x), n, h,
                    static_cast<const __nv_bfloat16*>(w_r), E, forced, out, hist_out, err_flag, s);
  else
    launch_router_t(static_cast<const float*>(x), n, h, static_cast<const float*>(w_r), E, forced,
                    out, hist_out, err_flag, s);
}

}  // namespace moeshard

// ===========================================================================
// tcgen05 router (bf16): logits for 128 tokens x EP experts per CTA on the
// tensor cores. A = x tile [128 tok][h] (TMA, K-major, 128-B swizzle),
// B = W_r^T [EP][h] (transposed + zero-padded once per forward into the
// workspace by router_transpose, TMA). D[t][e] lives in TMEM with the token
// on the lane axis, so each epilogue thread owns one token's whole logit row
// and computes max / argmax (lowest index) / sum-exp sequentially - no
// cross-thread reduction at all.
// ===========================================================================
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "gemm_tc.cuh"
#include "ptx.cuh"
#include "timeline.cuh"

namespace moeshard {
namespace {

constexpr int RTC_TOK = 128;         // tokens per CTA = hist-block size (TMEM lanes)
constexpr int RTC_MAX_STAGES = 16;

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp; exp2(-inf) = +0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int RTC_SMEM_BUDGET = 200 * 1024;

__global__ void router_transpose(const __nv_bfloat16* __restrict__ w_r, int h, int E, int EP,
                                 __nv_bfloat16* __restrict__ wt) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int k0 = blockIdx.x * 32, e0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, e = e0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < h && e < E) ? w_r[(size_t)k * E + e] : __float2bfloat16_rn(0.f);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int e = e0 + i, k = k0 + threadIdx.x;
    if (e < EP && k < h) wt[(size_t)e * h + k] = tile[threadIdx.x][i];
  }
}

// kMN: B = router_w [h][E] read directly (MN-major, 64-expert x 64-k TMA boxes);
// otherwise B = the transposed copy [EP][h] (K-major).
// One CTA = 128 tokens (one hist-block); 6 warps: 0-3 epilogue (thread = token =
// TMEM lane), 4 TMA producer, 5 MMA issuer.
// kK = 2 (top-2, reading R21): the two largest logits per token (ties: lowest index), two
// records per token (out[2 t + j], j = 0 the larger), both counted in the histogram.
template <bool kMN, int kK = 1>
__global__ void __launch_bounds__(192, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     int n, int h, int E, int EP, const int32_t* __restrict__ forced,
                     RouteRec* __restrict__ out, int32_t* __restrict__ hist_out,
                     int32_t* __restrict__ err_flag, int RTC_STAGES) {
  using namespace ptx;
  constexpr int kTok = RTC_TOK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int n_atoms = (EP + 63) / 64;
  const int b_bytes = kMN ? n_atoms * 8192 : EP * 128;
  __shared__ int32_t s_hist[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  constexpr int a_stage = kTok * 128;   // kTok rows x 64 k x 2 B
  uint8_t* sA = smem;
  uint8_t* sB = smem + RTC_STAGES * a_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + RTC_STAGES * b_bytes);
  uint64_t* empty = full + RTC_STAGES;
  uint64_t* done = empty + RTC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ncols = EP <= 32 ? 32 : EP <= 64 ? 64 : EP <= 128 ? 128 : 256;
  if (threadIdx.x == 0) TL_MIN(0);

  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < RTC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: x may come from the previous kernel, and the previous forward's FFN
  // still reads the route records this kernel overwrites
  griddep_wait();
  if (threadIdx.x == 0) { TL_MIN(1); TL_MAX(1); }
  // the previous forward's FFN is done with the "tables published" flag (tb.stats[6],
  // = err_flag + 3): clear it for this forward's grouping launch to set
  if (blockIdx.x == 0 && threadIdx.x == 0) err_flag[3] = 0;
  griddep_launch_dependents();
  const int tok0 = blockIdx.x * kTok;
  const int nkb = h / 64;

  if (warp == 4) {
    // TMA producer (warp-uniform loop, one elected lane issues)
    // x stays in L2 for the grouping launch, which re-reads every row (A/B: -0.35 us / step)
    const uint64_t pol_x = policy_evict_normal();
    const uint64_t pol_w = policy_evict_last();
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], a_stage + b_bytes);
        tma_load_2d(&tmX, &full[s], sA + s * a_stage, kb * 64, tok0, pol_x);
        if (kMN) {
          for (int a = 0; a < n_atoms; ++a)
            tma_load_2d(&tmW, &full[s], sB + s * b_bytes + a * 8192, a * 64, kb * 64, pol_w);
        } else {
          tma_load_2d(&tmW, &full[s], sB + s * b_bytes, kb * 64, 0, pol_w);  // box = EP rows
        }
      }
      __syncwarp();
      if (++s == RTC_STAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp == 5) {
    // MMA issuer (warp-uniform loop, one elected lane issues)
    const uint32_t idesc = idesc_bf16_f32(128, EP, kMN);
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint64_t ad = smem_desc_k_sw128(smem_u32(sA + s * a_stage));
      const uint64_t bd = kMN ? smem_desc_mn_sw128(smem_u32(sB + s * b_bytes), 8192)
                              : smem_desc_k_sw128(smem_u32(sB + s * b_bytes));
      const uint32_t bstep = kMN ? 128 : 2;   // K=16 step: 16 rows x 128 B (MN) or 32 B (K)
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_bf16_ss(tmem, ad + 2 * k, bd + bstep * k, idesc, (kb | k) != 0);
        mma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == RTC_STAGES) { s = 0; ph ^= 1; }
    }
    if (elect_one()) mma_commit(done);
    __syncwarp();
  } else {
    // epilogue: warps 0-3, thread = token (TMEM lane 32*warp + lane)
    const int t = tok0 + warp * 32 + lane;
    int sel = -1, sel2 = -1;
    bool bad = false;
    if (forced != nullptr && t < n) {
      sel = forced[static_cast<size_t>(t) * kK];
      if (sel < 0 || sel >= E) {
        bad = true;
        sel = sel < 0 ? 0 : E - 1;
      }
      if (kK == 2) {
        sel2 = forced[static_cast<size_t>(t) * kK + 1];
        if (sel2 < 0 || sel2 >= E) {
          bad = true;
          sel2 = sel2 < 0 ? 0 : E - 1;
        }
      }
    }
    mbar_wait(done, 0);
    tc_fence_after();
    if (threadIdx.x == 0) { TL_MIN(2); TL_MAX(2); }
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    // one pass over the logit row, 32 columns per TMEM load: columns >= E are
    // masked to -inf; chunk max by a tree, argmax = the smallest column attaining
    // it (lowest index on ties, R4) by a tree of index minima, then a running
    // (max, sum exp(l - max)) pair rescaled when the max moves. A later chunk
    // replaces the running argmax only with a strictly larger max, so ties across
    // chunks also resolve to the lowest index.
    constexpr float kLog2e = 1.4426950408889634f;
    float best = -INFINITY, lsel = 0.f, lsel2 = 0.f, sum = 0.f;
    int best_e = 0;
    float top1 = -INFINITY, top2 = -INFINITY;   // kK == 2: the two largest logits ...
    int top1_e = 0, top2_e = 0;                 // ... and their experts (lowest index on ties)
    for (int c0 = 0; c0 < EP; c0 += 32) {
      uint32_t r[32];
      if (c0 + 16 < EP) {
        tmem_ld32(taddr + c0, r);
      } else {
        uint32_t (&r16)[16] = *reinterpret_cast<uint32_t(*)[16]>(&r[0]);
        tmem_ld16(taddr + c0, r16);
#pragma unroll
        for (int j = 16; j < 32; ++j) r[j] = 0xff800000u;  // -inf
      }
      tmem_ld_wait();
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = (c0 + j < E) ? __uint_as_float(r[j]) : -INFINITY;
      float m[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) m[j] = fmaxf(v[j], v[j + 16]);
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) m[j] = fmaxf(m[j], m[j + w]);
      const float cmax = m[0];
      int ix[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        ix[j] = min(v[j] == cmax ? j : 32, v[j + 16] == cmax ? j + 16 : 32);
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) ix[j] = min(ix[j], ix[j + w]);
      if (sel >= c0 && sel < c0 + 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j == sel) lsel = v[j];
      }
      if (kK == 2) {
        if (sel2 >= c0 && sel2 < c0 + 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j == sel2) lsel2 = v[j];
        }
        // insertion in scan order: only a strictly larger value displaces, so ties keep the
        // lower expert index ahead
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = v[j];
          if (x > top1) {
            top2 = top1;
            top2_e = top1_e;
            top1 = x;
            top1_e = c0 + j;
          } else if (x > top2) {
            top2 = x;
            top2_e = c0 + j;
          }
        }
      }
      if (cmax > best) {
        sum *= fast_exp2((best - cmax) * kLog2e);   // best = -inf on the first chunk -> 0
        best = cmax;
        best_e = c0 + ix[0];
      }
      const float mb = best * kLog2e;
      float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        p0 += fast_exp2(fmaf(v[j], kLog2e, -mb));
        p1 += fast_exp2(fmaf(v[j + 1], kLog2e, -mb));
        p2 += fast_exp2(fmaf(v[j + 2], kLog2e, -mb));
        p3 += fast_exp2(fmaf(v[j + 3], kLog2e, -mb));
      }
      sum += (p0 + p1) + (p2 + p3);
    }
    if (t < n && kK == 1) {
      RouteRec rec;
      rec.expert = sel >= 0 ? sel : best_e;
      rec.gate = (sel >= 0 ? fast_exp2((lsel - best) * kLog2e) : 1.f) / sum;
      out[t] = rec;
      atomicAdd(&s_hist[rec.expert], 1);
      if (bad) atomicOr(err_flag, 1);
    } else if (t < n) {
      RouteRec r0, r1;
      r0.expert = sel >= 0 ? sel : top1_e;
      r1.expert = sel >= 0 ? sel2 : top2_e;
      r0.gate = fast_exp2(((sel >= 0 ? lsel : top1) - best) * kLog2e) / sum;
      r1.gate = fast_exp2(((sel >= 0 ? lsel2 : top2) - best) * kLog2e) / sum;
      out[2 * static_cast<size_t>(t)] = r0;
      out[2 * static_cast<size_t>(t) + 1] = r1;
      atomicAdd(&s_hist[r0.expert], 1);
      atomicAdd(&s_hist[r1.expert], 1);
      if (bad) atomicOr(err_flag, 1);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // the epilogue warps
    for (int e = threadIdx.x; e < E; e += kTok) hist_out[(size_t)blockIdx.x * E + e] = s_hist[e];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, ncols);
  if (threadIdx.x == 0) TL_MAX(0);
}

}  // namespace

TL_EXPORT(moeshard_tl_router)

// Ring stages: as deep as RTC_SMEM_BUDGET allows, except when the grid is more than one
// wave of one CTA per SM (C5: 256 blocks of 128 tokens on 148 SMs): then half the budget,
// so two CTAs share an SM and the grid runs as one wave.
int router_tc_stages(int EP, bool mn, int blocks, int num_sms) {
  const int b = mn ? ((EP + 63) / 64) * 8192 : EP * 128;
  const int a = RTC_TOK * 128;
  const int budget = blocks > num_sms ? 110 * 1024 : RTC_SMEM_BUDGET;   // 2 x 3 stages fit 228 KB
  return std::max(2, std::min(RTC_MAX_STAGES, budget / (a + b)));
}
size_t router_tc_smem_bytes(int EP, bool mn, int stages) {
  const int b = mn ? ((EP + 63) / 64) * 8192 : EP * 128;
  const int a = RTC_TOK * 128;
  return 1024 + stages * (a + b) + (2 * stages + 1) * 8 + 16;
}

namespace {
template <int kK>
cudaError_t launch_router_tc_k(const CUtensorMap& tmX, const CUtensorMap& tmW, bool mn_major,
                               const void* w_r, void* wt_r, int n, int h, int E, int EP,
                               const int32_t* forced, RouteRec* out, int32_t* hist_out,
                               int32_t* err_flag, cudaStream_t s, int num_sms) {
  static PerDeviceOnce attr;
  if (attr.need()) {
    cudaError_t e = cudaFuncSetAttribute(router_tc_kernel<true, kK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         RTC_SMEM_BUDGET + 2048);  // >= router_tc_smem_bytes(any EP)
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(router_tc_kernel<false, kK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, RTC_SMEM_BUDGET + 2048);
    if (e != cudaSuccess) return e;
    attr.done();
  }
  const dim3 grid(ceil_div(n, RTC_TOK));
  if (mn_major) {
    const int st = router_tc_stages(EP, true, grid.x, num_sms);
    return launch_pdl(router_tc_kernel<true, kK>, grid, dim3(192), router_tc_smem_bytes(EP, true, st),
                      s, tmX, tmW, n, h, E, EP, forced, out, hist_out, err_flag, st);
  }
  dim3 tg(ceil_div(h, 32), ceil_div(EP, 32)), tb(32, 8);
  router_transpose<<<tg, tb, 0, s>>>(static_cast<const __nv_bfloat16*>(w_r), h, E, EP,
                                     static_cast<__nv_bfloat16*>(wt_r));
  const int st = router_tc_stages(EP, false, grid.x, num_sms);
  router_tc_kernel<false, kK><<<grid, 192, router_tc_smem_bytes(EP, false, st), s>>>(
      tmX, tmW, n, h, E, EP, forced, out, hist_out, err_flag, st);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_router_tc(const CUtensorMap& tmX, const CUtensorMap& tmW, bool mn_major,
                             const void* w_r, void* wt_r, int n, int h, int E, int EP,
                             const int32_t* forced, RouteRec* out, int32_t* hist_out,
                             int32_t* err_flag, cudaStream_t s, int top_k, int num_sms) {
  if (n <= 0) return cudaSuccess;
  if (top_k == 2)
    return launch_router_tc_k<2>(tmX, tmW, mn_major, w_r, wt_r, n, h, E, EP, forced, out, hist_out,
                                 err_flag, s, num_sms);
  return launch_router_tc_k<1>(tmX, tmW, mn_major, w_r, wt_r, n, h, E, EP, forced, out, hist_out,
                               err_flag, s, num_sms);
}

}  // namespace moeshard
