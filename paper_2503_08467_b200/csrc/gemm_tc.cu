// gemm_tc.cu - Step 4 expert computation as ONE
// tcgen05 grouped GEMM per projection covering every expert's shard (the
// Sec. 3.3 launch fusion), bf16 x bf16 -> fp32 in TMEM.
//
// Swap-AB formulation: the weight shard is the MMA "A" operand (M = 128
// output features per tile) and the tokens of one expert are the "B"
// operand (N = 16..256 tokens, any multiple of 16), so an expert's ragged
// token count is padded to 16 rows, not to 128 (SURVEY.md §7 tile
// quantisation). Both operands are K-major in shared memory with the
// 128-B swizzle and arrive by TMA:
//   up:   D[f, t] = sum_k WiT[e][f][k] * Xp[t][k]      K = h,   f < F = d_ff/G
//         epilogue: H[t][f] = bf16(relu(D))                      (ReLU fused, R1)
//   down: D[c, t] = sum_f WoT[e][c][f] * H[t][f]       K = F,   c < h
//         epilogue: out[perm[t]][c] = bf16(gate[perm[t]] * D)   (gate + un-permute fused, R2)
//
// Persistent kernel, one CTA per SM, warp-specialised:
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      MMA issuer (one elected lane), double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld -> registers -> global (lane quadrant = warp % 4)
// Work units (expert e, 128-feature tile mt, token chunk c) are decoded on
// the device from the segment tables written by the grouping kernels, so no
// host round-trip is needed (CUDA-graph capturable). Units of the same
// (e, mt) are adjacent, so concurrently running CTAs share each weight tile
// through L2 and the weights stream from HBM once.
#include "common.cuh"
#include "gemm_tc.cuh"
#include "ptx.cuh"

namespace moeshard {
namespace {

using namespace ptx;

constexpr int BM = kTcFeatTile;  // 128
constexpr int BK = 64;           // 64 bf16 = 128 B = one swizzle atom row
constexpr int BN_MAX = kTcTokTile;
constexpr int B_BOX = 32;        // TMA box rows for the token operand
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_BYTES = BN_MAX * BK * 2;   // 32 KB
constexpr int B_BOX_BYTES = B_BOX * BK * 2;  // 4 KB
constexpr int TMEM_COLS = 512;             // 2 accumulators x 256 fp32 columns
constexpr int kThreads = 256;

struct Unit {
  int e, mt, tok0, ntok;
};

__device__ __forceinline__ Unit decode(int u, int n_mt, int E, const int32_t* pref,
                                       const int32_t* off, const int32_t* csz) {
  const int q = u / n_mt;
  int lo = 0, hi = E;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= q) lo = mid; else hi = mid;
  }
  Unit w;
  w.e = lo;
  const int nch = pref[lo + 1] - pref[lo];
  const int local = u - pref[lo] * n_mt;
  w.mt = local / nch;
  const int c = local - w.mt * nch;
  const int cs = csz[lo];
  w.tok0 = off[lo] + c * cs;
  w.ntok = min(cs, off[lo + 1] - w.tok0);
  return w;
}

template <bool kDown>
__global__ void __launch_bounds__(kThreads, 1)
    tc_grouped_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_pref = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_off = s_pref + (p.E + 1);
  int32_t* s_cs = s_off + (p.E + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i <= p.E; i += kThreads) {
    s_pref[i] = p.tb.tc_chunk_pref[i];
    s_off[i] = p.tb.offsets[i];
    if (i < p.E) s_cs[i] = p.tb.tc_chunk_size[i];
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_mt = p.n_mt;
  const int total = s_pref[p.E] * n_mt;
  const int nkb = p.K / BK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first();  // weights: streamed, shared only by siblings
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by n_mt tiles
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        const Unit w = decode(u, n_mt, p.E, s_pref, s_off, s_cs);
        const int nb = (w.ntok + B_BOX - 1) / B_BOX;
        const uint32_t bytes = A_BYTES + nb * B_BOX_BYTES;
        const int arow = w.e * p.rows_per_e + w.mt * BM;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d(&tmA, &full[stage], sA + stage * A_BYTES, kb * BK, arow, pol_w);
          for (int i = 0; i < nb; ++i)
            tma_load_2d(&tmB, &full[stage], sB + stage * B_BYTES + i * B_BOX_BYTES, kb * BK,
                        w.tok0 + i * B_BOX, pol_x);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        const Unit w = decode(u, n_mt, p.E, s_pref, s_off, s_cs);
        const int nmma = (w.ntok + 15) & ~15;
        const uint32_t idesc = idesc_bf16_f32(BM, nmma);
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN_MAX;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_k_sw128(smem_u32(sA + stage * A_BYTES));
          const uint64_t bd = smem_desc_k_sw128(smem_u32(sB + stage * B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[as]);
        as ^= 1;
        if (as == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int wq = warp & 3;
    int as = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit w = decode(u, n_mt, p.E, s_pref, s_off, s_cs);
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const int f = w.mt * BM + wq * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + as * BN_MAX;
      const int nmma = (w.ntok + 15) & ~15;
      for (int c0 = 0; c0 < nmma; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
        tmem_ld_wait();
        if (kDown) {
          int row = 0;
          float g = 0.f;
          const int tk = c0 + (lane & 15);
          if (tk < w.ntok) {
            row = p.perm[w.tok0 + tk];
            g = p.route[row].gate;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int rj = __shfl_sync(0xffffffffu, row, j);
            const float gj = __shfl_sync(0xffffffffu, g, j);
            if (c0 + j < w.ntok)
              p.out[(size_t)rj * p.ld_out + f] = __float2bfloat16_rn(gj * __uint_as_float(r[j]));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < w.ntok)
              p.out[(size_t)(w.tok0 + c0 + j) * p.ld_out + f] =
                  __float2bfloat16_rn(fmaxf(__uint_as_float(r[j]), 0.f));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

size_t smem_bytes(int E) {
  return 1024 + STAGES * (A_BYTES + B_BYTES) + (2 * STAGES + 4) * 8 + 16 + (3 * E + 2) * 4;
}

template <bool kDown>
cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const TcParams& p, int grid,
                     cudaStream_t s) {
  const size_t sm = smem_bytes(p.E);
  static bool attr_set = false;  // per template instance; the library is single-device
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_grouped_gemm<kDown>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes(kMaxExperts)));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  tc_grouped_gemm<kDown><<<grid, kThreads, sm, s>>>(tmA, tmB, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tc_gemm(bool down, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const TcParams& p, int grid, cudaStream_t s) {
  return down ? launch_t<true>(tmA, tmB, p, grid, s) : launch_t<false>(tmA, tmB, p, grid, s);
}

}  // namespace moeshard
