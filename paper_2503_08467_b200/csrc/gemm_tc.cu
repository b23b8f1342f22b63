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
//   warp 0      TMA producer of the weight tiles (one lane), A_STAGES-deep ring
//   warp 3      TMA producer of the token tiles (one lane), B_STAGES-deep ring
//   warp 1      MMA issuer (one lane), double-buffered TMEM accumulator
//   warp 2      TMEM allocator (and, dynamic scheduling, the unit scheduler)
//   warps 4-    epilogue: tcgen05.ld -> registers -> global (lane quadrant = warp % 4);
//               the fused kernel (tc_moe_ffn_2sm, the product path) has 8 of them, two per
//               quadrant, and transposes each 16-token chunk through stmatrix (the drain of
//               the accumulators bounds it: profiles/r02/experiments_r02.md)
// Work units (expert e, 128-feature tile mt, token chunk c) are decoded on
// the device from the segment tables written by the grouping kernels, so no
// host round-trip is needed (CUDA-graph capturable). Units of the same
// (e, mt) are adjacent, so concurrently running CTAs share each weight tile
// through L2 and the weights stream from HBM once.
#include "common.cuh"
#include "gemm_tc.cuh"
#include "ptx.cuh"
#include "timeline.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace moeshard {
namespace {

using namespace ptx;

constexpr int BM = kTcFeatTile;  // 128
constexpr int BK = 64;           // 64 bf16 = 128 B = one swizzle atom row
constexpr int BN_MAX = kTcTokTile;
constexpr int B_BOX = 32;        // TMA box rows for the token operand
constexpr int A_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_BYTES = BN_MAX * BK * 2;   // 32 KB
constexpr int B_BOX_BYTES = B_BOX * BK * 2;  // 4 KB
constexpr int TMEM_COLS = 512;             // 2 accumulators x 256 fp32 columns
constexpr int ACC_STRIDE = 256;            // TMEM columns between the two accumulators
constexpr int kThreads = 256;

struct Unit {
  int e, mt, tok0, ntok;
  int chunk;   // global token-chunk id (pref[e] + chunk of e)
};

// pref: cumulative chunks [E+1]; pos: internal segment starts; end: pos + count; csz: chunk size
__device__ __forceinline__ Unit decode(int u, int n_mt, int E, const int32_t* pref,
                                       const int32_t* pos, const int32_t* end,
                                       const int32_t* csz) {
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
  w.chunk = pref[lo] + c;
  const int cs = csz[lo];
  w.tok0 = pos[lo] + c * cs;
  w.ntok = min(cs, end[lo] - w.tok0);
  return w;
}

// Unit list of one launch: every (expert, tile, chunk) of the forward, or - launch-mode
// ablation - only expert p.only_e (optionally restricted to source rank p.only_g's rows),
// chunked on its own.
struct UnitList {
  int total;        // units in this launch
  int e, lo, hi, nc, cs;   // restricted mode: expert, row range, chunks, chunk rows
};
__device__ __forceinline__ UnitList unit_list(const TcParams& p, int n_units_per_chunk,
                                              const int32_t* pref, const int32_t* pos,
                                              const int32_t* end) {
  UnitList L{};
  if (p.only_e < 0) {
    L.total = pref[p.E] * n_units_per_chunk;
    L.e = -1;
    return L;
  }
  L.e = p.only_e;
  L.lo = pos[L.e];
  L.hi = end[L.e];
  if (p.only_g >= 0) {
    const int32_t* b = p.block_base;
    const int g = p.only_g;
    const int lo_rel = b[static_cast<size_t>(g) * p.nbr * p.E + L.e];
    const int hi_rel = g + 1 < p.n_src ? b[static_cast<size_t>(g + 1) * p.nbr * p.E + L.e]
                                       : end[L.e] - pos[L.e];
    L.hi = L.lo + hi_rel;
    L.lo += lo_rel;
  }
  tc_chunking(L.hi - L.lo, &L.nc, &L.cs);
  L.total = L.nc * n_units_per_chunk;
  return L;
}
__device__ __forceinline__ Unit unit_at(const UnitList& L, int u, int n_mt, int E,
                                        const int32_t* pref, const int32_t* pos,
                                        const int32_t* end, const int32_t* csz) {
  if (L.e < 0) return decode(u, n_mt, E, pref, pos, end, csz);
  Unit w;
  w.e = L.e;
  w.mt = u / L.nc;
  const int c = u - w.mt * L.nc;
  w.chunk = c;
  w.tok0 = L.lo + c * L.cs;
  w.ntok = min(L.cs, L.hi - w.tok0);
  return w;
}

// Epilogue of one tile: TMEM accumulator (lane = output feature of this
// warp's 32-feature slice, column = token) -> fused ReLU (up) or gate x (down)
// -> bf16 -> a per-warp 1 KB shared staging buffer [16 tokens][32 features]
// -> 16-B vector stores (up: row tok0+j of H; down: un-permute scatter to row
// perm[tok0+j] of the output). One 16-token chunk at a time.
// NH warps share one 32-feature quadrant: warp half eh (< NH) takes the 16-token column
// chunks eh, eh + NH, ... (NH = 2 halves the drain latency of a tile).
// down: the destination rows perm[j] and gates of a unit's tokens, fetched up front
// (lane holds tokens lane + 32 i) so the store loop has no dependent global loads. With
// p.gate_pad (gate per expert-ordered row, written by Step 2 beside perm_pad) both loads
// are independent: one latency instead of perm's then route[perm].gate's.
__device__ __forceinline__ void load_rows_gates(const TcParams& p, int tok0, int ntok, int lane,
                                                int (&rows_r)[BN_MAX / 32], float (&g_r)[BN_MAX / 32]) {
#pragma unroll
  for (int i = 0; i < BN_MAX / 32; ++i) {
    const int tk = lane + 32 * i;
    rows_r[i] = tk < ntok ? __ldg(p.perm + tok0 + tk) : 0;
    if (p.gate_pad) g_r[i] = tk < ntok ? __ldg(p.gate_pad + tok0 + tk) : 0.f;
  }
  if (!p.gate_pad) {
#pragma unroll
    for (int i = 0; i < BN_MAX / 32; ++i) {
      const int tk = lane + 32 * i;
      g_r[i] = tk < ntok ? __ldg(&p.route[rows_r[i]].gate) : 0.f;
    }
  }
}

// The same for an epilogue warp that drains column chunks eh, eh + NH, ... of a tile
// (store_tile_stm): register `it` holds the token of its it-th chunk at lane & 15, so every
// register index in the drain loop is a compile-time constant whatever eh is.
template <int NH>
__device__ __forceinline__ void load_rows_gates_chunked(const TcParams& p, int tok0, int ntok,
                                                        int lane, int eh,
                                                        int (&rows_r)[BN_MAX / 32],
                                                        float (&g_r)[BN_MAX / 32]) {
  constexpr int kChunks = (BN_MAX / 16 + NH - 1) / NH;
  static_assert(kChunks <= BN_MAX / 32, "two or more warps per lane quadrant");
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    const int tk = 16 * eh + 16 * NH * it + (lane & 15);
    rows_r[it] = tk < ntok ? __ldcg(p.perm + tok0 + tk) : 0;
    if (p.gate_pad) g_r[it] = tk < ntok ? __ldcg(p.gate_pad + tok0 + tk) : 0.f;
  }
  if (!p.gate_pad) {
#pragma unroll
    for (int it = 0; it < kChunks; ++it) {
      const int tk = 16 * eh + 16 * NH * it + (lane & 15);
      g_r[it] = tk < ntok ? __ldg(&p.route[rows_r[it]].gate) : 0.f;
    }
  }
}

// kPre: rows_r / g_r were loaded by the caller (load_rows_gates) ahead of the
// accumulator wait; otherwise (down) they are loaded here.
template <bool kDown, int NH = 1, bool kPre = false>
__device__ __forceinline__ void store_tile(const TcParams& p, int tok0, int ntok, int nmma,
                                           int fbase, uint32_t taddr, int lane, uint64_t pol_keep,
                                           __nv_bfloat16* stage, int eh, int (&rows_r)[BN_MAX / 32],
                                           float (&g_r)[BN_MAX / 32]) {
  uint16_t* st16 = reinterpret_cast<uint16_t*>(stage);
  if (kDown && !kPre) load_rows_gates(p, tok0, ntok, lane, rows_r, g_r);
  // TMEM reads are double-buffered: the load of the next chunk is in flight while
  // this one is converted and stored
  uint32_t rbuf[2][16];
  const int first = 16 * eh;
#ifdef MOESHARD_EXP_NO_TMEMLD
#pragma unroll
  for (int j = 0; j < 16; ++j) rbuf[0][j] = rbuf[1][j] = __float_as_uint(static_cast<float>(lane + j));
#else
  if (first < nmma) {
    tmem_ld16(taddr + first, rbuf[0]);
    tmem_ld_wait(rbuf[0]);
  }
#endif
#pragma unroll
  for (int it = 0; it < (BN_MAX / 16 + NH - 1) / NH; ++it) {
    const int c0 = first + 16 * NH * it;
    if (c0 >= nmma) break;
    uint32_t (&r)[16] = rbuf[it & 1];
    uint32_t (&rn)[16] = rbuf[(it + 1) & 1];
    const int cn = c0 + 16 * NH;
#ifndef MOESHARD_EXP_NO_TMEMLD
    if (cn < nmma) tmem_ld16(taddr + cn, rn);
#endif
    int row = 0;
    if (kDown) {
      // token c0 + (lane & 15) lives in lane (c0 & 16) + (lane & 15), register c0 / 32
      // (= 16 NH it / 32 for any eh: a compile-time index)
      const int ri = (16 * NH * it) >> 5;
      const int src = (c0 & 16) + (lane & 15);
      row = __shfl_sync(0xffffffffu, rows_r[ri], src);
      const float g = __shfl_sync(0xffffffffu, g_r[ri], src);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float gj = __shfl_sync(0xffffffffu, g, j);
        const __nv_bfloat16 v = __float2bfloat16_rn(gj * __uint_as_float(r[j]));
        st16[j * 32 + lane] = *reinterpret_cast<const uint16_t*>(&v);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16 v = __float2bfloat16_rn(fmaxf(__uint_as_float(r[j]), 0.f));
        st16[j * 32 + lane] = *reinterpret_cast<const uint16_t*>(&v);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int q = lane + 32 * i;  // 64 vectors of 16 B: 16 tokens x 4 parts
      const int j = q >> 2, part = q & 3;
      const uint4 v = reinterpret_cast<const uint4*>(stage)[q];
      if (kDown) {
        const int rj = __shfl_sync(0xffffffffu, row, j);
        if (c0 + j < ntok) {
          __nv_bfloat16* dst;
          if (p.p2p_n > 0) {   // the owner's receive slot for this rank, over NVLink
            const int o = rj / p.p2p_n;
            dst = p.p2p_out[o] + (size_t)(rj - o * p.p2p_n) * p.ld_out;
          } else {
            dst = p.out + (size_t)rj * p.ld_out;
          }
#ifdef MOESHARD_EXP_NO_STG
          if (v.x == 0x12345678u && v.y == 0x9abcdefu)
#endif
          *reinterpret_cast<uint4*>(dst + fbase + part * 8) = v;
        }
      } else if (c0 + j < ntok) {
#ifdef MOESHARD_EXP_NO_STG
        if (v.x == 0x12345678u && v.y == 0x9abcdefu)
#endif
        st_v4_hint(p.out + (size_t)(tok0 + c0 + j) * p.ld_out + fbase + part * 8, v, pol_keep);
      }
    }
    __syncwarp();
#ifndef MOESHARD_EXP_NO_TMEMLD
    if (cn < nmma) tmem_ld_wait(rn);
#endif
  }
}

// The fused kernel's epilogue of one tile, transposed by stmatrix: each 16-token column
// chunk is read from TMEM in the mma fragment layout (tcgen05.ld 16x256b: a thread holds two
// features x two adjacent tokens per 8 x 8 block), packed to bf16 pairs and written to the
// warp's staging buffer [16 tokens][32 features] with two stmatrix.trans.x4 (instead of 16
// two-byte shared stores), then stored as 16-B row segments as in store_tile. Rows of the
// staging buffer are kStmRow = 80 B apart (conflict-free stmatrix rows).
constexpr int kStmRow = 80;
constexpr int kStmStage = 16 * kStmRow;   // bytes per epilogue warp
template <bool kDown, int NH>
__device__ __forceinline__ void store_tile_stm(const TcParams& p, int tok0, int ntok, int nmma,
                                               int fbase, uint32_t taddr, int lane,
                                               uint64_t pol_keep, uint8_t* stage, int eh,
                                               int (&rows_r)[BN_MAX / 32],
                                               float (&g_r)[BN_MAX / 32]) {
  const int m = lane >> 3, k = lane & 7;   // stmatrix: matrix m, stored row (token) k
  const uint32_t row_addr = smem_u32(stage) + ((m >> 1) * 8 + k) * kStmRow + (m & 1) * 16;
  const int tq = 2 * (lane & 3);           // this thread's first token of each 8-token block
  uint32_t rb[2][2][8];                    // [buffer][lane half][regs]
  const int first = 16 * eh;
  if (first < nmma) {
    tmem_ld_16x256b_x2(taddr + first, rb[0][0]);
    tmem_ld_16x256b_x2(taddr + (16u << 16) + first, rb[0][1]);
    tmem_ld_wait8(rb[0][0], rb[0][1]);
  }
#pragma unroll
  for (int it = 0; it < (BN_MAX / 16 + NH - 1) / NH; ++it) {
    const int c0 = first + 16 * NH * it;
    if (c0 >= nmma) break;
    uint32_t (&ra)[2][8] = rb[it & 1];
    uint32_t (&rn)[2][8] = rb[(it + 1) & 1];
    const int cn = c0 + 16 * NH;
    if (cn < nmma) {
      tmem_ld_16x256b_x2(taddr + cn, rn[0]);
      tmem_ld_16x256b_x2(taddr + (16u << 16) + cn, rn[1]);
    }
    int row = 0;
    float g0 = 1.f, g1 = 1.f, g8 = 1.f, g9 = 1.f;
    if (kDown) {
      // this warp's it-th chunk: token c0 + i lives in lane i of register it
      // (load_rows_gates_chunked)
      row = __shfl_sync(0xffffffffu, rows_r[it], lane & 15);
      g0 = __shfl_sync(0xffffffffu, g_r[it], tq);
      g1 = __shfl_sync(0xffffffffu, g_r[it], tq + 1);
      g8 = __shfl_sync(0xffffffffu, g_r[it], tq + 8);
      g9 = __shfl_sync(0xffffffffu, g_r[it], tq + 9);
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint32_t* r = ra[hh];
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
      if (kDown) {
        v[0] *= g0; v[1] *= g1; v[2] *= g0; v[3] *= g1;
        v[4] *= g8; v[5] *= g9; v[6] *= g8; v[7] *= g9;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      // matrices: 0 = features 16hh+0..7 x tokens 0..7, 1 = features +8..15 x tokens 0..7,
      // 2 = features 0..7 x tokens 8..15, 3 = features 8..15 x tokens 8..15
      stmatrix_x4_trans(row_addr + hh * 32, pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                        pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int q = lane + 32 * i;  // 64 vectors of 16 B: 16 tokens x 4 parts
      const int j = q >> 2, part = q & 3;
      const uint4 v = *reinterpret_cast<const uint4*>(stage + j * kStmRow + part * 16);
      if (kDown) {
        const int rj = __shfl_sync(0xffffffffu, row, j);
        if (c0 + j < ntok) {
          __nv_bfloat16* dst;
          if (p.p2p_n > 0) {   // the owner's receive slot for this rank, over NVLink
            const int o = rj / p.p2p_n;
            dst = p.p2p_out[o] + (size_t)(rj - o * p.p2p_n) * p.ld_out;
          } else {
            dst = p.out + (size_t)rj * p.ld_out;
          }
          *reinterpret_cast<uint4*>(dst + fbase + part * 8) = v;
        }
      } else if (c0 + j < ntok) {
        st_v4_hint(p.out + (size_t)(tok0 + c0 + j) * p.ld_out + fbase + part * 8, v, pol_keep);
      }
    }
    __syncwarp();
    if (cn < nmma) tmem_ld_wait8(rn[0], rn[1]);
  }
}

// One-CTA kernel (M = 128): the unfused two-launch ablation when a projection has an
// odd number of 128-feature tiles.
template <bool kDown, int A_STAGES, int B_STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_grouped_gemm(const __grid_constant__ CUtensorMap tmB, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_STAGES * A_BYTES;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(sB + B_STAGES * B_BYTES);
  uint64_t* emptyA = fullA + A_STAGES;
  uint64_t* fullB = emptyA + A_STAGES;
  uint64_t* emptyB = fullB + B_STAGES;
  uint64_t* tfull = emptyB + B_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_pref = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_off = s_pref + (p.E + 1);   // internal segment starts (pos)
  int32_t* s_cs = s_off + (p.E + 1);
  int32_t* s_end = s_cs + p.E;           // pos + count

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i <= p.E; i += kThreads) {
    s_pref[i] = p.tb.tc_chunk_pref[i];
    s_off[i] = p.tb.pos[i];
    if (i < p.E) {
      s_cs[i] = p.tb.tc_chunk_size[i];
      s_end[i] = p.tb.pos[i] + p.tb.counts[i];
    }
  }
  if (warp == 3 && lane == 0) tma_prefetch_desc(&tmB);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < B_STAGES; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
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
  const UnitList UL = unit_list(p, n_mt, s_pref, s_off, s_end);
  const int total = UL.total;
  const int nkb = p.K / BK;

  if (warp == 0) {
    // -------------------------------------------------------------- weight producer
    const uint64_t pol_w = policy_evict_first();  // weights: streamed, shared only by siblings
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit w = unit_at(UL, u, n_mt, p.E, s_pref, s_off, s_end, s_cs);
      const __nv_bfloat16* tiles =
          p.a_tiles + (static_cast<size_t>(w.e) * n_mt + w.mt) * nkb * (BM * BK);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&emptyA[stage], phase ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&fullA[stage], A_BYTES);
          bulk_load(sA + stage * A_BYTES, tiles + static_cast<size_t>(kb) * (BM * BK), A_BYTES,
                    &fullA[stage], pol_w);
        }
        __syncwarp();
        if (++stage == A_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 3) {
    // -------------------------------------------------------------- token producer
    const uint64_t pol_x = policy_evict_last();   // activations: re-read by n_mt tiles
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit w = unit_at(UL, u, n_mt, p.E, s_pref, s_off, s_end, s_cs);
      const int nb = (w.ntok + B_BOX - 1) / B_BOX;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&emptyB[stage], phase ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&fullB[stage], nb * B_BOX_BYTES);
          for (int i = 0; i < nb; ++i)
            tma_load_2d(&tmB, &fullB[stage], sB + stage * B_BYTES + i * B_BOX_BYTES, kb * BK,
                        w.tok0 + i * B_BOX, pol_x);
        }
        __syncwarp();
        if (++stage == B_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    int sa = 0, sb = 0;
    uint32_t pa = 0, pb = 0;
    int as = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit w = unit_at(UL, u, n_mt, p.E, s_pref, s_off, s_end, s_cs);
      const int nmma = (w.ntok + 15) & ~15;
      const uint32_t idesc = idesc_bf16_f32(BM, nmma);
      mbar_wait(&tempty[as], aphase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * ACC_STRIDE;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&fullB[sb], pb);
        mbar_wait(&fullA[sa], pa);
        tc_fence_after();
        const uint64_t ad = smem_desc_k_sw128(smem_u32(sA + sa * A_BYTES));
        const uint64_t bd = smem_desc_k_sw128(smem_u32(sB + sb * B_BYTES));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&emptyA[sa]);
          mma_commit(&emptyB[sb]);
        }
        __syncwarp();
        if (++sa == A_STAGES) {
          sa = 0;
          pa ^= 1;
        }
        if (++sb == B_STAGES) {
          sb = 0;
          pb ^= 1;
        }
      }
      if (elect_one()) mma_commit(&tfull[as]);
      __syncwarp();
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int wq = warp & 3;
    __nv_bfloat16* stage = reinterpret_cast<__nv_bfloat16*>(
        (reinterpret_cast<uintptr_t>(s_end + p.E) + 15) & ~static_cast<uintptr_t>(15)) + wq * 512;
    const uint64_t pol_keep = policy_evict_last();  // H is re-read by the down product
    int as = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit w = unit_at(UL, u, n_mt, p.E, s_pref, s_off, s_end, s_cs);
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + as * ACC_STRIDE;
      int rows_r[BN_MAX / 32];
      float g_r[BN_MAX / 32];
      store_tile<kDown>(p, w.tok0, w.ntok, (w.ntok + 15) & ~15, w.mt * BM + wq * 32, taddr, lane,
                        pol_keep, stage, 0, rows_r, g_r);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
    if (kDown && p.p2p_n > 0) __threadfence_system();   // remote rows before the signal kernel
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}


// ===========================================================================
// CTA-pair variant (cta_group::2): the two CTAs of a cluster own adjacent
// 128-feature tiles (2p, 2p+1) of the same (expert, token chunk) and run ONE
// M=256 MMA per k-step issued by the leader. Each CTA stages its own 16 KB
// weight tile but only HALF of the token tile (N/2 rows): the token bytes an
// SM must ingest per weight byte are halved, which is what bounds the
// one-CTA kernel (weights from HBM + tokens from L2 share the per-SM fill
// bandwidth). Weights are fetched with TMA (no swizzle: the packed tiles are
// already the swizzled smem image) so the follower's loads can complete on
// the leader's barriers.
// ===========================================================================
constexpr int B2_BOX = 16;                       // token rows per TMA box (2 KB)
constexpr int B2_BYTES = (BN_MAX / 2) * BK * 2;  // 16 KB: half of a 256-token tile

template <bool kDown, int AS, int BS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_grouped_gemm_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + AS * A_BYTES;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(sB + BS * B2_BYTES);
  uint64_t* emptyA = fullA + AS;
  uint64_t* fullB = emptyA + AS;
  uint64_t* emptyB = fullB + BS;
  uint64_t* tfull = emptyB + BS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_pref = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_off = s_pref + (p.E + 1);   // internal segment starts (pos)
  int32_t* s_cs = s_off + (p.E + 1);
  int32_t* s_end = s_cs + p.E;           // pos + count

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  for (int i = threadIdx.x; i <= p.E; i += kThreads) {
    s_pref[i] = p.tb.tc_chunk_pref[i];
    s_off[i] = p.tb.pos[i];
    if (i < p.E) {
      s_cs[i] = p.tb.tc_chunk_size[i];
      s_end[i] = p.tb.pos[i] + p.tb.counts[i];
    }
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(&fullA[s], 2);   // leader arrive.expect_tx + follower arrive
      mbar_init(&emptyA[s], 1);  // leader's multicast commit
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(&fullB[s], 2);
      mbar_init(&emptyB[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (in the leader)
    }
    fence_mbar_init();
  }
  cluster_sync_all();
  if (warp == 2) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_mt = p.n_mt, n_mp = n_mt / 2;
  const UnitList UL = unit_list(p, n_mp, s_pref, s_off, s_end);
  const int total = UL.total;
  const int nkb = p.K / BK;
  const int cid = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(nclusters_x());

  if (warp == 0) {
    // -------------------------------------------------------------- weight producer (both CTAs)
    const uint64_t pol_w = policy_evict_first();
    const uint32_t leader_full = mapa_shared(smem_u32(fullA), 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = cid; u < total; u += ncl) {
      const Unit w = unit_at(UL, u, n_mp, p.E, s_pref, s_off, s_end, s_cs);
      const int mt = 2 * w.mt + static_cast<int>(rank);
      const int row0 = ((w.e * n_mt + mt) * nkb) * BM;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&emptyA[stage], phase ^ 1);
        const uint32_t fb = leader_full + stage * 8;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&fullA[stage], 2 * A_BYTES);
          else mbar_arrive_cluster(fb);
          tma_load_2d_2sm(&tmA, fb, sA + stage * A_BYTES, 0, row0 + kb * BM, pol_w);
        }
        __syncwarp();
        if (++stage == AS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 3) {
    // -------------------------------------------------------------- token producer (both CTAs)
    const uint64_t pol_x = policy_evict_last();
    const uint32_t leader_full = mapa_shared(smem_u32(fullB), 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = cid; u < total; u += ncl) {
      const Unit w = unit_at(UL, u, n_mp, p.E, s_pref, s_off, s_end, s_cs);
      const int half = ((w.ntok + 31) & ~31) / 2;     // rows per CTA
      const int nb = half / B2_BOX;
      const int r0 = w.tok0 + static_cast<int>(rank) * half;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&emptyB[stage], phase ^ 1);
        const uint32_t fb = leader_full + stage * 8;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&fullB[stage], 2 * nb * B2_BOX * BK * 2);
          else mbar_arrive_cluster(fb);
          for (int i = 0; i < nb; ++i)
            tma_load_2d_2sm(&tmB, fb, sB + stage * B2_BYTES + i * (B2_BOX * BK * 2), kb * BK,
                            r0 + i * B2_BOX, pol_x);
        }
        __syncwarp();
        if (++stage == BS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader only)
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int u = cid; u < total; u += ncl) {
        const Unit w = unit_at(UL, u, n_mp, p.E, s_pref, s_off, s_end, s_cs);
        const int nmma = (w.ntok + 31) & ~31;
        const uint32_t idesc = idesc_bf16_f32(2 * BM, nmma);
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * ACC_STRIDE;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&fullB[sb], pb);
          mbar_wait(&fullA[sa], pa);
          tc_fence_after();
          const uint64_t ad = smem_desc_k_sw128(smem_u32(sA + sa * A_BYTES));
          const uint64_t bd = smem_desc_k_sw128(smem_u32(sB + sb * B2_BYTES));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16_ss_2sm(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            mma_commit_2sm(&emptyA[sa], 0x3);
            mma_commit_2sm(&emptyB[sb], 0x3);
          }
          __syncwarp();
          if (++sa == AS) { sa = 0; pa ^= 1; }
          if (++sb == BS) { sb = 0; pb ^= 1; }
        }
        if (elect_one()) mma_commit_2sm(&tfull[as], 0x3);
        __syncwarp();
        as ^= 1;
        if (as == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int wq = warp & 3;
    __nv_bfloat16* stage = reinterpret_cast<__nv_bfloat16*>(
        (reinterpret_cast<uintptr_t>(s_end + p.E) + 15) & ~static_cast<uintptr_t>(15)) + wq * 512;
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    int as = 0;
    uint32_t aphase = 0;
    for (int u = cid; u < total; u += ncl) {
      const Unit w = unit_at(UL, u, n_mp, p.E, s_pref, s_off, s_end, s_cs);
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const int mt = 2 * w.mt + static_cast<int>(rank);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + as * ACC_STRIDE;
      int rows_r[BN_MAX / 32];
      float g_r[BN_MAX / 32];
      store_tile<kDown>(p, w.tok0, w.ntok, (w.ntok + 31) & ~31, mt * BM + wq * 32, taddr, lane,
                        pol_keep, stage, 0, rows_r, g_r);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + as * 8);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
    if (kDown && p.p2p_n > 0) __threadfence_system();   // remote rows before the signal kernel
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, TMEM_COLS);
}


// ===========================================================================
// Both projections in ONE persistent CTA-pair kernel. The work list is
// [all up pair-units (expert-major), all down pair-units (expert-major)];
// cluster c takes units c, c + #clusters, ... A down unit of token chunk q
// reads H rows written by every up unit of q (each feature tile), so its token
// producer waits until done[q] == 2 * n_mp_up (each CTA of each up pair-unit
// releases one count after its H tile is stored) - acquire, then an
// async-proxy fence before the TMA reads H. Units earlier in the list never
// wait on later ones, so with all clusters resident there is no deadlock.
// This removes the down-projection's wave-quantisation tail and the launch gap
// between the two products.
// ===========================================================================
struct FusedParams {
  TcParams up, dn;
  int32_t* done;       // [token chunks], zeroed by Step 2 before every forward
  bool dynamic;        // units taken from a global counter in list order (MOESHARD_FLAG_DYNAMIC_SCHED)
  bool early_tables;   // tables via a release flag from the grouping launch's CTA 0 (see kernel)
};

#ifndef MOESHARD_EPI_WARPS
#define MOESHARD_EPI_WARPS 8
#endif
#ifndef MOESHARD_EPI_STM
#define MOESHARD_EPI_STM 1
#endif
// Paired token chunks (kernel template kPair, chosen per launch): an expert whose segment
// is cut into several chunks of <= kPairMaxCs tokens is processed two chunks per unit - one
// weight stage feeds two MMAs (chunk a into accumulator slot s, chunk b into slot s ^ 1),
// so a weight tile enters shared memory once per two chunks instead of once per chunk (a
// unit's time is its weight stream, ~50 GB/s per SM: scripts/micro/wstream.cu). The two
// chunks are two "virtual tiles" of the accumulator sequence; a single-chunk unit is one.
// Pays where most experts get ~2 chunks of ~130-160 tokens (C5: 256 tokens per expert on
// average, -9 %); the launch picks it only when the assignments per expert average >= 256
// and F >= 4096 (narrower shards and top-2 C2 / C3 measured slower paired).
#ifndef MOESHARD_PAIR_MAX_CS
#define MOESHARD_PAIR_MAX_CS 192
#endif
// only chunks of <= kPairMaxCs tokens are paired: a pair of 256-token chunks is tensor-bound
// (2 x 0.385 us of MMA per k-step against 0.33 us for the weight tile) and would only lose
// the accumulator double buffering
constexpr int kPairMaxCs = MOESHARD_PAIR_MAX_CS;
constexpr int kEpiWarps = MOESHARD_EPI_WARPS;   // epilogue warps per CTA (multiple of 4)
constexpr int kFusedThreads = 128 + 32 * kEpiWarps;
static_assert(kEpiWarps % 4 == 0 && kEpiWarps <= 16, "1-4 epilogue warps per TMEM lane quadrant");
static_assert(MOESHARD_EPI_STM || kEpiWarps <= 8,
              "store_tile indexes its row registers statically only for 1-2 warps per quadrant");
constexpr int kUQ = 2;             // unit-queue slots (dynamic scheduling): small, so a
                                   // cluster never sits on units other clusters could run
constexpr int kUQConsumers = 5 + 2 * kEpiWarps;   // warps that read a slot: leader 0,1,3 + epilogue; follower 0,3 + epilogue
constexpr uint32_t kSchedRank = 0;   // the unit scheduler's CTA (leader)

template <int AS, int BS, bool kPair>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFusedThreads, 1)
    tc_moe_ffn_2sm(const __grid_constant__ CUtensorMap tmA_up, const __grid_constant__ CUtensorMap tmB_up,
                   const __grid_constant__ CUtensorMap tmA_dn, const __grid_constant__ CUtensorMap tmB_dn,
                   FusedParams fp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int E = fp.up.E;
  uint8_t* sA = smem;
  uint8_t* sB = smem + AS * A_BYTES;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(sB + BS * B2_BYTES);
  uint64_t* emptyA = fullA + AS;
  uint64_t* fullB = emptyA + AS;
  uint64_t* emptyB = fullB + BS;
  uint64_t* tfull = emptyB + BS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_pref = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_off = s_pref + (E + 1);     // internal segment starts (pos)
  int32_t* s_cs = s_off + (E + 1);
  int32_t* s_end = s_cs + E;             // pos + count
  int32_t* s_ppref = s_end + E;          // [E+1] cumulative units per (expert, m-tile pair)
  // per-warp epilogue staging (4 x 1 KB), then the unit queue (slots + barriers)
  __nv_bfloat16* s_stage = reinterpret_cast<__nv_bfloat16*>(
      (reinterpret_cast<uintptr_t>(s_ppref + E + 1) + 15) & ~static_cast<uintptr_t>(15));
  int* s_uq = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(s_stage) + kEpiWarps * kStmStage);
  uint64_t* uq_full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(s_uq + kUQ) + 7) & ~static_cast<uintptr_t>(7));
  uint64_t* uq_empty = uq_full + kUQ;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) TL_MIN(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA_up);
    tma_prefetch_desc(&tmA_dn);
  }
  if (warp == 3 && lane == 0) {
    tma_prefetch_desc(&tmB_up);
    tma_prefetch_desc(&tmB_dn);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(&fullA[s], 2);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(&fullB[s], 2);
      mbar_init(&emptyB[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    for (int q = 0; q < kUQ; ++q) {
      mbar_init(&uq_full[q], 1);
      mbar_init(&uq_empty[q], kUQConsumers);
    }
    fence_mbar_init();
  }
  // no cluster barrier here: the mbarrier inits reach the peer through the cluster barrier
  // after the tables below, before any remote arrive (A/B: -0.3 us)
  if (warp == 2) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
#ifndef MOESHARD_EARLY_ARRIVE
#define MOESHARD_EARLY_ARRIVE 1
#endif
  // the cluster barrier that publishes the mbarrier inits and the TMEM address to both CTAs
  // is split: arrive here, wait after the tables below (its latency hides behind them)
  if (MOESHARD_EARLY_ARRIVE) {
    tc_fence_before();
    cluster_arrive_release();
  }
  // PDL: everything above overlapped the grouping kernel's tail. early_tables: the
  // grouping launch's CTA 0 publishes the segment tables (release on tb.stats[6]) before
  // it copies its rows, so only the roles that read X_perm / perm / route wait for the
  // whole grid (griddepcontrol.wait below); the weight producer starts right away.
  if (fp.early_tables) {
    if (threadIdx.x == 0) {
      uint32_t it = 0;
      while (ld_acquire_gpu(fp.up.tb.stats + 6) == 0) {
        if (++it > (1u << 24)) {   // never published: fall back to the grid dependency
          griddep_wait();
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
  } else {
    griddep_wait();
  }
  for (int i = threadIdx.x; i <= E; i += kFusedThreads) {
    s_pref[i] = fp.up.tb.tc_chunk_pref[i];
    s_off[i] = fp.up.tb.pos[i];
    if (i < E) {
      s_cs[i] = fp.up.tb.tc_chunk_size[i];
      s_end[i] = fp.up.tb.pos[i] + fp.up.tb.counts[i];
    }
  }
  const int n_mp_up = (fp.up.n_mt + 1) / 2, n_mp_dn = (fp.dn.n_mt + 1) / 2;
  const int ncl = static_cast<int>(nclusters_x());
  if (kPair) {   // units per (expert, m-tile pair): ceil(chunks / 2), prefix by warp 0
    __syncthreads();
    if (warp == 0) {
      int run = 0;
      for (int b0 = 0; b0 < E; b0 += 32) {
        const int e = b0 + lane;
        const int nc = e < E ? s_pref[e + 1] - s_pref[e] : 0;
        const int np = (e < E && s_cs[e] <= kPairMaxCs) ? (nc + 1) >> 1 : nc;
        int inc = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (e < E) s_ppref[e] = run + inc - np;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) s_ppref[E] = run;
    }
  }
  if (MOESHARD_EARLY_ARRIVE) {
    __syncthreads();   // the tables in shared memory (the cluster barrier was arrived at above)
    cluster_wait_acquire();
  } else {
    tc_fence_before();
    cluster_sync_all();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  if (threadIdx.x == 0) { TL_MIN(1); TL_MAX(1); }   // tables read, roles start

  // pair-units cover m-tiles (2q, 2q+1); with an odd count the last pair has
  // both CTAs on the same m-tile (the follower's copy is computed, not stored)
  const int chunks = kPair ? s_ppref[E] : s_pref[E];   // (paired) chunk units
  const int total_up = chunks * n_mp_up;
  const int total = total_up + chunks * n_mp_dn;
  const int nkb_up = fp.up.K / BK, nkb_dn = fp.dn.K / BK;   // k-blocks per unit
  const int cid = static_cast<int>(cluster_id_x());
  const uint32_t sched_uq_empty = mapa_shared(smem_u32(uq_empty), kSchedRank);
  // k-th unit of this cluster: static round robin, or the k-th queue slot (dynamic)
  auto fetch = [&](int k) -> int {
    if (!fp.dynamic) return cid + k * ncl;
    const int slot = k % kUQ;
    mbar_wait_acquire_cluster(&uq_full[slot], static_cast<uint32_t>((k / kUQ) & 1));
    const int u = *reinterpret_cast<volatile int*>(&s_uq[slot]);
    __syncwarp();
    if (lane == 0) {
      if (rank == kSchedRank) mbar_arrive(&uq_empty[slot]);
      else mbar_arrive_cluster(sched_uq_empty + slot * 8);
    }
    return u;
  };
  // list position u -> (down?, decoded unit); with paired chunks, b = the unit's second
  // chunk (b.ntok = 0: a single-chunk unit)
  auto unit_at2 = [&](int u, bool& down, Unit& b) -> Unit {
    down = u >= total_up;
    const int v = down ? u - total_up : u;
    const int n_mp = down ? n_mp_dn : n_mp_up;
    if (!kPair) {
      b.ntok = 0;
      return decode(v, n_mp, E, s_pref, s_off, s_end, s_cs);
    }
    const int q = v / n_mp;
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_ppref[mid] <= q) lo = mid; else hi = mid;
    }
    const int npe = s_ppref[lo + 1] - s_ppref[lo];
    const int local = v - s_ppref[lo] * n_mp;
    Unit w;
    w.e = lo;
    w.mt = local / npe;
    const int nch = s_pref[lo + 1] - s_pref[lo], cs = s_cs[lo];
    const bool paired = cs <= kPairMaxCs;
    const int ca = (paired ? 2 : 1) * (local - w.mt * npe);
    w.chunk = s_pref[lo] + ca;
    w.tok0 = s_off[lo] + ca * cs;
    w.ntok = min(cs, s_end[lo] - w.tok0);
    b.e = lo;
    b.mt = w.mt;
    b.chunk = w.chunk + 1;
    b.tok0 = w.tok0 + cs;
    b.ntok = paired && ca + 1 < nch ? min(cs, s_end[lo] - b.tok0) : 0;
    return w;
  };
  auto unit_at = [&](int u, bool& down) -> Unit {
    Unit b;
    return unit_at2(u, down, b);
  };

  // unit scheduler (dynamic mode): the leader's otherwise idle warp 2
  const bool sched_warp = fp.dynamic && rank == kSchedRank && warp == 2;
  if (sched_warp) {
    {
      // ------------------------------------------------------------ unit scheduler
      const uint32_t peer_uq = mapa_shared(smem_u32(s_uq), kSchedRank ^ 1);
      const uint32_t peer_full = mapa_shared(smem_u32(uq_full), kSchedRank ^ 1);
      for (int k = 0;; ++k) {
        const int slot = k % kUQ;
        mbar_wait(&uq_empty[slot], static_cast<uint32_t>(((k / kUQ) & 1) ^ 1));
        int u = 0;
        if (lane == 0) {
          u = atomicAdd(fp.dn.tb.next_unit, 1);
          s_uq[slot] = u;
          st_shared_cluster_u32(peer_uq + slot * 4, static_cast<uint32_t>(u));
          mbar_arrive(&uq_full[slot]);
          mbar_arrive_release_cluster(peer_full + slot * 8);
        }
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= total) break;
      }
    }
  } else if (warp == 0) {
    // -------------------------------------------------------------- weight producer (both CTAs)
    // weight tiles are streamed once (evict_first) - except an expert's tiles when it has
    // several token chunks: its sibling units read the same tile at nearly the same time,
    // and evict_first would let the trailing reader miss L2 and re-read it from DRAM
    const uint64_t pol_once = policy_evict_first();
    const uint64_t pol_shared = policy_evict_normal();
    const uint32_t leader_full = mapa_shared(smem_u32(fullA), 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int k = 0, u = fetch(0); u < total; u = fetch(++k)) {
      bool down;
      const Unit w = unit_at(u, down);
      const int n_mt = down ? fp.dn.n_mt : fp.up.n_mt;
      const int nkb = down ? nkb_dn : nkb_up;
      const CUtensorMap* tm = down ? &tmA_dn : &tmA_up;
      const int mt = min(2 * w.mt + static_cast<int>(rank), n_mt - 1);
      const int row0 = ((w.e * n_mt + mt) * nkb) * BM;
      const int32_t* upf = kPair ? s_ppref : s_pref;   // units per (e, mt) > 1: siblings
      const uint64_t pol_w = (upf[w.e + 1] - upf[w.e] > 1) ? pol_shared : pol_once;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&emptyA[stage], phase ^ 1);
        const uint32_t fb = leader_full + stage * 8;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&fullA[stage], 2 * A_BYTES);
          else mbar_arrive_cluster(fb);
          tma_load_2d_2sm(tm, fb, sA + stage * A_BYTES, 0, row0 + kb * BM, pol_w);
        }
        __syncwarp();
        if (++stage == AS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 3) {
    // -------------------------------------------------------------- token producer (both CTAs)
    // X_perm rows (re-read by the up units' feature pair-tiles at nearly the same time) and
    // H rows (read by the down units) are kept in L2 (evict_last, persisting set-aside)
    const uint64_t pol_x = policy_evict_last();
    if (fp.early_tables) griddep_wait();   // X_perm rows and the route records are complete
    if (lane == 0) { TL_MIN(2); TL_MAX(2); }
    const uint32_t leader_full = mapa_shared(smem_u32(fullB), 0);
    int stage = 0;
    uint32_t phase = 0;
    // H rows of a token chunk complete? (acquire), then order the TMA after it
    auto wait_h = [&](int chunk, int k) {
      const int target = 2 * n_mp_up;   // both CTAs of every up pair-unit of (e, chunk)
      if (elect_one()) {
        uint32_t it = 0;
        while (ld_acquire_gpu(fp.done + chunk) < target) {
          if (++it > (1u << 24)) {   // a cluster never became resident: report, do not hang
            atomicOr(fp.up.tb.stats + 3, 8);
            break;
          }
          __nanosleep(128);
        }
        fence_proxy_async_global();
        if (leader) TR(cid, k, 7);
      }
      __syncwarp();
    };
    // one k-block of one chunk's token tile (this CTA's half of its rows) into the next stage
    auto load_b = [&](const CUtensorMap* tm, const Unit& w, int kb) {
      const int half = ((w.ntok + 31) & ~31) / 2;
      const int nb = half / B2_BOX;
      const int r0 = w.tok0 + static_cast<int>(rank) * half;
      const uint32_t stage_bytes = nb * B2_BOX * BK * 2;
      mbar_wait(&emptyB[stage], phase ^ 1);
      const uint32_t fb = leader_full + stage * 8;
      if (elect_one()) {
#ifdef MOESHARD_EXP_NO_BLOAD
        if (leader) mbar_arrive(&fullB[stage]);
        else mbar_arrive_cluster(fb);
#else
        if (leader) mbar_arrive_expect_tx(&fullB[stage], 2 * stage_bytes);
        else mbar_arrive_cluster(fb);
        for (int i = 0; i < nb; ++i)
          tma_load_2d_2sm(tm, fb, sB + stage * B2_BYTES + i * (B2_BOX * BK * 2), kb * BK,
                          r0 + i * B2_BOX, pol_x);
#endif
      }
      __syncwarp();
      if (++stage == BS) { stage = 0; phase ^= 1; }
    };
    for (int k = 0, u = fetch(0); u < total; u = fetch(++k)) {
      bool down;
      Unit wb;
      const Unit w = unit_at2(u, down, wb);
      const int nkb = down ? nkb_dn : nkb_up;
      const CUtensorMap* tm = down ? &tmB_dn : &tmB_up;
      if (down) {
        wait_h(w.chunk, k);
        if (wb.ntok > 0) wait_h(wb.chunk, k);
      }
      for (int kb = 0; kb < nkb; ++kb) {   // paired: chunk a, then chunk b, per k-block
        load_b(tm, w, kb);
        if (wb.ntok > 0) load_b(tm, wb, kb);
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader only)
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int k = 0, u = fetch(0); u < total; u = fetch(++k)) {
        bool down;
        Unit wb;
        const Unit w = unit_at2(u, down, wb);
        const bool two = wb.ntok > 0;   // paired chunks: a -> slot as, b -> slot as ^ 1
        const int nkb = down ? nkb_dn : nkb_up;
        const uint32_t idesc = idesc_bf16_f32(2 * BM, (w.ntok + 31) & ~31);
        const uint32_t idesc_b = idesc_bf16_f32(2 * BM, two ? (wb.ntok + 31) & ~31 : 32);
        const int as_b = as ^ 1;
        const uint32_t aphase_b = as_b == 0 ? aphase ^ 1 : aphase;   // the next virtual tile's
        if (lane == 0) TR(cid, k, 0);
        mbar_wait(&tempty[as], aphase ^ 1);
        if (two) mbar_wait(&tempty[as_b], aphase_b ^ 1);
        tc_fence_after();
        if (lane == 0) TR(cid, k, 1);
        const uint32_t d = tmem_base + as * ACC_STRIDE, d_b = tmem_base + as_b * ACC_STRIDE;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&fullB[sb], pb);
          if (kb == 0 && lane == 0) TR(cid, k, 2);
          mbar_wait(&fullA[sa], pa);
          tc_fence_after();
          if (kb == 0 && lane == 0) TR(cid, k, 3);
          const uint64_t ad = smem_desc_k_sw128(smem_u32(sA + sa * A_BYTES));
          if (elect_one()) {
            const uint64_t bd = smem_desc_k_sw128(smem_u32(sB + sb * B2_BYTES));
#ifndef MOESHARD_EXP_NO_MMA
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_bf16_ss_2sm(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0);
#endif
            mma_commit_2sm(&emptyB[sb], 0x3);
          }
          __syncwarp();
          if (++sb == BS) { sb = 0; pb ^= 1; }
          if (two) {   // the same weight stage, chunk b's token stage
            mbar_wait(&fullB[sb], pb);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t bd = smem_desc_k_sw128(smem_u32(sB + sb * B2_BYTES));
#ifndef MOESHARD_EXP_NO_MMA
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                mma_bf16_ss_2sm(d_b, ad + 2 * kk, bd + 2 * kk, idesc_b, (kb | kk) != 0);
#endif
              mma_commit_2sm(&emptyB[sb], 0x3);
            }
            __syncwarp();
            if (++sb == BS) { sb = 0; pb ^= 1; }
          }
          if (elect_one()) mma_commit_2sm(&emptyA[sa], 0x3);
          __syncwarp();
          if (++sa == AS) { sa = 0; pa ^= 1; }
        }
        if (elect_one()) {
          mma_commit_2sm(&tfull[as], 0x3);
          if (two) mma_commit_2sm(&tfull[as_b], 0x3);
        }
        __syncwarp();
        if (lane == 0) TR(cid, k, 4);
        for (int v = 0; v < (two ? 2 : 1); ++v) {
          as ^= 1;
          if (as == 0) aphase ^= 1;
        }
      }
    }
    if (leader && lane == 0) TL_MAX(3);   // last MMA issued
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int wq = warp & 3, eh = (warp - 4) >> 2;
#if !MOESHARD_EPI_STM
    __nv_bfloat16* stage = s_stage + (warp - 4) * 512;   // 1 KB per epilogue warp
#endif
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    if (fp.early_tables) griddep_wait();   // perm / route of the grouping launch
    int as = 0;
    uint32_t aphase = 0;
    for (int k = 0, u = fetch(0); u < total; u = fetch(++k)) {
      bool down;
      Unit wb;
      const Unit wa = unit_at2(u, down, wb);
      for (int vt = 0; vt < (wb.ntok > 0 ? 2 : 1); ++vt) {   // paired chunks: two tiles
      const Unit& w = vt ? wb : wa;
      // down: destination rows and gates loaded before the accumulator wait (their
      // latency hides behind it; at short K it was exposed once per tile)
      int rows_r[BN_MAX / 32];
      float g_r[BN_MAX / 32];
#if MOESHARD_EPI_STM
      if (down) load_rows_gates_chunked<kEpiWarps / 4>(fp.dn, w.tok0, w.ntok, lane, eh, rows_r, g_r);
#else
      if (down) load_rows_gates(fp.dn, w.tok0, w.ntok, lane, rows_r, g_r);
#endif
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      if (leader && warp == 4 && lane == 0) TR(cid, k, 5);
      const int mt = 2 * w.mt + static_cast<int>(rank);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + as * ACC_STRIDE;
#ifdef MOESHARD_EXP_NO_EPI
      if (false) {
#else
      if (mt < (down ? fp.dn.n_mt : fp.up.n_mt)) {   // else: duplicate of the leader's tile
#endif
#if MOESHARD_EPI_STM
        uint8_t* stg = reinterpret_cast<uint8_t*>(s_stage) + (warp - 4) * kStmStage;
        if (down)
          store_tile_stm<true, kEpiWarps / 4>(fp.dn, w.tok0, w.ntok, (w.ntok + 31) & ~31,
                                              mt * BM + wq * 32, taddr, lane, pol_keep, stg, eh,
                                              rows_r, g_r);
        else
          store_tile_stm<false, kEpiWarps / 4>(fp.up, w.tok0, w.ntok, (w.ntok + 31) & ~31,
                                               mt * BM + wq * 32, taddr, lane, pol_keep, stg, eh,
                                               rows_r, g_r);
#else
        if (down)
          store_tile<true, kEpiWarps / 4, true>(fp.dn, w.tok0, w.ntok, (w.ntok + 31) & ~31,
                                                mt * BM + wq * 32, taddr, lane, pol_keep, stage, eh,
                                                rows_r, g_r);
        else
          store_tile<false, kEpiWarps / 4, true>(fp.up, w.tok0, w.ntok, (w.ntok + 31) & ~31,
                                                 mt * BM + wq * 32, taddr, lane, pol_keep, stage, eh,
                                                 rows_r, g_r);
#endif
      }
      tc_fence_before();
      __syncwarp();
      if (leader && warp == 4 && lane == 0) TR(cid, k, 6);
      if (lane == 0) mbar_arrive_cluster(leader_tempty + as * 8);
      if (!down) {   // publish this CTA's H tile of the chunk
        // bar.sync orders every epilogue thread's H stores before thread 0's release
        // (cumulative at gpu scope), so the other warps need no fence of their own and
        // go straight on to the next tile
        asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");   // the epilogue warps
        if (warp == 4 && lane == 0) red_release_gpu_add(fp.done + w.chunk, 1);
      }
      as ^= 1;
      if (as == 0) aphase ^= 1;
      }   // virtual tiles
    }
    // (P2P: the remote partial rows are ordered before the peers' flags by the grid's completion
    // and the system-scope fence of rs_signal, the next launch; a fence per CTA here delayed
    // the end of the kernel by microseconds)
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, TMEM_COLS);
  if (threadIdx.x == 0) TL_MAX(0);
}

size_t smem_bytes(int E, int as, int bs) {
  return 1024 + as * A_BYTES + bs * B_BYTES + (2 * as + 2 * bs + 4) * 8 + 16 + (4 * E + 2) * 4 +
         16 + 4 * 1024;
}

size_t smem_bytes_2sm(int E, int as, int bs) {
  return 1024 + as * A_BYTES + bs * B2_BYTES + (2 * as + 2 * bs + 4) * 8 + 16 + (5 * E + 3) * 4 +
         16 + kEpiWarps * kStmStage + 96;   // + epilogue staging (per epilogue warp) + unit queue
}

template <bool kDown, int AS, int BS>
cudaError_t launch_1sm(const CUtensorMap& tmB, const TcParams& p, int grid, cudaStream_t s) {
  static PerDeviceOnce attr;  // per template instance and device
  if (attr.need()) {
    cudaError_t e = cudaFuncSetAttribute(tc_grouped_gemm<kDown, AS, BS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes(kMaxExperts, AS, BS)));
    if (e != cudaSuccess) return e;
    attr.done();
  }
  tc_grouped_gemm<kDown, AS, BS><<<grid, kThreads, smem_bytes(p.E, AS, BS), s>>>(tmB, p);
  return cudaGetLastError();
}

template <bool kDown, int AS, int BS>
cudaError_t launch_2sm(const CUtensorMap& tmA, const CUtensorMap& tmB, const TcParams& p, int grid,
                       cudaStream_t s) {
  static PerDeviceOnce attr;
  if (attr.need()) {
    cudaError_t e = cudaFuncSetAttribute(tc_grouped_gemm_2sm<kDown, AS, BS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes_2sm(kMaxExperts, AS, BS)));
    if (e != cudaSuccess) return e;
    attr.done();
  }
  tc_grouped_gemm_2sm<kDown, AS, BS><<<grid & ~1, kThreads, smem_bytes_2sm(p.E, AS, BS), s>>>(
      tmA, tmB, p);
  return cudaGetLastError();
}

// ring depths: (6, 6) for the CTA pair (A 16 KB, B 16 KB stages), (4, 4) for one CTA
// (B 32 KB stages); profiles/r01_gemm_experiments.md §3
template <bool kDown>
cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmB2,
                     const TcParams& p, int grid, cudaStream_t s) {
  if (p.n_mt % 2 == 0) return launch_2sm<kDown, 6, 6>(tmA, tmB2, p, grid, s);
  return launch_1sm<kDown, 4, 4>(tmB, p, grid, s);
}

}  // namespace

TL_EXPORT(moeshard_tl_ffn)
TR_EXPORT(moeshard_tr_ffn)

cudaError_t launch_tc_moe_ffn(const CUtensorMap& tmA_up, const CUtensorMap& tmB_up,
                              const CUtensorMap& tmA_dn, const CUtensorMap& tmB_dn,
                              const TcParams& up, const TcParams& dn, int32_t* done, bool dynamic,
                              bool early_tables, bool pair_chunks, int grid, cudaStream_t s) {
#ifndef MOESHARD_FFN_AS
#define MOESHARD_FFN_AS 6
#define MOESHARD_FFN_BS 6
#endif
  constexpr int AS = MOESHARD_FFN_AS, BS = MOESHARD_FFN_BS;
  static PerDeviceOnce attr;
  if (attr.need()) {
    for (auto* k : {tc_moe_ffn_2sm<AS, BS, false>, tc_moe_ffn_2sm<AS, BS, true>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem_bytes_2sm(kMaxExperts, AS, BS)));
      if (e != cudaSuccess) return e;
    }
    attr.done();
  }
  FusedParams fp{up, dn, done, dynamic, early_tables};
  return launch_pdl(pair_chunks ? tc_moe_ffn_2sm<AS, BS, true> : tc_moe_ffn_2sm<AS, BS, false>,
                    dim3(grid & ~1), dim3(kFusedThreads), smem_bytes_2sm(up.E, AS, BS), s,
                    tmA_up, tmB_up, tmA_dn, tmB_dn, fp);
}

cudaError_t launch_tc_gemm(bool down, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmB2, const TcParams& p, int grid, cudaStream_t s) {
  return down ? launch_t<true>(tmA, tmB, tmB2, p, grid, s)
              : launch_t<false>(tmA, tmB, tmB2, p, grid, s);
}

namespace {
// One CTA per 128 x 64 tile: coalesced read of src[e][kb*64 .. +64][mt*128 .. +128]
// (rows of M), transpose through shared memory, write the swizzled 16 KB block.
__global__ void __launch_bounds__(256) pack_a_tiles(const __nv_bfloat16* __restrict__ src,
                                                    __nv_bfloat16* __restrict__ dst, int K, int M) {
  __shared__ __nv_bfloat16 t[64][128 + 8];
  const int mt = blockIdx.x, kb = blockIdx.y, e = blockIdx.z;
  const int n_mt = M / BM, nkb = K / BK;
  const __nv_bfloat16* s = src + static_cast<size_t>(e) * K * M;
  for (int q = threadIdx.x; q < 64 * 16; q += 256) {      // 64 k-rows x 16 chunks of 8 m
    const int kk = q / 16, c = q % 16;
    const uint4 v = *reinterpret_cast<const uint4*>(s + static_cast<size_t>(kb * BK + kk) * M +
                                                    mt * BM + c * 8);
    *reinterpret_cast<uint4*>(&t[kk][c * 8]) = v;
  }
  __syncthreads();
  __nv_bfloat16* d = dst + ((static_cast<size_t>(e) * n_mt + mt) * nkb + kb) * (BM * BK);
  for (int q = threadIdx.x; q < BM * 8; q += 256) {       // 128 rows x 8 chunks of 8 k
    const int r = q / 8, j = q % 8;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[j * 8 + i][r];
    *reinterpret_cast<uint4*>(d + r * BK + ((j ^ (r & 7)) * 8)) = *reinterpret_cast<uint4*>(v);
  }
}
}  // namespace

void launch_pack_a_tiles(const void* src, void* dst, int E, int K, int M, cudaStream_t s) {
  dim3 grid(M / BM, K / BK, E);
  pack_a_tiles<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                    static_cast<__nv_bfloat16*>(dst), K, M);
}

}  // namespace moeshard
