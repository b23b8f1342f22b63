// gemm_tc.cuh - host interface of the tcgen05 grouped GEMM (gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace moeshard {

// Weight storage of the tcgen05 path ("A" operand): for every expert e, every
// 128-row tile mt of the output features and every 64-wide k-block kb, the
// 128 x 64 bf16 tile A[e][mt*128 + r][kb*64 + c] is stored as one contiguous
// 16 KB block, rows of 128 B with the 128-B swizzle already applied
// (16-B chunk j of row r stored at chunk j ^ (r % 8)) - i.e. byte-for-byte
// the shared-memory image the MMA descriptor expects. Blocks are ordered
// [e][mt][kb], so one (e, mt) tile row streams as K/64 * 16 KB contiguous
// bytes: sequential HBM reads, fetched with plain bulk copies.
//   src [E][K][M] row-major  (w_in_shard: K = h, M = F;  w_out_shard: K = F, M = h)
void launch_pack_a_tiles(const void* src, void* dst, int E, int K, int M, cudaStream_t s);

struct TcParams {
  int K;              // reduction length: h (up) or F = d_ff/G (down); multiple of 64
  int n_mt;           // output tiles of 128 features: F/128 (up) or h/128 (down)
  const __nv_bfloat16* a_tiles;  // packed weight tiles (launch_pack_a_tiles)
  int E;              // experts
  Tables tb;          // device segment tables of the current forward
  __nv_bfloat16* out; // up: H [N][F]; down: out [N or n][h] in global token order
  int ld_out;         // F (up) or h (down)
  const int32_t* perm;     // down: perm[j] = global token id of expert-ordered row j
  const RouteRec* route;   // down: gate per global token
  const float* gate_pad = nullptr;   // down (fused kernel): gate per expert-ordered row
  // launch-mode ablation (Sec. 3.3, MOESHARD_FLAG_LAUNCH_PER_EXPERT / _PER_SOURCE): this
  // launch covers only expert only_e (>= 0) and, if only_g >= 0, only the tokens of source
  // rank only_g: rows [pos[e] + base[g*nbr][e], pos[e] + base[(g+1)*nbr][e]) of its segment
  // (base = Step 2's per-block prefix [n_src*nbr][E], the last rank ends at counts[e])
  int only_e = -1, only_g = -1;
  const int32_t* block_base = nullptr;
  int nbr = 0, n_src = 1;
  // down, peer-memory exchange (MOESHARD_FLAG_P2P): p2p_n > 0 sends the partial row of
  // global token t to its owner o = t / p2p_n, row t - o * p2p_n of p2p_out[o]
  int p2p_n = 0;
  __nv_bfloat16* p2p_out[kMaxWorld] = {};
};

// tcgen05 router (router.cu): logits/softmax/top-1 per 128-token CTA, plus the
// CTA's per-expert token histogram hist_out[blockIdx][E].
// tmX: x [n][h] box {64, 128}. mn_major: tmW = router_w [h][E] box {64 experts, 64 k}
// (E % 8 == 0); else router_w is first transposed to wt_r [EP][h] (zero rows E..EP-1)
// and tmW = wt_r box {64, EP}.
size_t router_tc_smem_bytes(int EP, bool mn_major, int stages);
cudaError_t launch_router_tc(const CUtensorMap& tmX, const CUtensorMap& tmW, bool mn_major,
                             const void* w_r, void* wt_r, int n, int h, int E, int EP,
                             const int32_t* forced, RouteRec* out, int32_t* hist_out,
                             int32_t* err_flag, cudaStream_t s, int top_k, int num_sms);

// grid = number of persistent CTAs (normally the SM count).
//   tmA:  packed weight tiles as a [rows][64] bf16 tensor, box {64, 128}, no swizzle
//   tmB:  activations [N][K], box {64, 32}, 128-B swizzle   (one-CTA kernel)
//   tmB2: activations [N][K], box {64, 16}, 128-B swizzle   (CTA-pair kernel)
// The CTA-pair (cta_group::2) kernel is used when n_mt is even.
// Both projections in one persistent CTA-pair launch (needs F/128 and h/128 even).
// done: [E] int32 zeroed before the launch (Step 2 does it).
// tmB_up: X_perm [N][h] box {64, 16}; tmB_dn: H [N][F] box {64, 16}.
// dynamic: units taken from a global counter (correct when not every cluster is
// resident); early_tables: the weight stream starts on the grouping launch's
// "tables published" flag instead of the whole-grid dependency.
cudaError_t launch_tc_moe_ffn(const CUtensorMap& tmA_up, const CUtensorMap& tmB_up,
                              const CUtensorMap& tmA_dn, const CUtensorMap& tmB_dn,
                              const TcParams& up, const TcParams& dn, int32_t* done, bool dynamic,
                              bool early_tables, bool pair_chunks, int grid, cudaStream_t s);

// Both products of one expert and <= 128 of its tokens per cluster of F/128 CTAs with H
// kept on chip (expert_mlp.cu); applicable when expert_mlp_supported(h, F, E).
//   tmX128: X_perm [N][h] box {64, 128}, 128-B swizzle; tmWi / tmWo: packed weight tiles
//   dn: the down-projection parameters (output, perm_pad, route, P2P slots, tables, E)
bool expert_mlp_supported(int h, int F, int E);
cudaError_t launch_tc_expert_mlp(const CUtensorMap& tmX128, const CUtensorMap& tmWi,
                                 const CUtensorMap& tmWo, const TcParams& dn, int h, int F,
                                 int num_sms, cudaStream_t s);

cudaError_t launch_tc_gemm(bool down, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmB2, const TcParams& p, int grid, cudaStream_t s);

}  // namespace moeshard
