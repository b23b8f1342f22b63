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
  // up, fused kernel: if gather != nullptr the token tile is gathered straight
  // from x_all rows gather[j] (TMA gather4) instead of the expert-ordered copy
  const int32_t* gather = nullptr;
  int n_rows = 0;          // rows of the gathered tensor (N)
  // fused kernel: H stored transposed, H^T [F][ld_ht] (tokens contiguous). The up
  // epilogue then writes each feature row directly; the down product reads it as
  // an MN-major B operand.
  bool ht = false;
  int ld_ht = 0;           // token stride of H^T (N_max)
  // cp.async gather instead of TMA gather4: rows gsrc[gather[j]] ([n_rows][K] bf16)
  bool gather_cp = false;
  const __nv_bfloat16* gsrc = nullptr;
  int gather_depth = 4;    // stages in flight before one is published (<= ring depth - 1)
  // down, peer-memory exchange (MOESHARD_FLAG_P2P): p2p_n > 0 sends the partial row of
  // global token t to its owner o = t / p2p_n, row t - o * p2p_n of p2p_out[o]
  int p2p_n = 0;
  __nv_bfloat16* p2p_out[kMaxWorld] = {};
};

// Step 2 outputs for the fused route+group launch (world = 1): see launch_route_group_tc.
struct RouteGroupArgs {
  Tables tb;
  int32_t* base;        // [NB][E] workspace: tokens of e in earlier hist-blocks
  int32_t* tot;         // [E] workspace
  int32_t* perm;        // [N] public compact permutation
  const uint4* x;       // hidden [n][h] (row_vecs 16-B vectors per row)
  uint4* x_perm;        // internal expert-ordered rows (nullptr: no row copy)
  int row_vecs;         // h * 2 / 16, <= 128
  int n_mt_up, n_mt_dn; // 128-row tiles of the two products (tile statistics)
  int32_t* bar;         // 2 ints (grid barrier), zero-initialised once
};

// tcgen05 router (router.cu): logits/softmax/top-1 per 128-token CTA, plus the
// CTA's per-expert token histogram hist_out[blockIdx][E].
// tmX: x [n][h] box {64, 128}. mn_major: tmW = router_w [h][E] box {64 experts, 64 k}
// (E % 8 == 0); else router_w is first transposed to wt_r [EP][h] (zero rows E..EP-1)
// and tmW = wt_r box {64, EP}.
size_t router_tc_smem_bytes(int EP, bool mn_major, int tok);
// pf / pf_bytes / pf_ctas: extra CTAs that prefetch the first pf_bytes of the
// layer's packed up-projection tiles into L2 (0 CTAs disables).
cudaError_t launch_router_tc(const CUtensorMap& tmX, const CUtensorMap& tmW, bool mn_major,
                             const void* w_r, void* wt_r, int n, int h, int E, int EP,
                             const int32_t* forced, RouteRec* out, int32_t* hist_out,
                             int32_t* err_flag, const void* pf, long long pf_bytes, int pf_ctas,
                             int tok, cudaStream_t s);

// Router + the whole of Step 2 in one launch (world = 1, ceil(n/128) <= SMs,
// router_w MN-major (E % 8 == 0), h <= 1024): routes 128 tokens per CTA like
// launch_router_tc, then (grid barriers) per-expert block scans, segment
// tables, stable permutation and the X_perm row copy.
cudaError_t launch_route_group_tc(const CUtensorMap& tmX, const CUtensorMap& tmW, int n, int h,
                                  int E, int EP, const int32_t* forced, RouteRec* out,
                                  int32_t* hist_out, int32_t* err_flag, const RouteGroupArgs& ga,
                                  cudaStream_t s);

// grid = number of persistent CTAs (normally the SM count).
//   tmA:  packed weight tiles as a [rows][64] bf16 tensor, box {64, 128}, no swizzle
//   tmB:  activations [N][K], box {64, 32}, 128-B swizzle   (one-CTA kernel)
//   tmB2: activations [N][K], box {64, 16}, 128-B swizzle   (CTA-pair kernel)
// The CTA-pair (cta_group::2) kernel is used when n_mt is even.
// Both projections in one persistent CTA-pair launch (needs F/128 and h/128 even).
// done: [E] int32 zeroed before the launch (Step 2 does it).
// tmB_up: X_perm [N][h] box {64, 16} - or, when up.gather != nullptr, x_all [N][h]
// box {64, 1} for TMA gather4.
// cp_src != nullptr: the kernel itself copies X_perm[j] = cp_src[perm_pad[j]] (rows of
// cp_row_vecs 16-B vectors) into cp_dst before the up-projection reads it (Step 2
// then skips its row copy); per-expert release/acquire on tb.copied.
cudaError_t launch_tc_moe_ffn(const CUtensorMap& tmA_up, const CUtensorMap& tmB_up,
                              const CUtensorMap& tmA_dn, const CUtensorMap& tmB_dn,
                              const TcParams& up, const TcParams& dn, int32_t* done,
                              const void* cp_src, void* cp_dst, int cp_row_vecs, bool dynamic,
                              bool early_tables, int grid, cudaStream_t s);

cudaError_t launch_tc_gemm(bool down, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmB2, const TcParams& p, int grid, cudaStream_t s);

}  // namespace moeshard
