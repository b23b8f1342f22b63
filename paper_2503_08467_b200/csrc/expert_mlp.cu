// expert_mlp.cu - Step 4 for small shards, H kept on chip.
//
// When a rank's shard is narrow (F = d_ff / G <= 512: G = 8 for Switch-Base / -Large), the
// two grouped products of one expert and one chunk of <= 128 of its tokens are computed by
// ONE cluster of CS = F / 128 CTAs, and the intermediate H = relu(X W_i^{e,r}) never leaves
// the chip (§3.3 fusion):
//
//   CTA j (cluster rank j), chunk rows t < 128 (token on the TMEM lane axis, M = 128):
//     up    D_up[t, f]  = sum_k X[t, k] Wi^T[128 j + f, k]        f < 128, K = h
//           -> relu -> bf16 -> H[t, 128 j + f] stored into this CTA's shared memory and, with
//           asynchronous DSMEM stores (st.async, byte completion on the peer's hfull), into
//           every peer's (the MMA A-operand image: K-major, 128-B swizzle)
//     down  D_dn[t, c]  = sum_f H[t, f] Wo^T[C_j + c, f]            c < h / CS, K = F
//           -> gate[t] x -> bf16 -> row perm[t] (or its owner's receive slot, P2P) of the
//           output, columns C_j = [j h/CS, (j+1) h/CS)
//
// so every CTA streams 1/CS of the expert's weights, and no H row is written to or read
// from global memory (the two-phase fused kernel round-trips H through L2/HBM and makes
// each down unit wait for every up unit of its chunk). Units carry no cross-cluster
// dependency, so the kernel is correct whether or not all clusters are resident.
//
// Issue order per cluster: up(0), up(1), dn(0), up(2), dn(1), ... (the next unit's up product
// runs on the tensor core while this unit's H is drained and exchanged; two up accumulators).
// Roles (384 threads): warp 0 TMA producer (one ring of 32 KB stages: X tile + W_i tile
// for an up k-step, the CTA's 1-2 W_o tiles for a down k-step), warp 1 MMA issuer, warp 2
// TMEM allocator, warps 4-7 the H drain (TMEM -> relu -> every CTA's H), warps 8-11 the
// output drain (TMEM -> gate x -> global), so a unit's output drain overlaps the next
// unit's H drain and exchange (TMEM lane quadrant = warp % 4 for both groups). The H
// exchange uses st.async rather than smem->smem bulk copies (those queue behind the
// producer's in-flight TMA loads: 5-8 us per unit) or blocking st.shared::cluster (8 us).
// Barriers per CTA: full/empty per ring stage; upfull/uptempty and dnfull/dntempty between
// MMA and drains; hfull (the 4 local H-drain warps arrive, one with the (CS-1) x 32 KB the
// peers deliver) before the down MMAs read H; hempty (CS arrivals: every CTA's down-MMA commit, multicast) before the
// next unit's H slices may be written into any CTA of the cluster.
#include "common.cuh"
#include "gemm_tc.cuh"
#include "group.cuh"
#include "ptx.cuh"

#include <algorithm>

namespace moeshard {
namespace {

using namespace ptx;

constexpr int kMlpTok = 128;            // tokens per unit (M of both products)
constexpr int kTile = 128 * 64 * 2;     // one 128-row x 64-wide bf16 tile = 16 KB
constexpr int kStage = 2 * kTile;       // ring stage: 32 KB
constexpr int kThreadsMlp = 384;
constexpr int kColUp = 0, kColDn = 256; // TMEM columns: up accumulator x 2 buffers, down
constexpr int kSmemBudget = 225 * 1024; // H + ring (barriers and alignment on top)
constexpr size_t kMaxSmem = 232448;     // opt-in dynamic shared memory per CTA (sm_100)

// asynchronous 16-B store into a peer CTA's shared memory; completion is counted (bytes) on
// the peer's mbarrier at bar_cluster, the storing thread does not wait for it
__device__ __forceinline__ void st_async_v4(uint32_t addr, uint4 v, uint32_t bar_cluster) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
      ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar_cluster)
      : "memory");
}
// arrive once on the barrier at the same offset in every CTA of `mask` when this thread's
// previously issued MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

struct MlpArgs {
  TcParams dn;          // output, perm_pad, route, P2P slots, tables (tb), E
  int h, F;             // d_model, shard width (= CS * 128)
};

// Unit u of the forward -> expert, first row, rows (chunks of <= 128 rows, near equal).
__device__ __forceinline__ void mlp_unit(int u, int E, const int32_t* pref, const int32_t* pos,
                                         const int32_t* cnt, int& e, int& tok0, int& ntok) {
  int lo = 0, hi = E;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= u) lo = mid; else hi = mid;
  }
  e = lo;
  const int nch = pref[lo + 1] - pref[lo], c = u - pref[lo];
  const int cs = (cnt[lo] + nch - 1) / nch;
  tok0 = pos[lo] + c * cs;
  ntok = min(cs, cnt[lo] - c * cs);
}

template <int CS, int NCT>
__global__ void __launch_bounds__(kThreadsMlp, 1)
    tc_expert_mlp(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWi,
                  const __grid_constant__ CUtensorMap tmWo, MlpArgs a) {
  static_assert(CS >= 1 && CS <= 8 && (NCT == 1 || NCT == 2), "cluster / tile shape");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const TcParams& p = a.dn;
  const int E = p.E, h = a.h, F = a.F;
  const int nkb_up = h / 64, nkb_dn = F / 64;
  const int h_bytes = nkb_dn * kTile;                     // H: F/64 tiles of [128 t][64 f]
  const int S = min(6, (kSmemBudget - h_bytes) / kStage);  // ring stages
  uint8_t* sH = smem;
  uint8_t* sR = smem + h_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sR + S * kStage);
  uint64_t* empty = full + S;
  uint64_t* upfull = empty + S;        // [2]
  uint64_t* uptempty = upfull + 2;     // [2]
  uint64_t* dnfull = uptempty + 2;
  uint64_t* dntempty = dnfull + 1;
  uint64_t* hfull = dntempty + 1;
  uint64_t* hempty = hfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + 1);
  int32_t* s_pref = reinterpret_cast<int32_t*>(tmem_slot + 4);   // [E + 1] units per expert
  int32_t* s_pos = s_pref + (E + 1);
  int32_t* s_cnt = s_pos + E;
  int32_t* s_warp = s_cnt + E;                                     // [33] scan scratch

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t j = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmWi);
    tma_prefetch_desc(&tmWo);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&upfull[b], 1);
      mbar_init(&uptempty[b], 4);
    }
    mbar_init(dnfull, 1);
    mbar_init(dntempty, 4);
    mbar_init(hfull, 4);
    mbar_init(hempty, CS);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  // PDL: the prologue above overlapped the grouping launch; tables, X_perm, perm and the
  // route records are its outputs
  griddep_wait();
  int nch = 0;
  if (threadIdx.x < E) {
    const int c = p.tb.counts[threadIdx.x];
    nch = (c + kMlpTok - 1) / kMlpTok;
    s_pos[threadIdx.x] = p.tb.pos[threadIdx.x];
    s_cnt[threadIdx.x] = c;
  }
  int total;
  const int pre = block_excl_scan<kThreadsMlp>(nch, s_warp, total);
  if (threadIdx.x < E) s_pref[threadIdx.x] = pre;
  if (threadIdx.x == 0) s_pref[E] = total;
  tc_fence_before();
  cluster_sync_all();   // barrier inits and TMEM allocation visible cluster-wide
  tc_fence_after();
  griddep_launch_dependents();
  const uint32_t tmem = *tmem_slot;
  const int cid = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(nclusters_x());

  // This cluster's units in the software-pipelined issue order up(0), up(1), dn(0), up(2),
  // dn(1), ...: step i issues up(i) (i < nu) then dn(i-1) (i >= 1), so the tensor core
  // computes the next unit's up product while the epilogue drains this unit's H and the
  // slices travel between the CTAs (the up accumulator is double-buffered in TMEM).
  const int nu = cid < total ? (total - cid + ncl - 1) / ncl : 0;
  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    const uint64_t pol_x = policy_evict_last();    // the chunk's rows: read by all CS CTAs
    const uint64_t pol_w = policy_evict_normal();  // sibling chunks of an expert re-read them
    const int n_mt_up = F / 128, n_mt_dn = h / 128;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i <= nu; ++i) {
      if (i < nu) {
        int e, tok0, ntok;
        mlp_unit(cid + i * ncl, E, s_pref, s_pos, s_cnt, e, tok0, ntok);
        for (int kb = 0; kb < nkb_up; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full[s], kStage);
            uint8_t* st = sR + s * kStage;
            tma_load_2d(&tmX, &full[s], st, kb * 64, tok0, pol_x);
            tma_load_2d(&tmWi, &full[s], st + kTile, 0,
                        ((e * n_mt_up + static_cast<int>(j)) * nkb_up + kb) * 128, pol_w);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
      if (i >= 1) {
        int e, tok0, ntok;
        mlp_unit(cid + (i - 1) * ncl, E, s_pref, s_pos, s_cnt, e, tok0, ntok);
        for (int kb = 0; kb < nkb_dn; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full[s], NCT * kTile);
            uint8_t* st = sR + s * kStage;
#pragma unroll
            for (int q = 0; q < NCT; ++q)
              tma_load_2d(&tmWo, &full[s], st + q * kTile, 0,
                          ((e * n_mt_dn + static_cast<int>(j) * NCT + q) * nkb_dn + kb) * 128, pol_w);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t id_up = idesc_bf16_f32(128, 128);
    const uint32_t id_dn = idesc_bf16_f32(128, NCT * 128);
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i <= nu; ++i) {
      if (i < nu) {
        const int b = i & 1;                       // up accumulator buffer
        mbar_wait(&uptempty[b], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb_up; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = smem_desc_k_sw128(smem_u32(sR + s * kStage));
            const uint64_t bd = smem_desc_k_sw128(smem_u32(sR + s * kStage + kTile));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss(tmem + kColUp + b * 128, ad + 2 * kk, bd + 2 * kk, id_up, (kb | kk) != 0);
            mma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (elect_one()) mma_commit(&upfull[b]);
        __syncwarp();
      }
      if (i >= 1) {
        const uint32_t par = (i - 1) & 1;
        mbar_wait(dntempty, par ^ 1);   // the previous unit's down accumulator was drained
        mbar_wait(hfull, par);            // every slice of this unit's H is in this CTA
        fence_proxy_async_shared();       // H was written by the generic proxy (st / st.async)
        tc_fence_after();
        for (int kb = 0; kb < nkb_dn; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = smem_desc_k_sw128(smem_u32(sH + kb * kTile));
            const uint64_t bd = smem_desc_k_sw128(smem_u32(sR + s * kStage));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss(tmem + kColDn, ad + 2 * kk, bd + 2 * kk, id_dn, (kb | kk) != 0);
            mma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (elect_one()) {
          mma_commit(dnfull);
          mma_commit_mc(hempty, static_cast<uint16_t>((1u << CS) - 1));   // H free, cluster-wide
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- H drain + exchange
    const int wq = warp & 3;
    const int t = wq * 32 + lane;                         // chunk row = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    uint32_t hbar[CS], hrow[CS];                          // every CTA's hfull / H row base
#pragma unroll
    for (int q = 0; q < CS; ++q) {
      hbar[q] = mapa_shared(smem_u32(hfull), q);
      hrow[q] = mapa_shared(smem_u32(sH + t * 128), q);
    }
    uint8_t* my_row = sH + t * 128;
    for (int k = 0; k < nu; ++k) {
      const int b = k & 1;
      mbar_wait(&upfull[b], (k >> 1) & 1);
      mbar_wait(hempty, (k & 1) ^ 1);   // every CTA's down MMAs of the previous unit are done
      tc_fence_after();
      if (wq == 0 && lane == 0)         // the bytes the peers' st.async will deliver here
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(hfull)),
                     "r"((CS - 1) * 2 * kTile) : "memory");
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kColUp + b * 128 + c0, r);
        tmem_ld_wait();
        const uint32_t tile = (2 * j + c0 / 64) * kTile;
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {   // 8 features = one 16-B chunk
          uint32_t w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const __nv_bfloat162 v = __floats2bfloat162_rn(fmaxf(__uint_as_float(r[8 * q8 + 2 * i]), 0.f),
                                                           fmaxf(__uint_as_float(r[8 * q8 + 2 * i + 1]), 0.f));
            w[i] = *reinterpret_cast<const uint32_t*>(&v);
          }
          const uint32_t off = tile + ((((c0 % 64) / 8 + q8) ^ (t & 7)) << 4);
          const uint4 v4 = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint4*>(my_row + off) = v4;
#pragma unroll
          for (int q = 1; q < CS; ++q) {
            const uint32_t peer = (j + q) % CS;
            st_async_v4(hrow[peer] + off, v4, hbar[peer]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&uptempty[b]);
        mbar_arrive(hfull);
      }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------------- output drain
    const int wq = warp & 3;
    const int t = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const int cj = h / CS;                                // output columns of this CTA
    for (int k = 0; k < nu; ++k) {
      int e, tok0, ntok;
      mlp_unit(cid + k * ncl, E, s_pref, s_pos, s_cnt, e, tok0, ntok);
      mbar_wait(dnfull, k & 1);
      tc_fence_after();
      const bool valid = t < ntok;
      int row = 0;
      float g = 0.f;
      if (valid) {
        row = __ldg(p.perm + tok0 + t);
        g = __ldg(&p.route[row].gate);
      }
      __nv_bfloat16* dst;
      if (p.p2p_n > 0) {   // the owner's receive slot for this rank, over NVLink
        const int o = row / p.p2p_n;
        dst = p.p2p_out[o] + static_cast<size_t>(row - o * p.p2p_n) * p.ld_out;
      } else {
        dst = p.out + static_cast<size_t>(row) * p.ld_out;
      }
      dst += j * cj;
#pragma unroll 1
      for (int c0 = 0; c0 < NCT * 128; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kColDn + c0, r);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const __nv_bfloat162 v = __floats2bfloat162_rn(g * __uint_as_float(r[8 * q + 2 * i]),
                                                             g * __uint_as_float(r[8 * q + 2 * i + 1]));
              w[i] = *reinterpret_cast<const uint32_t*>(&v);
            }
            *reinterpret_cast<uint4*>(dst + c0 + 8 * q) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dntempty);
    }
    if (p.p2p_n > 0) __threadfence_system();   // remote rows before the signal kernel
  }
  tc_fence_before();
  cluster_sync_all();   // no CTA leaves while a peer may still copy into its H
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

size_t mlp_smem_bytes(int E, int F) {
  const int h_bytes = (F / 64) * kTile;
  const int S = std::min(6, (kSmemBudget - h_bytes) / kStage);
  return 1024 + h_bytes + S * kStage + (2 * S + 8) * 8 + 16 + (3 * E + 1 + 33) * 4;
}

template <int CS, int NCT>
cudaError_t launch_mlp(const CUtensorMap& tmX, const CUtensorMap& tmWi, const CUtensorMap& tmWo,
                       const MlpArgs& a, int num_sms, cudaStream_t s) {
  static PerDeviceOnce attr;
  if (attr.need()) {
    cudaError_t e = cudaFuncSetAttribute(
        tc_expert_mlp<CS, NCT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(std::min<size_t>(mlp_smem_bytes(kMaxExperts, CS * 128), kMaxSmem)));
    if (e != cudaSuccess) return e;
    attr.done();
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreadsMlp);
  cfg.dynamicSmemBytes = mlp_smem_bytes(a.dn.E, a.F);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // Persistent grid = the clusters that can be resident at once. A cluster must fit in one
  // GPC, so e.g. only 45 three-CTA clusters fit on 148 SMs (not 49); launching more would
  // run the rest as a second wave after the first finished.
  static int max_cl[9] = {0};   // per cluster size, first device queried (all B200s alike)
  if (max_cl[CS] == 0) {
    cfg.gridDim = dim3((num_sms / CS) * CS);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tc_expert_mlp<CS, NCT>, &cfg) != cudaSuccess || n <= 0)
      n = num_sms / CS;
    cudaGetLastError();
    max_cl[CS] = std::min(n, num_sms / CS);
  }
  cfg.gridDim = dim3(max_cl[CS] * CS);
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, tc_expert_mlp<CS, NCT>, tmX, tmWi, tmWo, a);
}

}  // namespace

bool expert_mlp_supported(int h, int F, int E) {
  if (F % 128 || E > kThreadsMlp) return false;
  const int cs = F / 128;
  if (cs < 2 || cs > 4 || h % (128 * cs)) return false;
  const int nct = h / (128 * cs);
  return (nct == 1 || nct == 2) && mlp_smem_bytes(E, F) <= kMaxSmem;
}

cudaError_t launch_tc_expert_mlp(const CUtensorMap& tmX128, const CUtensorMap& tmWi,
                                 const CUtensorMap& tmWo, const TcParams& dn, int h, int F,
                                 int num_sms, cudaStream_t s) {
  MlpArgs a{dn, h, F};
  const int cs = F / 128, nct = h / (128 * cs);
  switch (cs * 10 + nct) {
    case 21: return launch_mlp<2, 1>(tmX128, tmWi, tmWo, a, num_sms, s);
    case 22: return launch_mlp<2, 2>(tmX128, tmWi, tmWo, a, num_sms, s);
    case 31: return launch_mlp<3, 1>(tmX128, tmWi, tmWo, a, num_sms, s);
    case 32: return launch_mlp<3, 2>(tmX128, tmWi, tmWo, a, num_sms, s);
    case 41: return launch_mlp<4, 1>(tmX128, tmWi, tmWo, a, num_sms, s);
    case 42: return launch_mlp<4, 2>(tmX128, tmWi, tmWo, a, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace moeshard
