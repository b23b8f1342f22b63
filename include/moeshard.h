/*
 * moeshard.h - C ABI of the B200-native MoEShard sharded Switch-MoE layer.
 *
 * The operation (arXiv 2503.08467, "Accelerating MoE Model Inference with
 * Expert Sharding", PAPER.md = the paper's LaTeX source):
 *
 *   Every GPU g of G calls forward(x) on its own tokens x [n, h]
 *   (Alg. 1). Each GPU holds one shard of EVERY
 *   expert: columns [g*d_ff/G, (g+1)*d_ff/G) of W_i and the same rows of W_o
 *   (Sec. 3.2). The router is replicated
 *   (PAPER.md:249). The five steps are
 *     1 route      m_expert <- router(x)
 *     2 metadata   groupPerExpert / countPerExpert, send
 *     3 scatter    replicate all tokens on all GPUs
 *     4 compute    every GPU runs all tokens through its   PAPER.md:203-209, 282-287,
 *                  shard of their expert, fused over all    339-345 (Sec. 3.3)
 *                  experts/GPUs into one grouped product
 *     5 gather     partial outputs back to the owner GPU
 *                  and point-wise summed (aggregateTokens)
 *   and GPU g's output is, for each of its tokens t,
 *     y_t = g_t * relu(x_t W_i^{e_t}) W_o^{e_t}   summed over the G shards,
 *   g_t = softmax(x_t W_r)[e_t], e_t = argmax (lowest index on ties).
 *   Readings of the paper used here are listed in DESIGN.md ("Readings").
 *
 * Conventions (all entry points):
 *   - Return MOESHARD_OK (0) or a negative moeshard_status; no exceptions
 *     cross the ABI. moeshard_last_error() gives the detailed text (e.g.
 *     both shapes on a shape error).
 *   - Ownership: the CALLER owns every buffer it passes (hidden, router_w,
 *     hidden_out, workspace, weight storage, routing outputs); the library
 *     never frees caller memory and performs no device allocation inside
 *     moeshard_forward. The library owns only its context object and, for
 *     world > 1 (or MOESHARD_FLAG_FORCE_COLLECTIVES), an NCCL communicator.
 *   - Pointers marked [dev] are device pointers on the context's device;
 *     [host] are host pointers. `stream` is a cudaStream_t passed as void*.
 *   - moeshard_forward is enqueue-only on `stream`: no host synchronisation,
 *     no data-dependent launch geometry, CUDA-graph capturable. With a
 *     communicator the token AllGather runs on a context-owned side stream
 *     forked from `stream` by an event and joined back before the call
 *     returns, so `stream` still orders all of the call's work.
 *   - Collective calls (moeshard_init, moeshard_forward) must be made by all
 *     `world` ranks in the same order with the same `layer` and `n_local`
 *     (with MOESHARD_FLAG_UNEVEN_TOKENS n_local may differ between ranks).
 */
#ifndef MOESHARD_H
#define MOESHARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOESHARD_OK = 0,
  MOESHARD_ERR_INVALID_ARG = -1,  /* null pointer, negative size, bad enum */
  MOESHARD_ERR_SHAPE = -2,        /* shape mismatch (message names both shapes) */
  MOESHARD_ERR_DIVISIBILITY = -3, /* d_ff not divisible by world */
  MOESHARD_ERR_BOUNDS = -4,       /* rank/layer/n_local out of range */
  MOESHARD_ERR_CONFIG = -5,       /* unsupported configuration or device (not sm_100) */
  MOESHARD_ERR_NOT_LOADED = -6,   /* forward on a layer whose shards were never loaded */
  MOESHARD_ERR_PROTOCOL = -7,     /* ranks disagree (collective contract violated) */
  MOESHARD_ERR_CUDA = -8,         /* CUDA runtime / driver error */
  MOESHARD_ERR_NCCL = -9          /* NCCL error */
} moeshard_status;

typedef enum {
  MOESHARD_BF16 = 0, /* bf16 storage, fp32 accumulation, tcgen05 tensor cores */
  MOESHARD_FP32 = 1  /* fp32 validation mode: fp32 everywhere, FFMA on CUDA cores */
} moeshard_dtype;

/* config.flags (any other bit is rejected with MOESHARD_ERR_INVALID_ARG; bits 0x8-0x40,
 * 0x100, 0x400 and 0x800 held round-1 experiments that measured slower and were removed) */
#define MOESHARD_FLAG_FORCE_COLLECTIVES 0x1u /* run the AllGather/ReduceScatter path even at world = 1 */
#define MOESHARD_FLAG_SIMT_GEMM 0x2u         /* bf16 mode: CUDA-core grouped GEMM (ablation / debug) */
#define MOESHARD_FLAG_UNFUSED_GEMM 0x4u      /* bf16 mode: up and down products as two launches (ablation) */
#define MOESHARD_FLAG_NO_L2_PERSIST 0x80u    /* bf16 mode: leave the device's persisting-L2 limit alone (see moeshard_init) */
#define MOESHARD_FLAG_DYNAMIC_SCHED 0x1000u  /* fused FFN: clusters take work units from a global counter (correct even when not every cluster is resident, e.g. ranks sharing a GPU); default static round robin */
#define MOESHARD_FLAG_UNEVEN_TOKENS 0x2000u  /* world > 1: ranks may pass different n_local each forward; token slots of max_tokens_per_rank rows per rank, routing tables [world * max_tokens_per_rank] with expert -1 in unused slots */
#define MOESHARD_FLAG_P2P 0x200u             /* bf16: Steps 3 and 5 by device-initiated stores into peer GPU memory instead of NCCL (see moeshard_p2p_*) */
#define MOESHARD_FLAG_SERIAL_AG 0x4000u      /* NCCL transport: token AllGather on the caller's stream after the router (default: a side stream, overlapping the router) */
/* The paper's comparison system instead of MoEShard: expert parallelism with
 * the DeepSpeed capacity of PAPER.md:393-398. Rank r hosts the E/world whole experts
 * [r*E/world, (r+1)*E/world) - moeshard_load_expert_shards then takes w_in [E/world][h][d_ff]
 * and w_out [E/world][d_ff][h] - and every admitted token is computed only by its expert's host:
 * all-to-all scatter and gather over peer memory (requires MOESHARD_FLAG_P2P and E % world == 0;
 * token slots of max_tokens_per_rank rows as with MOESHARD_FLAG_UNEVEN_TOKENS). Each expert
 * admits at most cap = ceil(CF * n_local / E) tokens of a rank's minibatch, first come (token
 * order); a dropped token's output row is zero. CF = config.ep_capacity_factor, or min(E, 50)
 * when <= 0. Baseline for measurement; MoEShard itself never drops a token. */
#define MOESHARD_FLAG_EXPERT_PARALLEL 0x8000u
/* Sec. 3.3 ablation (the paper's "without MegaBlocks" mode): instead of one
 * fused grouped launch, one up + one down tcgen05 launch per expert (2E launches; the paper's
 * first optimisation alone) ... */
#define MOESHARD_FLAG_LAUNCH_PER_EXPERT 0x10000u
/* ... or per (source rank, expert) (2 E world launches; neither optimisation). bf16 only. */
#define MOESHARD_FLAG_LAUNCH_PER_SOURCE 0x20000u
/* Narrow shards (d_ff/world in {256, 384, 512}, e.g. world = 8): run both products of each
 * expert's <= 128-token chunk in one thread-block cluster of d_ff/world/128 CTAs with the
 * intermediate H kept on chip (exchanged over distributed shared memory) instead of the
 * default two-phase fused FFN (H through L2). Bitwise-identical results; measured 5% faster
 * at the C2 G = 8 shard and 44% slower at C5 G = 8, hence opt-in. Ignored
 * where the shape does not qualify. */
#define MOESHARD_FLAG_ONCHIP_H 0x40000u

/* moeshard_forward_stages masks: ROUTE = Step 1 + the token exchange (Step 3 push),
 * COMPUTE = Steps 2 and 4 (+ the Step 5 send in P2P mode), REDUCE = the Step 5 aggregate. */
#define MOESHARD_STAGE_ROUTE 0x1
#define MOESHARD_STAGE_COMPUTE 0x2
#define MOESHARD_STAGE_REDUCE 0x4
#define MOESHARD_STAGE_ALL 0x7
#define MOESHARD_P2P_HANDLE_BYTES 64

typedef struct {
  int32_t d_model;             /* h; multiple of 128 */
  int32_t d_ff;                /* FULL expert hidden width; d_ff/world multiple of 128 */
  int32_t n_experts;           /* E, 1 <= E <= 256 */
  int32_t n_layers;            /* number of weight slots (MoE layers) this context serves */
  int32_t max_tokens_per_rank; /* upper bound on n_local */
  int32_t dtype;               /* moeshard_dtype */
  uint32_t flags;              /* MOESHARD_FLAG_* */
  float ep_capacity_factor;    /* MOESHARD_FLAG_EXPERT_PARALLEL only: CF (<= 0: min(E, 50)) */
  int32_t top_k;               /* experts per token (0 or 1: Switch top-1; 2: top-2 - PAPER.md:85
                                * "typically one or two" - the 2 largest logits, each weighted by
                                * its softmax probability, the two expert outputs summed, reading
                                * R21). top_k = 2 needs bf16 and the fused tcgen05 path (no P2P,
                                * EP, UNEVEN_TOKENS, SIMT/UNFUSED/LAUNCH_* or ONCHIP_H), and
                                * moeshard_forward's forced_expert then [n_local*2]. */
} moeshard_config;

typedef struct moeshard_ctx moeshard_ctx;

/* NCCL unique id for world > 1 (or FORCE_COLLECTIVES): call on rank 0 only,
 * broadcast the 128 bytes to all ranks (e.g. torch.distributed), pass to
 * moeshard_init. out: [host] 128 bytes. */
int moeshard_get_unique_id(uint8_t out[128]);

/* Bytes of device workspace moeshard_init needs for this config and world
 * size (activations, routing tables, permutation; sized for
 * world * max_tokens_per_rank tokens). bytes: [host] out. */
int moeshard_workspace_size(const moeshard_config* cfg, int world, size_t* bytes);

/* Bytes of device weight storage per layer: 2 * E * h * (d_ff/world) elements
 * of the config dtype (the same count, 2 * (E/world) * h * d_ff, for the
 * MOESHARD_FLAG_EXPERT_PARALLEL baseline). bytes_per_layer: [host] out. */
int moeshard_weight_storage_size(const moeshard_config* cfg, int world, size_t* bytes_per_layer);

/* Create a context for `rank` of `world` on CUDA `device`.
 * uid: [host] 128 bytes from moeshard_get_unique_id (ignored - may be NULL - when
 *      no NCCL communicator is needed: world == 1 without FORCE_COLLECTIVES, or
 *      MOESHARD_FLAG_P2P).
 * workspace: [dev] caller-owned, >= moeshard_workspace_size bytes, 256-B
 *      aligned, must stay alive until moeshard_destroy.
 * Errors: DIVISIBILITY (d_ff % world), CONFIG (shape limits, device not
 * sm_100), BOUNDS (rank not in [0, world)), NCCL, CUDA. Collective when a
 * communicator is created.
 * Side effect (bf16 mode, unless MOESHARD_FLAG_NO_L2_PERSIST): raises the
 * device's persisting-L2 limit (cudaLimitPersistingL2CacheSize) to 64 MB (or
 * the device maximum) so the kernels' evict_last lines - H between the two
 * products, the token rows re-read by every feature tile - stay in L2 while
 * the expert weights stream through it; never lowers an existing limit. */
int moeshard_init(moeshard_ctx** out, const moeshard_config* cfg, int rank, int world,
                  const uint8_t uid[128], void* workspace, size_t ws_bytes, int device);

/* loadShard (Alg. 1 Step 4): install this rank's shard
 * of every expert of `layer`.
 *   w_in_shard  [dev] [E][h][d_ff/world] row-major: columns rank*F..(rank+1)*F of W_i
 *   w_out_shard [dev] [E][d_ff/world][h] row-major: the same rows of W_o
 *   weight_storage [dev] caller-owned, >= moeshard_weight_storage_size bytes;
 *     the library repacks the shards into it (K-major: W_i^T, W_o^T per
 *     expert) and keeps using it until destroy or a reload of that layer.
 * The repack is enqueued on `stream`; the inputs may be freed after it. */
int moeshard_load_expert_shards(moeshard_ctx* ctx, int layer, const void* w_in_shard,
                                const void* w_out_shard, void* weight_storage, size_t bytes,
                                void* stream);

/* The MoEShard forward of one MoE layer (Alg. 1).
 *   hidden       [dev] [n_local][h] this rank's tokens (dtype of the config)
 *   router_w     [dev] [h][E] replicated router weight
 *   hidden_out   [dev] [n_local][h] MoE FFN output for this rank's tokens
 *                (no residual: Alg. 1 returns the aggregated tokens)
 *   forced_expert [dev] nullable [n_local] int32: the paper's replaced router
 *                (PAPER.md:368-372): e_t is taken from here, g_t is still
 *                softmax(x_t W_r)[e_t]; the router kernel still runs. Ids
 *                outside [0, E) are clamped and raise the sticky device error
 *                reported by moeshard_check().
 * n_local must satisfy 0 <= n_local <= max_tokens_per_rank and be equal on
 * all ranks - unless the context has MOESHARD_FLAG_UNEVEN_TOKENS: then every
 * rank passes its own n_local (0 included, and every rank must still call),
 * tokens travel in slots of max_tokens_per_rank rows per rank and the unused
 * tail of a slot is routed nowhere (the per-GPU sizes of Alg. 1 Step 2,
 * PAPER.md:191-195). Enqueue-only on `stream`. Errors: BOUNDS, NOT_LOADED,
 * INVALID_ARG, CUDA, NCCL. */
int moeshard_forward(moeshard_ctx* ctx, int layer, const void* hidden, int n_local,
                     const void* router_w, void* hidden_out, const int32_t* forced_expert,
                     void* stream);

/* Routing of the most recent forward (Steps 1-2), copied on `stream` into
 * caller device buffers (any may be NULL):
 *   (top_k = 2: one entry per (token, choice) assignment a = 2 t + j, j = 0 the larger logit:
 *    expert_all / gate_all / perm have world*n_local*2 entries, perm lists assignment ids)
 *   expert_all [dev] int32 [world*n_local]  e_t for all global tokens t = r*n + i
 *              (MOESHARD_FLAG_UNEVEN_TOKENS: [world*max_tokens_per_rank], t = r*cap + i,
 *              -1 where slot r has no token i; gate_all / perm likewise)
 *   gate_all   [dev] fp32  [world*n_local]  g_t
 *   counts     [dev] int32 [E]              m_sizes summed over ranks
 *   offsets    [dev] int32 [E+1]            exclusive scan of counts
 *   perm       [dev] int32 [world*n_local]  global token ids grouped by expert,
 *                                           ascending inside each expert */
/* moeshard_forward split into stages (a mask of MOESHARD_STAGE_*), run in order
 * ROUTE -> COMPUTE -> REDUCE with the same layer / n_local; moeshard_forward ==
 * all three. Lets a caller interleave other work between the exchange steps, or
 * drive several ranks that share one GPU in lock-step (each stage's waits are then
 * already satisfied). Errors: as moeshard_forward; PROTOCOL if n_local differs
 * from the ROUTE stage's or P2P is configured but not connected. */
int moeshard_forward_stages(moeshard_ctx* ctx, int layer, const void* hidden, int n_local,
                            const void* router_w, void* hidden_out, const int32_t* forced_expert,
                            int stages, void* stream);

/* Peer-memory exchange (MOESHARD_FLAG_P2P). Each rank's context owns one
 * exchange region - the only device memory the library allocates (cudaMalloc in
 * moeshard_init, freed by moeshard_destroy): flags, the rank-major x_all / route
 * records / block histograms every rank pushes into (Step 3), and G receive
 * slots the down-projection epilogues of all ranks store their partial output
 * rows into (Step 5). Setup, once, after moeshard_init on every rank:
 *   1. moeshard_p2p_export: this region's CUDA IPC handle (64 bytes [host] out);
 *   2. exchange the handles between the ranks (e.g. torch.distributed all_gather);
 *   3. moeshard_p2p_open: map a peer's handle in this process ([host] out:
 *      device pointer; closed at destroy). Ranks that share a process use
 *      moeshard_p2p_region's pointers directly instead;
 *   4. moeshard_p2p_connect(regions[world]): [host] array of every rank's region
 *      as seen from this process; regions[rank] must be this context's own.
 * moeshard_forward then needs no NCCL: every cross-rank wait inside it is a
 * bounded spin on a flag in the local region; a peer that never arrives makes
 * moeshard_check return PROTOCOL instead of hanging. Errors: CONFIG (context
 * without MOESHARD_FLAG_P2P), INVALID_ARG, PROTOCOL, CUDA. */
int moeshard_p2p_region(moeshard_ctx* ctx, void** dev_ptr, size_t* bytes);
int moeshard_p2p_export(moeshard_ctx* ctx, uint8_t handle[MOESHARD_P2P_HANDLE_BYTES]);
int moeshard_p2p_open(moeshard_ctx* ctx, const uint8_t handle[MOESHARD_P2P_HANDLE_BYTES],
                      void** dev_ptr);
int moeshard_p2p_connect(moeshard_ctx* ctx, void* const* regions);

int moeshard_get_routing(moeshard_ctx* ctx, int32_t* expert_all, float* gate_all, int32_t* counts,
                         int32_t* offsets, int32_t* perm, void* stream);

/* MOESHARD_FLAG_EXPERT_PARALLEL: the admission of the most recent forward, copied on `stream`
 * into caller device buffers (any may be NULL):
 *   owner    [dev] int32 [n_local]  rank hosting the expert of local token i, -1 if the
 *                                   expert's capacity dropped it (its output row is zero)
 *   expert   [dev] int32 [n_local]  e_i (global expert id) of local token i
 *   gate     [dev] fp32  [n_local]  g_i
 *   received [dev] int32 [E/world]  tokens (of all ranks) this rank's experts computed
 * (moeshard_get_routing on an EP context describes the host side: expert_all / gate_all /
 * perm over the world * max_tokens_per_rank received slots with LOCAL expert ids, -1 where
 * not received; counts / offsets over the E/world local experts.)
 * Errors: CONFIG (not an EP context), INVALID_ARG. */
int moeshard_get_ep_admission(moeshard_ctx* ctx, int32_t* owner, int32_t* expert, float* gate,
                              int32_t* received, void* stream);

/* Per-forward work counters of the most recent forward ([host] out, syncs
 * the stream): tokens seen, grouped-GEMM tiles executed by the up and down
 * products, and rows executed (tile padding included). */
typedef struct {
  int64_t n_tokens_global;
  int64_t tiles_up;
  int64_t tiles_down;
  int64_t rows_executed_up;   /* sum over tiles of the MMA N (tokens) actually issued */
  int64_t kernel_launches;    /* cumulative count of this context's kernel launches */
} moeshard_stats;
int moeshard_get_stats(moeshard_ctx* ctx, moeshard_stats* out, void* stream);

/* Phase timing (measurement only). enable != 0 starts recording CUDA events
 * at the phase boundaries of every moeshard_forward (ring of 1024 forwards)
 * and resets the accumulators; enable == 0 stops. moeshard_get_phase_ms
 * synchronises and writes into out[0..n) the total milliseconds spent, over
 * all forwards recorded since enabling, in the phases
 *   0 router, 1 token/metadata AllGather, 2 grouping (offsets, stable
 *   permutation, row gather), 3 grouped GEMM up, 4 grouped GEMM down,
 *   5 ReduceScatter
 * and returns the number of forwards in *count. */
int moeshard_profile(moeshard_ctx* ctx, int enable);
int moeshard_get_phase_ms(moeshard_ctx* ctx, float* out, int n, int* count);

/* Synchronise `stream` and report the sticky device error (forced id out of
 * range) and any asynchronous CUDA/NCCL error. */
int moeshard_check(moeshard_ctx* ctx, void* stream);

/* Text of the last error on this context (or of the last failed call made
 * with a NULL context, e.g. moeshard_init). Never NULL. */
const char* moeshard_last_error(const moeshard_ctx* ctx);
const char* moeshard_status_string(int status);

/* Release the communicator and the context. Caller memory is untouched. */
int moeshard_destroy(moeshard_ctx* ctx);

/* Library version string, e.g. "moeshard-b200 0.1 sm_100a". */
const char* moeshard_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MOESHARD_H */
