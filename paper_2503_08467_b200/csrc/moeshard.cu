// moeshard.cu - host orchestrator behind the C ABI (include/moeshard.h).
//
// Owns: the context, the carve-up of the caller's workspace, the per-layer
// packed weight tiles and their TMA descriptors, and either an NCCL
// communicator (world > 1; libnccl is dlopen'ed - with torch loaded this is the
// same library torch.distributed uses) or, with MOESHARD_FLAG_P2P, one exchange
// region mapped by every rank (p2p.cu). moeshard_forward(_stages) enqueues
// Alg. 1 on the caller's stream, kernels chained with
// programmatic dependent launch:
//
//   ROUTE    1 router_tc_kernel (local tokens: logits, softmax, top-1, block    Step 1
//              histograms)
//            2 ncclGroup{AllGather tokens, route records, histograms} or       Steps 2+3
//              push_tokens into every rank's region (P2P)
//   COMPUTE  3 group_block_scan + group_scatter_gather (offsets, stable perm,  Step 2 + Sec. 3.3
//              X_perm)                                                         concatenation
//            4 tc_moe_ffn_2sm: both grouped products in one persistent launch  Step 4
//              (ReLU; gate + un-permute scatter; P2P: partial rows stored into
//              their owner's receive slot)
//   REDUCE   5 ncclReduceScatter(sum), or reduce_partials over the receive     Step 5
//              slots (P2P)
//
// No host synchronisation and no allocation inside forward.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/moeshard.h"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "p2p.cuh"

using namespace moeshard;

namespace {

thread_local std::string g_err = "no error";

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  // optional (NCCL >= 2.18): a second communicator over the same ranks for the side stream
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  const char* env = getenv("MOESHARD_NCCL_LIB");
  if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define LOAD(name, sym)                                          \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, sym)); \
  if (!api.name) return api;
  LOAD(GetUniqueId, "ncclGetUniqueId");
  LOAD(CommInitRank, "ncclCommInitRank");
  LOAD(CommDestroy, "ncclCommDestroy");
  LOAD(CommGetAsyncError, "ncclCommGetAsyncError");
  LOAD(AllGather, "ncclAllGather");
  LOAD(ReduceScatter, "ncclReduceScatter");
  LOAD(GroupStart, "ncclGroupStart");
  LOAD(GroupEnd, "ncclGroupEnd");
  LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
  api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(dlsym(h, "ncclCommSplit"));
  api.ok = true;
  return api;
}

// ------------------------------------------------------------------ TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor [outer][inner] (inner contiguous), box [box_outer][64], 128-B swizzle.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
               uint32_t box_outer, bool swizzle = true) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr int kRouterTok = 128;    // tokens per tcgen05 router CTA (= TMEM lanes)
constexpr int kL2PersistMB = 64;   // measured best of 0/32/48/64/79 MB on c2
constexpr uint32_t kKnownFlags =
    MOESHARD_FLAG_FORCE_COLLECTIVES | MOESHARD_FLAG_SIMT_GEMM | MOESHARD_FLAG_UNFUSED_GEMM |
    MOESHARD_FLAG_NO_L2_PERSIST | MOESHARD_FLAG_DYNAMIC_SCHED | MOESHARD_FLAG_UNEVEN_TOKENS |
    MOESHARD_FLAG_P2P | MOESHARD_FLAG_SERIAL_AG | MOESHARD_FLAG_EXPERT_PARALLEL |
    MOESHARD_FLAG_LAUNCH_PER_EXPERT | MOESHARD_FLAG_LAUNCH_PER_SOURCE | MOESHARD_FLAG_ONCHIP_H;

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Workspace carve-up, shared by moeshard_workspace_size and moeshard_init.
struct Layout {
  size_t wt_r, route, block_hist, block_base, ints, done, perm, perm_pad, gate_pad, x_all, x_perm, H, partial,
      y_assign,
      ep_route, ep_hist, ep_owner, total;
  int n_ints;
  size_t npad;   // rows of the internal expert-ordered layout: N_max + 32 per expert, rounded to 64
};

Layout make_layout(const moeshard_config& c, int world) {
  const bool p2p = (c.flags & MOESHARD_FLAG_P2P) != 0;   // x_all / partials live in the region
  const bool coll = !p2p && (world > 1 || (c.flags & MOESHARD_FLAG_FORCE_COLLECTIVES));
  const size_t elt = c.dtype == MOESHARD_BF16 ? 2 : 4;
  const size_t Nmax = static_cast<size_t>(world) * c.max_tokens_per_rank;
  const size_t K = c.top_k > 1 ? static_cast<size_t>(c.top_k) : 1;   // assignments per token
  const size_t Amax = Nmax * K;
  // hist-blocks: >= 64 tokens each (128 for the tcgen05 router), per rank
  const size_t nb = std::max<size_t>(1, world * ((c.max_tokens_per_rank + 63) / 64));
  const bool ep = (c.flags & MOESHARD_FLAG_EXPERT_PARALLEL) != 0;
  const size_t E = c.n_experts, h = c.d_model, F = ep ? c.d_ff : c.d_ff / world;
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L.wt_r = take(static_cast<size_t>(round_up(c.n_experts, 16)) * h * elt);  // W_r^T, padded
  L.route = take(Amax * sizeof(RouteRec));
  L.block_hist = take(nb * E * 4);
  L.block_base = take(nb * E * 4);
  // counts, offsets, tc_chunk_pref, tc_chunk_size, simt_chunk_pref, stats[8], block_tot, pos,
  // next_unit
  L.n_ints = static_cast<int>(E + (E + 1) + (E + 1) + E + (E + 1) + 8 + E + (E + 1) + 1);
  L.npad = (Amax + kSegAlign * E + 63) / 64 * 64;
  L.ints = take(L.n_ints * 4);
  L.done = take((Amax / kTcTokTile + E + 8) * 4);   // per token chunk: <= A/256 + E chunks
  L.perm = take(Amax * 4);
  L.perm_pad = take(L.npad * 4);
  L.gate_pad = take(L.npad * 4);
  L.x_all = coll ? take(Nmax * h * elt) : 0;
  L.x_perm = take(L.npad * h * elt);
  L.H = take(L.npad * F * elt);
  L.partial = coll ? take(Nmax * h * elt) : 0;
  L.y_assign = K > 1 ? take(Amax * h * elt) : 0;   // top-k: one output row per assignment
  // EP baseline: this rank's own routing (the regions carry the hosts' copies)
  const size_t nmax = static_cast<size_t>(c.max_tokens_per_rank);
  L.ep_route = ep ? take(nmax * sizeof(RouteRec)) : 0;
  L.ep_hist = ep ? take(((nmax + 127) / 128 + 1) * E * 4) : 0;
  L.ep_owner = ep ? take(nmax * 4) : 0;
  L.total = off;
  return L;
}

}  // namespace

struct LayerW {
  bool loaded = false;
  CUtensorMap tm_in{}, tm_out{};  // packed weight tiles viewed as [rows][64], box 128 rows
  void* wt_in = nullptr;   // [E][F][h]  (W_i^T shard, K-major for the up product)
  void* wt_out = nullptr;  // [E][h][F]  (W_o^T shard, K-major for the down product)
};

struct moeshard_ctx {
  moeshard_config cfg{};
  int rank = 0, world = 1, device = 0, num_sms = 148;
  int h = 0, F = 0, E = 0, elt = 2;
  // EP baseline (MOESHARD_FLAG_EXPERT_PARALLEL): Et = experts hosted here (E / world), F = d_ff;
  // MoEShard: Et = E, F = d_ff / world. The router always sees all E experts.
  bool ep = false;
  int Et = 0;
  float ep_cf = 0.f;
  RouteRec* ep_route = nullptr;
  int32_t *ep_hist = nullptr, *ep_owner = nullptr;
  bool coll = false, use_tc = true;
  Layout L{};
  char* ws = nullptr;
  RouteRec* route = nullptr;
  int32_t *block_hist = nullptr, *block_base = nullptr, *block_tot = nullptr, *perm = nullptr;
  Tables tb{};
  void *x_all = nullptr, *x_perm = nullptr, *H = nullptr, *partial = nullptr;
  int K = 1;                    // top_k: (token, expert) assignments per token
  void* y_assign = nullptr;     // top_k > 1: [A_max][h] one output row per assignment
  CUtensorMap tm_xperm{}, tm_H{}, tm_xperm16{}, tm_H16{}, tm_xperm128{}, tm_wt_r{};
  void* wt_r = nullptr;
  int EP = 16;
  std::vector<LayerW> layers;
  ncclComm_t comm = nullptr;
  // the token AllGather forked onto s_x runs on its own communicator (split from comm): two
  // streams never issue concurrent operations on one communicator, whatever NCCL's ordering
  ncclComm_t comm_x = nullptr;
  // Step 3 token AllGather overlapped with Step 1 (x does not depend on the routing): the
  // AllGather of x runs on s_x, forked from the caller's stream before the router and joined
  // after the metadata AllGather (MOESHARD_FLAG_SERIAL_AG: everything on the caller's stream)
  bool overlap_ag = true;
  cudaStream_t s_x = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // peer-memory exchange (MOESHARD_FLAG_P2P): this rank's region (library-owned) and
  // every rank's region as mapped here; opened IPC mappings are closed at destroy
  bool p2p = false, connected = false;
  char* region = nullptr;
  P2PLayout PL{};
  P2PArgs pa{};
  std::vector<void*> ipc_opened;
  int last_n = 0;
  int64_t launches = 0;  // cumulative kernel launches of this context
  // phase profiling (measurement only)
  bool prof = false;
  static constexpr int kRing = 1024, kEv = 7;
  std::vector<cudaEvent_t> ev;  // kRing * kEv
  int prof_count = 0;
  std::string err = "no error";
  void mark(int phase, cudaStream_t s) {
    if (prof) cudaEventRecord(ev[(prof_count % kRing) * kEv + phase], s);
  }
};

namespace {

int fail(moeshard_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_err = buf;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                            \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(ctx, MOESHARD_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    ncclResult_t _r = (expr);                                                                \
    if (_r != ncclSuccess)                                                                   \
      return fail(ctx, MOESHARD_ERR_NCCL, "%s failed: %s", #expr, nccl().GetErrorString(_r)); \
  } while (0)

// an internal step that already recorded its error: propagate the status code
#define CUDA_TRY_RET(ctx, expr) \
  do {                          \
    const int _st = (expr);     \
    if (_st != MOESHARD_OK) return _st; \
  } while (0)

namespace {

// Step 3: replicate every rank's tokens into x_all (rank-major slots of
// ns rows). With MOESHARD_FLAG_UNEVEN_TOKENS the n rows go to this rank's slot first and the
// AllGather sends the whole slot in place.
int allgather_tokens(moeshard_ctx* c, const void* hidden, int n, int ns, bool uneven,
                     ncclDataType_t ndt, cudaStream_t st) {
  const void* xsend = hidden;
  if (uneven) {
    char* slot = static_cast<char*>(c->x_all) + static_cast<size_t>(c->rank) * ns * c->h * c->elt;
    if (n > 0)
      CUDA_TRY(c, cudaMemcpyAsync(slot, hidden, static_cast<size_t>(n) * c->h * c->elt,
                                  cudaMemcpyDeviceToDevice, st));
    xsend = slot;
  }
  NCCL_TRY(c, nccl().AllGather(xsend, c->x_all, static_cast<size_t>(ns) * c->h, ndt,
                               st == c->s_x && c->comm_x ? c->comm_x : c->comm, st));
  return MOESHARD_OK;
}

}  // namespace

// Step 5 send (peer memory): the down epilogue stores the partial row of global token t into
// its owner's receive slot for this rank
void set_p2p_out(const moeshard_ctx* c, TcParams& dn, int ns) {
  dn.p2p_n = ns;
  for (int g = 0; g < c->world; ++g)
    dn.p2p_out[g] = reinterpret_cast<__nv_bfloat16*>(
        c->pa.peers[g] + c->PL.off_recv + static_cast<size_t>(c->rank) * c->pa.n_max * c->h * 2);
}

int validate(const moeshard_config* c, int world) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "config is NULL");
  if (world < 1) return fail(nullptr, MOESHARD_ERR_BOUNDS, "world=%d must be >= 1", world);
  if (c->dtype != MOESHARD_BF16 && c->dtype != MOESHARD_FP32)
    return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "dtype=%d is not BF16(0)/FP32(1)", c->dtype);
  if (c->n_experts < 1 || c->n_experts > 256)
    return fail(nullptr, MOESHARD_ERR_CONFIG, "n_experts=%d outside [1, 256]", c->n_experts);
  if (c->d_model < 128 || c->d_model % 128)
    return fail(nullptr, MOESHARD_ERR_CONFIG, "d_model=%d must be a positive multiple of 128",
                c->d_model);
  if (c->d_ff < 1 || c->d_ff % world)
    return fail(nullptr, MOESHARD_ERR_DIVISIBILITY,
                "d_ff=%d is not divisible by world=%d (PAPER.md:169, 329-330)", c->d_ff, world);
  const bool ep = (c->flags & MOESHARD_FLAG_EXPERT_PARALLEL) != 0;
  if (!ep && (c->d_ff / world) % 128)
    return fail(nullptr, MOESHARD_ERR_CONFIG, "d_ff/world=%d must be a multiple of 128",
                c->d_ff / world);
  if (ep && (!(c->flags & MOESHARD_FLAG_P2P) || c->n_experts % world || c->d_ff % 128))
    return fail(nullptr, MOESHARD_ERR_CONFIG,
                "MOESHARD_FLAG_EXPERT_PARALLEL needs MOESHARD_FLAG_P2P, E %% world == 0 and d_ff %% 128 "
                "== 0 (E=%d, world=%d, d_ff=%d)", c->n_experts, world, c->d_ff);
  if (c->n_layers < 1) return fail(nullptr, MOESHARD_ERR_CONFIG, "n_layers=%d < 1", c->n_layers);
  if (c->top_k < 0 || c->top_k > 2 || c->top_k > c->n_experts)
    return fail(nullptr, MOESHARD_ERR_CONFIG, "top_k=%d not in {0, 1, 2} or > n_experts=%d",
                c->top_k, c->n_experts);
  if (c->top_k == 2 &&
      (c->dtype != MOESHARD_BF16 ||
       (c->flags & (MOESHARD_FLAG_P2P | MOESHARD_FLAG_EXPERT_PARALLEL | MOESHARD_FLAG_UNEVEN_TOKENS |
                    MOESHARD_FLAG_SIMT_GEMM | MOESHARD_FLAG_UNFUSED_GEMM |
                    MOESHARD_FLAG_LAUNCH_PER_EXPERT | MOESHARD_FLAG_LAUNCH_PER_SOURCE |
                    MOESHARD_FLAG_ONCHIP_H))))
    return fail(nullptr, MOESHARD_ERR_CONFIG,
                "top_k=2 needs bf16 and the fused tcgen05 path (no P2P / EXPERT_PARALLEL / "
                "UNEVEN_TOKENS / SIMT_GEMM / UNFUSED_GEMM / LAUNCH_* / ONCHIP_H)");
  if (c->flags & ~kKnownFlags)
    return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "flags=0x%x has unknown bits (0x%x)", c->flags,
                c->flags & ~kKnownFlags);
  if ((c->flags & MOESHARD_FLAG_P2P) &&
      (c->dtype != MOESHARD_BF16 || world > kMaxWorld ||
       (c->flags & (MOESHARD_FLAG_SIMT_GEMM | MOESHARD_FLAG_UNFUSED_GEMM | MOESHARD_FLAG_FORCE_COLLECTIVES))))
    return fail(nullptr, MOESHARD_ERR_CONFIG,
                "MOESHARD_FLAG_P2P needs bf16, the fused tcgen05 FFN, no FORCE_COLLECTIVES and "
                "world <= %d (world=%d)", kMaxWorld, world);
  if (c->max_tokens_per_rank < 0 ||
      static_cast<long long>(c->max_tokens_per_rank) * world > (1LL << 30))
    return fail(nullptr, MOESHARD_ERR_CONFIG, "max_tokens_per_rank=%d out of range",
                c->max_tokens_per_rank);
  return MOESHARD_OK;
}

}  // namespace

extern "C" {

const char* moeshard_version(void) { return "moeshard-b200 0.1 sm_100a"; }

const char* moeshard_status_string(int s) {
  switch (s) {
    case MOESHARD_OK: return "MOESHARD_OK";
    case MOESHARD_ERR_INVALID_ARG: return "MOESHARD_ERR_INVALID_ARG";
    case MOESHARD_ERR_SHAPE: return "MOESHARD_ERR_SHAPE";
    case MOESHARD_ERR_DIVISIBILITY: return "MOESHARD_ERR_DIVISIBILITY";
    case MOESHARD_ERR_BOUNDS: return "MOESHARD_ERR_BOUNDS";
    case MOESHARD_ERR_CONFIG: return "MOESHARD_ERR_CONFIG";
    case MOESHARD_ERR_NOT_LOADED: return "MOESHARD_ERR_NOT_LOADED";
    case MOESHARD_ERR_PROTOCOL: return "MOESHARD_ERR_PROTOCOL";
    case MOESHARD_ERR_CUDA: return "MOESHARD_ERR_CUDA";
    case MOESHARD_ERR_NCCL: return "MOESHARD_ERR_NCCL";
    default: return "MOESHARD_ERR_UNKNOWN";
  }
}

const char* moeshard_last_error(const moeshard_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

int moeshard_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "out is NULL");
  if (!nccl().ok) return fail(nullptr, MOESHARD_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NCCL_TRY(nullptr, nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, 128);
  return MOESHARD_OK;
}

int moeshard_workspace_size(const moeshard_config* cfg, int world, size_t* bytes) {
  int st = validate(cfg, world);
  if (st) return st;
  if (!bytes) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = make_layout(*cfg, world).total;
  return MOESHARD_OK;
}

int moeshard_weight_storage_size(const moeshard_config* cfg, int world, size_t* bytes) {
  int st = validate(cfg, world);
  if (st) return st;
  if (!bytes) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "bytes is NULL");
  const size_t elt = cfg->dtype == MOESHARD_BF16 ? 2 : 4;
  *bytes = 2 * static_cast<size_t>(cfg->n_experts) * cfg->d_model * (cfg->d_ff / world) * elt;
  return MOESHARD_OK;
}

int moeshard_init(moeshard_ctx** out, const moeshard_config* cfg, int rank, int world,
                  const uint8_t uid[128], void* workspace, size_t ws_bytes, int device) {
  if (!out) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int st = validate(cfg, world);
  if (st) return st;
  if (rank < 0 || rank >= world)
    return fail(nullptr, MOESHARD_ERR_BOUNDS, "rank=%d not in [0, world=%d)", rank, world);
  Layout L = make_layout(*cfg, world);
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "workspace NULL or not 256-B aligned");
  if (ws_bytes < L.total)
    return fail(nullptr, MOESHARD_ERR_SHAPE, "workspace has %zu bytes, needs %zu", ws_bytes,
                L.total);
  int ndev = 0;
  CUDA_TRY(nullptr, cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return fail(nullptr, MOESHARD_ERR_BOUNDS, "device=%d not in [0, %d)", device, ndev);
  CUDA_TRY(nullptr, cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(nullptr, cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(nullptr, MOESHARD_ERR_CONFIG,
                "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device,
                prop.major, prop.minor);

  auto* c = new moeshard_ctx();
  c->cfg = *cfg;
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->h = cfg->d_model;
  c->ep = (cfg->flags & MOESHARD_FLAG_EXPERT_PARALLEL) != 0;
  c->F = c->ep ? cfg->d_ff : cfg->d_ff / world;
  c->E = cfg->n_experts;
  c->Et = c->ep ? cfg->n_experts / world : cfg->n_experts;
  c->ep_cf = cfg->ep_capacity_factor > 0.f ? cfg->ep_capacity_factor
                                          : static_cast<float>(std::min(cfg->n_experts, 50));
  c->elt = cfg->dtype == MOESHARD_BF16 ? 2 : 4;
  c->p2p = (c->cfg.flags & MOESHARD_FLAG_P2P) != 0;
  // coll: tokens of all ranks are exchanged (rank-major x_all / route / hist buffers)
  c->coll = world > 1 || (c->cfg.flags & MOESHARD_FLAG_FORCE_COLLECTIVES) || c->p2p;
  c->use_tc = cfg->dtype == MOESHARD_BF16 && !(c->cfg.flags & MOESHARD_FLAG_SIMT_GEMM);
  // L2 set-aside for the kernels' evict_last lines (H between the two products, the
  // expert-ordered token rows re-read by every feature tile): without it the
  // 128-B-line hints lose to the weight stream. Raised, never lowered; device-wide.
  if (c->use_tc && !(c->cfg.flags & MOESHARD_FLAG_NO_L2_PERSIST)) {
    size_t want = static_cast<size_t>(kL2PersistMB) << 20, cur = 0;
    want = std::min(want, static_cast<size_t>(prop.persistingL2CacheMaxSize));
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess && cur < want)
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    cudaGetLastError();   // a refused set-aside is not an error (e.g. MIG, MPS)
  }
  c->L = L;
  c->ws = static_cast<char*>(workspace);
  c->route = reinterpret_cast<RouteRec*>(c->ws + L.route);
  c->wt_r = c->ws + L.wt_r;
  c->EP = round_up(c->E, 16);
  c->block_hist = reinterpret_cast<int32_t*>(c->ws + L.block_hist);
  c->block_base = reinterpret_cast<int32_t*>(c->ws + L.block_base);
  int32_t* ints = reinterpret_cast<int32_t*>(c->ws + L.ints);
  const int E = c->E;
  c->tb.counts = ints;
  c->tb.offsets = ints + E;
  c->tb.tc_chunk_pref = c->tb.offsets + (E + 1);
  c->tb.tc_chunk_size = c->tb.tc_chunk_pref + (E + 1);
  c->tb.simt_chunk_pref = c->tb.tc_chunk_size + E;
  c->tb.stats = c->tb.simt_chunk_pref + (E + 1);
  c->tb.done = reinterpret_cast<int32_t*>(c->ws + L.done);
  c->block_tot = c->tb.stats + 8;
  c->tb.pos = c->block_tot + E;
  c->tb.next_unit = c->tb.pos + (E + 1);
  c->tb.perm_pad = reinterpret_cast<int32_t*>(c->ws + L.perm_pad);
  c->tb.gate_pad = reinterpret_cast<float*>(c->ws + L.gate_pad);
  c->perm = reinterpret_cast<int32_t*>(c->ws + L.perm);
  c->x_all = c->coll && !c->p2p ? c->ws + L.x_all : nullptr;
  c->x_perm = c->ws + L.x_perm;
  c->H = c->ws + L.H;
  c->partial = c->coll && !c->p2p ? c->ws + L.partial : nullptr;
  c->K = cfg->top_k > 1 ? cfg->top_k : 1;
  c->y_assign = c->K > 1 ? c->ws + L.y_assign : nullptr;
  if (c->ep) {
    c->ep_route = reinterpret_cast<RouteRec*>(c->ws + L.ep_route);
    c->ep_hist = reinterpret_cast<int32_t*>(c->ws + L.ep_hist);
    c->ep_owner = reinterpret_cast<int32_t*>(c->ws + L.ep_owner);
  }
  c->layers.resize(cfg->n_layers);
  cudaError_t e = cudaMemset(ints, 0, L.n_ints * 4);
  if (e == cudaSuccess) e = cudaMemset(c->tb.done, 0, L.perm - L.done);
  if (e != cudaSuccess) {
    delete c;
    return fail(nullptr, MOESHARD_ERR_CUDA, "cudaMemset: %s", cudaGetErrorString(e));
  }
  const int Nmax = world * cfg->max_tokens_per_rank;
  if (c->use_tc && Nmax > 0) {
    const uint64_t np = L.npad;
    if (!make_tmap(&c->tm_xperm, c->x_perm, c->h, np, 32) ||
        !make_tmap(&c->tm_H, c->H, c->F, np, 32) ||
        !make_tmap(&c->tm_xperm16, c->x_perm, c->h, np, 16) ||
        !make_tmap(&c->tm_H16, c->H, c->F, np, 16) ||
        !make_tmap(&c->tm_xperm128, c->x_perm, c->h, np, 128) ||
        !make_tmap(&c->tm_wt_r, c->wt_r, c->h, c->EP, c->EP)) {
      delete c;
      return fail(nullptr, MOESHARD_ERR_CUDA, "cuTensorMapEncodeTiled failed for activations");
    }
  }
  if (c->p2p) {
    // the exchange region: the one device allocation the library owns (CUDA IPC needs
    // the base of a cudaMalloc); x_all / route records / block histograms live in it
    const int nbr_max = (cfg->max_tokens_per_rank + 63) / 64;
    c->PL = p2p_layout(world, std::max(1, cfg->max_tokens_per_rank), c->h, E, std::max(1, nbr_max));
    void* reg = nullptr;
    cudaError_t er = cudaMalloc(&reg, c->PL.total);
    if (er == cudaSuccess) er = cudaMemset(reg, 0, c->PL.total);
    if (er != cudaSuccess) {
      if (reg) cudaFree(reg);
      delete c;
      return fail(nullptr, MOESHARD_ERR_CUDA, "exchange region (%zu B): %s", c->PL.total,
                  cudaGetErrorString(er));
    }
    c->region = static_cast<char*>(reg);
    c->x_all = c->region + c->PL.off_x;
    c->route = reinterpret_cast<RouteRec*>(c->region + c->PL.off_route);
    c->block_hist = reinterpret_cast<int32_t*>(c->region + c->PL.off_hist);
    c->pa.self = c->region;
    c->pa.rank = rank;
    c->pa.world = world;
    c->pa.n_max = std::max(1, cfg->max_tokens_per_rank);
    c->pa.off_x = c->PL.off_x;
    c->pa.off_route = c->PL.off_route;
    c->pa.off_hist = c->PL.off_hist;
    c->pa.off_recv = c->PL.off_recv;
  } else if (c->coll) {
    if (!uid) {
      delete c;
      return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "uid is NULL but a communicator is needed");
    }
    if (!nccl().ok) {
      delete c;
      return fail(nullptr, MOESHARD_ERR_NCCL, "libnccl.so.2 could not be loaded");
    }
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(nullptr, MOESHARD_ERR_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
    // the side-stream token AllGather needs its own communicator (collective over the ranks:
    // every rank's moeshard_init reaches this point); without ncclCommSplit it runs serially
    c->overlap_ag = !(c->cfg.flags & MOESHARD_FLAG_SERIAL_AG) && nccl().CommSplit != nullptr;
    if (c->overlap_ag) {
      r = nccl().CommSplit(c->comm, 0, rank, &c->comm_x, nullptr);
      if (r != ncclSuccess) {
        moeshard_destroy(c);
        return fail(nullptr, MOESHARD_ERR_NCCL, "ncclCommSplit: %s", nccl().GetErrorString(r));
      }
    }
    if (c->overlap_ag &&
        (cudaStreamCreateWithFlags(&c->s_x, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
      moeshard_destroy(c);
      return fail(nullptr, MOESHARD_ERR_CUDA, "side stream / events for the token AllGather");
    }
  }
  *out = c;
  return MOESHARD_OK;
}

int moeshard_load_expert_shards(moeshard_ctx* c, int layer, const void* w_in_shard,
                                const void* w_out_shard, void* storage, size_t bytes,
                                void* stream) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  if (layer < 0 || layer >= c->cfg.n_layers)
    return fail(c, MOESHARD_ERR_BOUNDS, "layer=%d not in [0, %d)", layer, c->cfg.n_layers);
  if (!w_in_shard || !w_out_shard || !storage)
    return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL shard or storage pointer");
  if (reinterpret_cast<uintptr_t>(storage) & 255)
    return fail(c, MOESHARD_ERR_INVALID_ARG, "weight storage must be 256-B aligned");
  const size_t per = static_cast<size_t>(c->Et) * c->h * c->F * c->elt;   // Et experts' slices
  if (bytes < 2 * per)
    return fail(c, MOESHARD_ERR_SHAPE, "weight storage has %zu bytes, needs %zu", bytes, 2 * per);
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LayerW& lw = c->layers[layer];
  lw.wt_in = storage;
  lw.wt_out = static_cast<char*>(storage) + per;
  if (c->use_tc) {
    // swizzled contiguous 128 x 64 tiles of W_i^T [E][F][h] and W_o^T [E][h][F]
    launch_pack_a_tiles(w_in_shard, lw.wt_in, c->Et, c->h, c->F, s);
    launch_pack_a_tiles(w_out_shard, lw.wt_out, c->Et, c->F, c->h, s);
    const uint64_t rows = static_cast<uint64_t>(c->Et) * c->F * c->h / 64;
    if (!make_tmap(&lw.tm_in, lw.wt_in, 64, rows, 128, false) ||
        !make_tmap(&lw.tm_out, lw.wt_out, 64, rows, 128, false))
      return fail(c, MOESHARD_ERR_CUDA, "cuTensorMapEncodeTiled failed for weight tiles");
  } else {
    // W_i^r [E][h][F] -> [E][F][h];  W_o^r [E][F][h] -> [E][h][F]
    launch_transpose(c->cfg.dtype, w_in_shard, lw.wt_in, c->Et, c->h, c->F, s);
    launch_transpose(c->cfg.dtype, w_out_shard, lw.wt_out, c->Et, c->F, c->h, s);
  }
  CUDA_TRY(c, cudaGetLastError());
  lw.loaded = true;
  return MOESHARD_OK;
}

int moeshard_forward(moeshard_ctx* c, int layer, const void* hidden, int n, const void* router_w,
                     void* hidden_out, const int32_t* forced, void* stream) {
  return moeshard_forward_stages(c, layer, hidden, n, router_w, hidden_out, forced,
                                 MOESHARD_STAGE_ALL, stream);
}

int moeshard_forward_stages(moeshard_ctx* c, int layer, const void* hidden, int n,
                            const void* router_w, void* hidden_out, const int32_t* forced,
                            int stages, void* stream) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  if (stages <= 0 || (stages & ~MOESHARD_STAGE_ALL))
    return fail(c, MOESHARD_ERR_INVALID_ARG, "stages=%d is not a non-empty MOESHARD_STAGE_* mask",
                stages);
  if (c->p2p && !c->connected)
    return fail(c, MOESHARD_ERR_PROTOCOL, "MOESHARD_FLAG_P2P: moeshard_p2p_connect was not called");
  if (layer < 0 || layer >= c->cfg.n_layers)
    return fail(c, MOESHARD_ERR_BOUNDS, "layer=%d not in [0, %d)", layer, c->cfg.n_layers);
  if (!c->layers[layer].loaded)
    return fail(c, MOESHARD_ERR_NOT_LOADED, "layer %d has no expert shards loaded", layer);
  if (n < 0 || n > c->cfg.max_tokens_per_rank)
    return fail(c, MOESHARD_ERR_BOUNDS, "n_local=%d not in [0, max_tokens_per_rank=%d]", n,
                c->cfg.max_tokens_per_rank);
  if (n > 0 && (!hidden || !router_w || !hidden_out))
    return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL hidden/router_w/hidden_out");
  CUDA_TRY(c, cudaSetDevice(c->device));   // kernel attributes and launches target this device
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LayerW& lw = c->layers[layer];
  const int h = c->h, F = c->F, E = c->E, Et = c->Et;   // Et: experts computed here
  if (!(stages & MOESHARD_STAGE_ROUTE) && n != c->last_n)
    return fail(c, MOESHARD_ERR_PROTOCOL, "n_local=%d differs from the ROUTE stage's %d", n,
                c->last_n);
  c->last_n = n;
  // MOESHARD_FLAG_UNEVEN_TOKENS: ranks may pass different n_local (the paper's Step 2
  // exchanges the per-GPU sizes): every rank's tokens occupy a slot of
  // ns = max_tokens_per_rank rows, the unused tail of a slot is marked invalid (expert -1)
  // and routes nowhere. Without the flag every rank passes the same n and ns = n.
  // The EP baseline always uses slots (a host receives rows of every rank's slot).
  const bool uneven = c->coll && (c->cfg.flags & (MOESHARD_FLAG_UNEVEN_TOKENS | MOESHARD_FLAG_EXPERT_PARALLEL));
  if (n == 0 && !uneven) return MOESHARD_OK;
  const int ns = uneven ? c->cfg.max_tokens_per_rank : n;   // rows per rank slot
  const bool st_route = stages & MOESHARD_STAGE_ROUTE, st_compute = stages & MOESHARD_STAGE_COMPUTE,
             st_reduce = stages & MOESHARD_STAGE_REDUCE;
  const ncclDataType_t ndt = c->cfg.dtype == MOESHARD_BF16 ? ncclBfloat16 : ncclFloat32;
  int32_t* err_flag = c->tb.stats + 3;

  c->mark(0, s);
  // Step 3 (tokens) forked ahead of Step 1: the AllGather of x overlaps the router
  const bool ag_x_side = st_route && c->coll && !c->p2p && c->overlap_ag;
  if (ag_x_side) {
    CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
    CUDA_TRY(c, cudaStreamWaitEvent(c->s_x, c->ev_fork, 0));
    CUDA_TRY_RET(c, allgather_tokens(c, hidden, n, ns, uneven, ndt, c->s_x));
    CUDA_TRY(c, cudaEventRecord(c->ev_join, c->s_x));
  }
  // Step 1: route local tokens
  // (EP: the router's output stays in the workspace; the dispatch writes the hosts' copies)
  RouteRec* my_route =
      c->ep ? c->ep_route : c->route + (c->coll ? static_cast<size_t>(c->rank) * ns * c->K : 0);
  // tokens per hist-block = tokens per router CTA (128 for the tcgen05 router, 64 for SIMT)
  const int HB = c->use_tc ? kRouterTok : 64;
  const int nbr_own = (n + HB - 1) / HB;                // hist-blocks this rank's router fills
  const int nbr = (ns + HB - 1) / HB;                   // hist-blocks per rank slot
  const int NB = (c->coll ? c->world : 1) * nbr;
  int32_t* my_hist = c->ep ? c->ep_hist
                           : c->block_hist + (c->coll ? static_cast<size_t>(c->rank) * nbr * E : 0);
  const uint32_t kLaunchModes = MOESHARD_FLAG_LAUNCH_PER_EXPERT | MOESHARD_FLAG_LAUNCH_PER_SOURCE;
  const bool fused = c->use_tc && !(c->cfg.flags & (MOESHARD_FLAG_UNFUSED_GEMM | kLaunchModes)) &&
                     F % kTcFeatTile == 0 && h % kTcFeatTile == 0;   // odd tile counts: see FFN kernel
  if (!st_route || n == 0) {
    // (routing ran in an earlier call, or this rank has no tokens this time)
  } else if (c->use_tc) {
    CUtensorMap tm_x, tm_w;
    const bool mn = (E % 8) == 0;
    if (!make_tmap(&tm_x, hidden, h, n, HB) ||
        (mn && !make_tmap(&tm_w, router_w, E, h, 64)))
      return fail(c, MOESHARD_ERR_CUDA, "cuTensorMapEncodeTiled failed for hidden/router_w");
    CUDA_TRY(c, launch_router_tc(tm_x, mn ? tm_w : c->tm_wt_r, mn, router_w, c->wt_r, n, h, E,
                                 c->EP, forced, my_route, my_hist, err_flag, s, c->K, c->num_sms));
    c->launches += mn ? 1 : 2;
  } else {
    launch_router(c->cfg.dtype, hidden, n, h, router_w, E, forced, my_route, my_hist, err_flag, s);
    c->launches += 1;
  }
  if (st_route && uneven && !c->ep) {
    // the rest of this rank's slot: no token (expert -1), empty hist-blocks
    if (ns > n)
      CUDA_TRY(c, cudaMemsetAsync(my_route + n, 0xFF, static_cast<size_t>(ns - n) * sizeof(RouteRec), s));
    if (nbr > nbr_own)
      CUDA_TRY(c, cudaMemsetAsync(my_hist + static_cast<size_t>(nbr_own) * E, 0,
                                  static_cast<size_t>(nbr - nbr_own) * E * 4, s));
  }
  c->mark(1, s);
  // Steps 2+3: metadata + token scatter (replicate all tokens on all GPUs)
  const void* x_all = c->coll ? c->x_all : hidden;
  if (st_route && c->ep) {
    // EP all-to-all scatter: admitted rows only to their expert's host (capacity, first come)
    const int cap = static_cast<int>(std::ceil(static_cast<double>(c->ep_cf) * n / E));
    CUDA_TRY(c, launch_ep_dispatch(c->pa, hidden, n, h * c->elt / 16, c->ep_route, c->ep_hist, E, Et,
                                   cap, c->ep_owner, s));
    c->launches += 1;
  } else if (st_route && c->p2p) {
    // Step 3 over peer memory: push this rank's tokens / records / histograms to every rank
    CUDA_TRY(c, launch_p2p_push(c->pa, hidden, n, ns, h * c->elt / 16, nbr, E, c->num_sms, s));
    c->launches += 2;   // push + publish
  } else if (st_route && c->coll) {
    if (!ag_x_side) CUDA_TRY_RET(c, allgather_tokens(c, hidden, n, ns, uneven, ndt, s));
    NCCL_TRY(c, nccl().GroupStart());
    NCCL_TRY(c, nccl().AllGather(my_route, c->route, static_cast<size_t>(ns) * 2 * c->K, ncclInt32,
                                 c->comm, s));
    NCCL_TRY(c, nccl().AllGather(my_hist, c->block_hist, static_cast<size_t>(nbr) * E, ncclInt32,
                                 c->comm, s));
    NCCL_TRY(c, nccl().GroupEnd());
    if (ag_x_side) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_join, 0));
  }
  c->mark(2, s);
  if (st_compute) {
    if (c->p2p) {   // every rank's Step-3 data has landed here (bounded wait)
      CUDA_TRY(c, launch_p2p_wait_tokens(c->pa, err_flag, s));
      c->launches += 1;
    }
    // Step 2 grouping + Sec. 3.3 per-expert concatenation across GPUs
    launch_group_blocks(c->block_hist, NB, Et, c->block_base, c->block_tot, c->tb,
                        F / kTcFeatTile, h / kTcFeatTile, c->route, x_all, ns, nbr, HB,
                        h * c->elt, c->perm, c->x_perm, s, c->K);
    c->launches += 2;
    c->mark(3, s);
    // Step 4: expert computation, one grouped product per projection
    void* P = c->coll && !c->p2p ? c->partial : hidden_out;
    // opt-in for narrow shards (F <= 512, e.g. G = 8): both products per expert chunk in one
    // cluster, H on chip (expert_mlp.cu)
    const bool mlp = fused && (c->cfg.flags & MOESHARD_FLAG_ONCHIP_H) &&
                     expert_mlp_supported(h, F, Et);
    if (mlp) {
      TcParams dn{F, h / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_out), Et, c->tb,
                  static_cast<__nv_bfloat16*>(P), h, c->tb.perm_pad, c->route};
      if (c->p2p) set_p2p_out(c, dn, ns);
      CUDA_TRY(c, launch_tc_expert_mlp(c->tm_xperm128, lw.tm_in, lw.tm_out, dn, h, F, c->num_sms, s));
      c->mark(4, s);
      c->launches += 1;
      if (c->p2p) {
        CUDA_TRY(c, launch_p2p_signal_partials(c->pa, s));
        c->launches += 1;
      }
    } else if (fused) {
      // paired token chunks when the assignments per expert average >= 256 (most experts
      // then get two chunks of ~130-160 tokens) and the shard is F >= 4096 wide (C5 at G = 1:
      // -9 %; at F = 2048-3072, top-2 C2/C3 measured +4 %; gemm_tc.cu kPair)
      const long long n_assign = static_cast<long long>(c->coll ? c->world : 1) * ns * c->K;
#ifndef MOESHARD_PAIR_MIN_F
#define MOESHARD_PAIR_MIN_F 4096
#endif
      const bool pair_chunks = n_assign >= 256LL * Et && F >= MOESHARD_PAIR_MIN_F;
      TcParams up{h, F / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_in), Et, c->tb,
                  static_cast<__nv_bfloat16*>(c->H), F, nullptr, nullptr};
      // top_k > 1: each (token, expert) assignment's row goes to y_assign, summed per token below
      TcParams dn{F, h / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_out), Et, c->tb,
                  static_cast<__nv_bfloat16*>(c->K > 1 ? c->y_assign : P), h, c->tb.perm_pad,
                  c->route};
      dn.gate_pad = c->tb.gate_pad;
      if (c->p2p) set_p2p_out(c, dn, ns);
      CUDA_TRY(c, launch_tc_moe_ffn(lw.tm_in, c->tm_xperm16, lw.tm_out, c->tm_H16, up, dn,
                                    c->tb.done, (c->cfg.flags & MOESHARD_FLAG_DYNAMIC_SCHED) != 0,
                                    /*early_tables=*/n > 0 && !c->ep,
                                    /*pair_chunks=*/pair_chunks, c->num_sms, s));
      if (c->K > 1) {   // y[t] = sum_j y_assign[K t + j] (R21); rank-major rows of all ranks
        launch_combine_assignments(c->y_assign, P, (c->coll ? c->world : 1) * ns, h * c->elt, c->K,
                                   c->num_sms, s);
        c->launches += 1;
      }
      c->mark(4, s);
      c->launches += 1;
      if (c->p2p) {
        CUDA_TRY(c, launch_p2p_signal_partials(c->pa, s));
        c->launches += 1;
      }
    } else if (c->use_tc && (c->cfg.flags & kLaunchModes)) {
      // Sec. 3.3 ablation: the launch fusion undone. One up + one down
      // launch per expert (2 Et launches: the paper's per-expert mode after its first
      // optimisation) or per (source rank, expert) (2 Et G launches: no optimisation). Each
      // launch reads the device tables and exits at once when its token range is empty, so
      // the host never synchronises (graph-capturable); the arithmetic is the grouped one.
      const bool per_src = (c->cfg.flags & MOESHARD_FLAG_LAUNCH_PER_SOURCE) != 0;
      const int n_src = c->coll ? c->world : 1;
      TcParams up{h, F / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_in), Et, c->tb,
                  static_cast<__nv_bfloat16*>(c->H), F, nullptr, nullptr};
      TcParams dn{F, h / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_out), Et, c->tb,
                  static_cast<__nv_bfloat16*>(P), h, c->tb.perm_pad, c->route};
      for (TcParams* q : {&up, &dn}) {
        q->block_base = c->block_base;
        q->nbr = nbr;
        q->n_src = n_src;
      }
      if (c->p2p) set_p2p_out(c, dn, ns);
      for (int e = 0; e < Et; ++e)
        for (int g = 0; g < (per_src ? n_src : 1); ++g) {
          up.only_e = dn.only_e = e;
          up.only_g = dn.only_g = per_src ? g : -1;
          CUDA_TRY(c, launch_tc_gemm(false, lw.tm_in, c->tm_xperm, c->tm_xperm16, up, c->num_sms, s));
          CUDA_TRY(c, launch_tc_gemm(true, lw.tm_out, c->tm_H, c->tm_H16, dn, c->num_sms, s));
          c->launches += 2;
        }
      c->mark(4, s);
      if (c->p2p) {
        CUDA_TRY(c, launch_p2p_signal_partials(c->pa, s));
        c->launches += 1;
      }
    } else if (c->use_tc) {
      TcParams up{h, F / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_in), Et, c->tb,
                  static_cast<__nv_bfloat16*>(c->H), F, nullptr, nullptr};
      CUDA_TRY(c, launch_tc_gemm(false, lw.tm_in, c->tm_xperm, c->tm_xperm16, up, c->num_sms, s));
      c->mark(4, s);
      TcParams dn{F, h / kTcFeatTile, static_cast<const __nv_bfloat16*>(lw.wt_out), Et, c->tb,
                  static_cast<__nv_bfloat16*>(P), h, c->tb.perm_pad, c->route};
      CUDA_TRY(c, launch_tc_gemm(true, lw.tm_out, c->tm_H, c->tm_H16, dn, c->num_sms, s));
      c->launches += 2;
    } else {
      launch_simt_up(c->cfg.dtype, c->x_perm, lw.wt_in, h, F, Et, c->tb, c->H, c->num_sms, s);
      c->mark(4, s);
      launch_simt_down(c->cfg.dtype, c->H, lw.wt_out, F, h, Et, c->tb, c->tb.perm_pad, c->route, P,
                       c->num_sms, s);
      c->launches += 2;
    }
    CUDA_TRY(c, cudaGetLastError());
  }
  c->mark(5, s);
  // Step 5: gather partial outputs to their owner and sum (aggregateTokens)
  if (st_reduce && c->ep) {   // EP all-to-all gather: each token's row from its host
    CUDA_TRY(c, launch_ep_combine(c->pa, n, h * c->elt / 16, c->ep_owner, hidden_out, err_flag,
                                  c->num_sms, s));
    c->launches += 1;
  } else if (st_reduce && c->p2p) {
    CUDA_TRY(c, launch_p2p_reduce(c->pa, n, h * c->elt / 16, hidden_out, err_flag, c->num_sms, s));
    c->launches += 2;   // wait_partials + reduce
  } else if (st_reduce && c->coll && !uneven) {
    NCCL_TRY(c, nccl().ReduceScatter(c->partial, hidden_out, static_cast<size_t>(n) * h, ndt,
                                     ncclSum, c->comm, s));
  } else if (st_reduce && c->coll) {
    // whole slots, then this rank's n rows (x_all's slot is free once the FFN has run)
    char* slot = static_cast<char*>(c->x_all) + static_cast<size_t>(c->rank) * ns * h * c->elt;
    NCCL_TRY(c, nccl().ReduceScatter(c->partial, slot, static_cast<size_t>(ns) * h, ndt, ncclSum,
                                     c->comm, s));
    if (n > 0)
      CUDA_TRY(c, cudaMemcpyAsync(hidden_out, slot, static_cast<size_t>(n) * h * c->elt,
                                  cudaMemcpyDeviceToDevice, s));
  }
  c->mark(6, s);
  if (c->prof) c->prof_count++;
  return MOESHARD_OK;
}

int moeshard_p2p_region(moeshard_ctx* c, void** dev_ptr, size_t* bytes) {
  if (!c || !dev_ptr) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL ctx or dev_ptr");
  if (!c->p2p) return fail(c, MOESHARD_ERR_CONFIG, "context was not created with MOESHARD_FLAG_P2P");
  *dev_ptr = c->region;
  if (bytes) *bytes = c->PL.total;
  return MOESHARD_OK;
}

int moeshard_p2p_export(moeshard_ctx* c, uint8_t handle[MOESHARD_P2P_HANDLE_BYTES]) {
  if (!c || !handle) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL ctx or handle");
  if (!c->p2p) return fail(c, MOESHARD_ERR_CONFIG, "context was not created with MOESHARD_FLAG_P2P");
  static_assert(sizeof(cudaIpcMemHandle_t) == MOESHARD_P2P_HANDLE_BYTES, "IPC handle size");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t hd;
  CUDA_TRY(c, cudaIpcGetMemHandle(&hd, c->region));
  memcpy(handle, &hd, sizeof(hd));
  return MOESHARD_OK;
}

int moeshard_p2p_open(moeshard_ctx* c, const uint8_t handle[MOESHARD_P2P_HANDLE_BYTES],
                      void** dev_ptr) {
  if (!c || !handle || !dev_ptr) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  void* p = nullptr;
  CUDA_TRY(c, cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  c->ipc_opened.push_back(p);
  *dev_ptr = p;
  return MOESHARD_OK;
}

int moeshard_p2p_connect(moeshard_ctx* c, void* const* regions) {
  if (!c || !regions) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL ctx or regions");
  if (!c->p2p) return fail(c, MOESHARD_ERR_CONFIG, "context was not created with MOESHARD_FLAG_P2P");
  if (regions[c->rank] != c->region)
    return fail(c, MOESHARD_ERR_PROTOCOL, "regions[rank=%d] is not this context's own region",
                c->rank);
  for (int g = 0; g < c->world; ++g) {
    if (!regions[g]) return fail(c, MOESHARD_ERR_INVALID_ARG, "regions[%d] is NULL", g);
    c->pa.peers[g] = static_cast<char*>(regions[g]);
  }
  c->connected = true;
  return MOESHARD_OK;
}

int moeshard_get_routing(moeshard_ctx* c, int32_t* expert_all, float* gate_all, int32_t* counts,
                         int32_t* offsets, int32_t* perm, void* stream) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool uneven = c->coll && (c->cfg.flags & (MOESHARD_FLAG_UNEVEN_TOKENS | MOESHARD_FLAG_EXPERT_PARALLEL));
  const size_t N = static_cast<size_t>(c->coll ? c->world : 1) *
                   (uneven ? c->cfg.max_tokens_per_rank : c->last_n) * c->K;   // assignments
  if (N > 0) {
    if (expert_all)
      CUDA_TRY(c, cudaMemcpy2DAsync(expert_all, 4, &c->route[0].expert, sizeof(RouteRec), 4, N,
                                    cudaMemcpyDeviceToDevice, s));
    if (gate_all)
      CUDA_TRY(c, cudaMemcpy2DAsync(gate_all, 4, &c->route[0].gate, sizeof(RouteRec), 4, N,
                                    cudaMemcpyDeviceToDevice, s));
    if (perm) CUDA_TRY(c, cudaMemcpyAsync(perm, c->perm, N * 4, cudaMemcpyDeviceToDevice, s));
  }
  if (counts)
    CUDA_TRY(c, cudaMemcpyAsync(counts, c->tb.counts, c->Et * 4, cudaMemcpyDeviceToDevice, s));
  if (offsets)
    CUDA_TRY(c, cudaMemcpyAsync(offsets, c->tb.offsets, (c->Et + 1) * 4, cudaMemcpyDeviceToDevice,
                                s));
  return MOESHARD_OK;
}

int moeshard_get_ep_admission(moeshard_ctx* c, int32_t* owner, int32_t* expert, float* gate,
                              int32_t* received, void* stream) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  if (!c->ep) return fail(c, MOESHARD_ERR_CONFIG, "context was not created with MOESHARD_FLAG_EXPERT_PARALLEL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = static_cast<size_t>(c->last_n);
  if (n > 0) {
    if (owner) CUDA_TRY(c, cudaMemcpyAsync(owner, c->ep_owner, n * 4, cudaMemcpyDeviceToDevice, s));
    if (expert)
      CUDA_TRY(c, cudaMemcpy2DAsync(expert, 4, &c->ep_route[0].expert, sizeof(RouteRec), 4, n,
                                    cudaMemcpyDeviceToDevice, s));
    if (gate)
      CUDA_TRY(c, cudaMemcpy2DAsync(gate, 4, &c->ep_route[0].gate, sizeof(RouteRec), 4, n,
                                    cudaMemcpyDeviceToDevice, s));
  }
  if (received)
    CUDA_TRY(c, cudaMemcpyAsync(received, c->tb.counts, c->Et * 4, cudaMemcpyDeviceToDevice, s));
  return MOESHARD_OK;
}

int moeshard_get_stats(moeshard_ctx* c, moeshard_stats* out, void* stream) {
  if (!c || !out) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL ctx or out");
  int32_t st[8];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(c, cudaMemcpyAsync(st, c->tb.stats, sizeof(st), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  out->n_tokens_global = static_cast<int64_t>(c->coll ? c->world : 1) * c->last_n;
  out->tiles_up = c->last_n ? st[0] : 0;
  out->tiles_down = c->last_n ? st[1] : 0;
  out->rows_executed_up = c->last_n ? st[2] : 0;
  out->kernel_launches = c->launches;
  return MOESHARD_OK;
}

int moeshard_profile(moeshard_ctx* c, int enable) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (enable && c->ev.empty()) {
    c->ev.resize(moeshard_ctx::kRing * moeshard_ctx::kEv);
    for (auto& e : c->ev) CUDA_TRY(c, cudaEventCreate(&e));
  }
  c->prof = enable != 0;
  c->prof_count = 0;
  return MOESHARD_OK;
}

int moeshard_get_phase_ms(moeshard_ctx* c, float* out, int n, int* count) {
  if (!c || !out || n < 0) return fail(c, MOESHARD_ERR_INVALID_ARG, "NULL ctx/out or n < 0");
  const int kEv = moeshard_ctx::kEv;
  for (int i = 0; i < n; ++i) out[i] = 0.f;
  const int m = std::min(c->prof_count, moeshard_ctx::kRing);
  if (count) *count = m;
  if (m == 0) return MOESHARD_OK;
  CUDA_TRY(c, cudaEventSynchronize(c->ev[((c->prof_count - 1) % moeshard_ctx::kRing) * kEv + kEv - 1]));
  for (int f = 0; f < m; ++f)
    for (int p = 0; p + 1 < kEv && p < n; ++p) {
      float ms = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev[f * kEv + p], c->ev[f * kEv + p + 1]));
      out[p] += ms;
    }
  return MOESHARD_OK;
}

int moeshard_check(moeshard_ctx* c, void* stream) {
  if (!c) return fail(nullptr, MOESHARD_ERR_INVALID_ARG, "ctx is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(c, cudaStreamSynchronize(s));
  CUDA_TRY(c, cudaGetLastError());
  int32_t flag = 0;
  CUDA_TRY(c, cudaMemcpy(&flag, c->tb.stats + 3, 4, cudaMemcpyDeviceToHost));
  if (c->comm) {
    ncclResult_t ar = ncclSuccess;
    NCCL_TRY(c, nccl().CommGetAsyncError(c->comm, &ar));
    if (ar != ncclSuccess)
      return fail(c, MOESHARD_ERR_NCCL, "NCCL async error: %s", nccl().GetErrorString(ar));
  }
  if (flag) {
    cudaMemset(c->tb.stats + 3, 0, 4);
    if (flag & 8)
      return fail(c, MOESHARD_ERR_CUDA,
                  "FFN: a down-projection unit waited too long for its H tiles (the kernel's "
                  "clusters were not all resident - another kernel held SMs?)");
    if (flag & 4)
      return fail(c, MOESHARD_ERR_PROTOCOL,
                  "MOESHARD_FLAG_P2P: a peer's tokens or partial outputs never arrived (wait timed "
                  "out; did every rank call moeshard_forward?)");
    return fail(c, MOESHARD_ERR_BOUNDS, "forced_expert contained ids outside [0, %d)", c->E);
  }
  return MOESHARD_OK;
}

int moeshard_destroy(moeshard_ctx* c) {
  if (!c) return MOESHARD_OK;
  if (c->comm_x && nccl().ok) nccl().CommDestroy(c->comm_x);
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  cudaSetDevice(c->device);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->region) cudaFree(c->region);
  for (auto& e : c->ev) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s_x) cudaStreamDestroy(c->s_x);
  delete c;
  return MOESHARD_OK;
}

}  // extern "C"
