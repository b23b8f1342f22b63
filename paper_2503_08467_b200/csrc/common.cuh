// common.cuh - shared device helpers for the moeshard kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "moeshard kernels target sm_100a (B200) only"
#endif

namespace moeshard {

constexpr int kMaxExperts = 256;      // router instantiations cover E <= 256
constexpr int kMaxWorld = 8;          // ranks of one NVLink/NVSwitch box (peer-memory exchange)
#ifndef MOESHARD_TOK_TILE
#define MOESHARD_TOK_TILE 256
#endif
constexpr int kTcTokTile = MOESHARD_TOK_TILE;  // max tokens per tcgen05 tile (UMMA N <= 256)
constexpr int kTcFeatTile = 128;      // weight rows per tcgen05 tile (UMMA M)
constexpr int kSimtTokTile = 64;      // tokens per SIMT tile
constexpr int kSimtFeatTile = 64;     // output features per SIMT tile
constexpr int kSegAlign = 32;         // expert segments in the internal expert-ordered layout
                                      // start on multiples of 32 rows (padding rows unused)

// Routing record of one token, gathered across ranks in one NCCL AllGather
// (Step 2 metadata folded into the token exchange): expert id + gate bits.
struct __align__(8) RouteRec {
  int32_t expert;
  float gate;
};

// Device-side per-forward tables written by the scan kernel.
struct Tables {
  int32_t* counts;         // [E]
  int32_t* offsets;        // [E+1]
  int32_t* tc_chunk_pref;  // [E+1] cumulative tcgen05 token chunks
  int32_t* tc_chunk_size;  // [E]
  int32_t* simt_chunk_pref;  // [E+1]
  int32_t* stats;          // [8]: 0 tiles_up, 1 tiles_down, 2 rows_up, 3 error flag
  int32_t* done;           // [chunks] up-projection tiles completed per token chunk (fused GEMM), zeroed by Step 2
  int32_t* pos;            // [E+1] internal segment starts (exclusive scan of round_up(count, 32))
  int32_t* perm_pad;       // [N + 32E] internal row -> global token id (padding rows: stale)
  float* gate_pad;         // [N + 32E] internal row -> gate of that token (written with perm_pad)
  int32_t* next_unit;      // [1] the fused FFN's dynamic work counter, zeroed by Step 2
};

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int round_up(int a, int b) { return ceil_div(a, b) * b; }

// Token chunking of one expert's segment for the tcgen05 tiles: split n_e
// tokens into ceil(n_e/256) near-equal chunks of a multiple of 32 tokens
// (the CTA-pair kernel splits a chunk's rows evenly over the two SMs in
// 16-row TMA boxes).
__host__ __device__ __forceinline__ void tc_chunking(int n_e, int* n_chunks, int* chunk) {
  if (n_e <= 0) { *n_chunks = 0; *chunk = 0; return; }
  int c0 = ceil_div(n_e, kTcTokTile);
  int cs = round_up(ceil_div(n_e, c0), 32);
  *chunk = cs;
  *n_chunks = ceil_div(n_e, cs);
}

// Kernel attributes (cudaFuncSetAttribute) are per device: a call site records the
// devices it has configured (a process may drive several GPUs; a repeat is harmless).
struct PerDeviceOnce {
  unsigned long long mask = 0ull;
  bool need() const {
    int d = 0;
    cudaGetDevice(&d);
    return d >= 64 || !((__atomic_load_n(&mask, __ATOMIC_ACQUIRE) >> d) & 1ull);
  }
  void done() {
    int d = 0;
    cudaGetDevice(&d);
    if (d < 64) __atomic_fetch_or(&mask, 1ull << d, __ATOMIC_RELEASE);
  }
};

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel in the stream drains; it must call
// griddepcontrol.wait before touching memory the predecessor writes or reads.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace moeshard

// ---------------------------------------------------------------------------
// Host-side launcher declarations (implemented in the .cu files)
// ---------------------------------------------------------------------------
namespace moeshard {

// SIMT router (fp32 mode / ablation): 64-token CTAs; hist_out [ceil(n/64)][E] per-block counts.
void launch_router(int dtype, const void* x, int n, int h, const void* w_r, int E,
                   const int32_t* forced, RouteRec* out, int32_t* hist_out, int32_t* err_flag,
                   cudaStream_t s);

// Step 2 from the routers' per-block histograms: per-expert block scan, then one CTA
// group per hist-block of HB <= 128 tokens (offsets, stable scatter to the compact
// public perm and to the padded internal layout, row gather into X_perm).
// base [NB][E] and tot [E] are workspace outputs of the block scan.
void launch_group_blocks(const int32_t* hist, int NB, int E, int32_t* base, int32_t* tot,
                         Tables tb, int n_mt_up_tc, int n_mt_down_tc, const RouteRec* route,
                         const void* x_all, int n, int nbr, int HB, int row_bytes, int32_t* perm,
                         void* x_perm, cudaStream_t s, int top_k = 1);

void launch_transpose(int dtype, const void* src, void* dst, int batch, int rows, int cols,
                      cudaStream_t s);

// top_k > 1 (bf16): y[t] = sum_{j < K} y_assign[K t + j] over the n_tok tokens (rows of row_bytes).
void launch_combine_assignments(const void* y_assign, void* y, int n_tok, int row_bytes, int K,
                                int num_sms, cudaStream_t s);

// SIMT grouped GEMMs (fp32 validation mode, and bf16 ablation).
void launch_simt_up(int dtype, const void* x_perm, const void* wt_in, int K, int F, int E, Tables tb,
                    void* H, int num_sms, cudaStream_t s);
void launch_simt_down(int dtype, const void* H, const void* wt_out, int K, int h, int E, Tables tb,
                      const int32_t* perm, const RouteRec* route, void* out, int num_sms,
                      cudaStream_t s);

}  // namespace moeshard
