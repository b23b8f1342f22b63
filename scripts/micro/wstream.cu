// Weight-stream probe: how fast can one persistent CTA per SM stream packed 16 KB weight
// tiles from HBM into a shared-memory ring, as a function of the access pattern, the copy
// engine (1-D bulk vs 2-D tensor TMA), the L2 eviction hint and the ring depth?
// Question (VERDICT r01 item 5 / DESIGN §12): the fused FFN moves its weights at ~5.4 TB/s
// against ~7 TB/s for a pure read stream - is the weight access pattern part of the gap?
//   pattern 0 "ffn":   CTA pair q streams units u = q, q + 74, ...; a unit is 12 tiles of
//                      16 KB per CTA, CTA r of the pair reads the r-th 192 KB half (the
//                      [e][mt][kb] packing, pair-tiles adjacent)
//   pattern 1 "inter": at step i CTA c reads tile c + i * grid (globally sequential)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wstream wstream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int TILE = 16384;

__global__ void __launch_bounds__(128) stream(const __grid_constant__ CUtensorMap tm,
                                              const uint8_t* __restrict__ buf, long long ntiles,
                                              int S, int pattern, int tensor, int hint,
                                              long long per_cta_tiles, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smx[];
  __shared__ uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int cta = blockIdx.x, G = gridDim.x;
  const int pair = cta >> 1, r = cta & 1, npairs = G >> 1;
  auto tile_of = [&](long long i) -> long long {
    if (pattern == 1) return (cta + i * G) % ntiles;
    const long long u = pair + (i / 12) * npairs;   // unit of this pair
    return (u * 24 + r * 12 + (i % 12)) % ntiles;
  };
  uint32_t phase = 0;
  unsigned long long acc = 0;
  for (long long i = 0; i < per_cta_tiles + S; ++i) {
    const int s = static_cast<int>(i % S);
    const uint32_t bar = smem_u32(&full[s]);
    if (i >= S) {
      asm volatile(
          "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(bar),
          "r"(phase));
      acc += smx[s * TILE];
      if (s == S - 1) phase ^= 1;
    }
    if (i < per_cta_tiles) {
      const long long t = tile_of(i);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE) : "memory");
      const uint32_t dst = smem_u32(smx + s * TILE);
      if (tensor) {
        const int row = static_cast<int>(t * 128);
        if (hint)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
                       ::"r"(dst), "l"(&tm), "r"(0), "r"(row), "r"(bar), "l"(pol) : "memory");
        else
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(dst), "l"(&tm), "r"(0), "r"(row), "r"(bar) : "memory");
      } else {
        const uint8_t* src = buf + t * TILE;
        if (hint)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(dst), "l"(src), "r"(TILE), "r"(bar), "l"(pol) : "memory");
        else
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(dst), "l"(src), "r"(TILE), "r"(bar) : "memory");
      }
    }
  }
  sink[cta] = acc;
}

// The same stream with NI issuing warps per CTA (lane 0 of warp w streams tiles w, w + NI, ...
// of the CTA's share through its own S-stage ring): is the ~50 GB/s per SM a per-issuer or a
// per-SM limit?
__global__ void __launch_bounds__(128) stream_multi(const __grid_constant__ CUtensorMap tm,
                                                    long long ntiles, int S, int NI,
                                                    long long per_cta_tiles,
                                                    unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smx[];
  __shared__ uint64_t full[4][16];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= NI) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint8_t* ring = smx + static_cast<size_t>(w) * S * TILE;
  const int cta = blockIdx.x, G = gridDim.x;
  const long long mine = (per_cta_tiles - w + NI - 1) / NI;
  uint32_t phase = 0;
  unsigned long long acc = 0;
  for (long long i = 0; i < mine + S; ++i) {
    const int s = static_cast<int>(i % S);
    const uint32_t bar = smem_u32(&full[w][s]);
    if (i >= S) {
      asm volatile(
          "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(bar),
          "r"(phase));
      acc += ring[s * TILE];
      if (s == S - 1) phase ^= 1;
    }
    if (i < mine) {
      const long long t = (cta + (i * NI + w) * G) % ntiles;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE) : "memory");
      const uint32_t dst = smem_u32(ring + s * TILE);
      const int row = static_cast<int>(t * 128);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
                   ::"r"(dst), "l"(&tm), "r"(0), "r"(row), "r"(bar), "l"(pol) : "memory");
    }
  }
  sink[cta * 4 + w] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 576ull << 20;   // one C2 weight set (2 * 64 * 768 * 3072 * 2 B)
  const int NSETS = 4;                 // rotate: every launch reads a set not in L2
  uint8_t* buf;
  cudaMalloc(&buf, bytes * NSETS);
  cudaMemset(buf, 1, bytes * NSETS);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap tm[NSETS];
  for (int k = 0; k < NSETS; ++k) {
    cuuint64_t dims[2] = {64, bytes / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    enc(&tm[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf + k * bytes, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * TILE + 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long ntiles = bytes / TILE;
  const long long per_cta = ntiles / sms;   // one pass over the set per launch
  for (int persist : {0, 64}) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(persist) << 20);
    for (int pattern : {0, 1})
      for (int tensor : {0, 1})
        for (int hint : {0, 1})
          for (int S : {4, 6, 8, 12}) {
            float best = 1e9f;
            for (int rep = 0; rep < 6; ++rep) {
              const int k = rep % NSETS;
              cudaEventRecord(a);
              stream<<<sms, 128, S * TILE + 1024>>>(tm[k], buf + k * bytes, ntiles, S, pattern, tensor, hint,
                                                    per_cta, sink);
              cudaEventRecord(b);
              cudaEventSynchronize(b);
              float ms = 0;
              cudaEventElapsedTime(&ms, a, b);
              if (rep >= 2 && ms < best) best = ms;
            }
            const double gb = static_cast<double>(per_cta) * sms * TILE / 1e9;
            printf("persist %2d MB  pattern %-5s  %-6s  hint %-11s  stages %2d: %7.1f us  %6.0f GB/s\n", persist,
                   pattern ? "inter" : "ffn", tensor ? "tma2d" : "bulk1d", hint ? "evict_first" : "none", S,
                   best * 1e3, gb / (best * 1e-3));
          }
  }
  // per-SM rate with only part of the GPU streaming (the FFN's tail: do the late clusters
  // speed up when the others have finished?) - fixed tiles per CTA, growing CTA count
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  for (int S : {6, 12})
    for (int grid : {16, 37, 74, 111, sms}) {
      float best = 1e9f;
      for (int rep = 0; rep < 6; ++rep) {
        const int k = rep % NSETS;
        cudaEventRecord(a);
        stream<<<grid, 128, S * TILE + 1024>>>(tm[k], buf + k * bytes, ntiles, S, 1, 1, 1, per_cta, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 2 && ms < best) best = ms;
      }
      const double gb = static_cast<double>(per_cta) * grid * TILE / 1e9;
      printf("partial grid %3d CTAs  stages %2d: %7.1f us  %6.0f GB/s total  %5.1f GB/s per SM\n", grid, S,
             best * 1e3, gb / (best * 1e-3), gb / (best * 1e-3) / grid);
    }
  cudaFuncSetAttribute(stream_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * TILE + 1024);
  for (int NI : {1, 2, 3})
    for (int grid : {16, 74, sms}) {
      const int S = 12 / NI;
      float best = 1e9f;
      for (int rep = 0; rep < 6; ++rep) {
        const int k = rep % NSETS;
        cudaEventRecord(a);
        stream_multi<<<grid, 128, NI * S * TILE + 1024>>>(tm[k], ntiles, S, NI, per_cta, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 2 && ms < best) best = ms;
      }
      const double gb = static_cast<double>(per_cta) * grid * TILE / 1e9;
      printf("issuers %d x %2d stages, grid %3d: %7.1f us  %6.0f GB/s total  %5.1f GB/s per SM\n", NI, S,
             grid, best * 1e3, gb / (best * 1e-3), gb / (best * 1e-3) / grid);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
