// timeline.cuh - measurement-only build (-DMOESHARD_TIMELINE): %globaltimer stamps of
// kernel milestones (slot 2i = earliest, 2i+1 = latest over CTAs) per translation unit,
// read by the exported <tu>_timeline(out, reset). Compiled out of the product library.
#pragma once
#ifdef MOESHARD_TIMELINE
#include <cuda_runtime.h>
static __device__ unsigned long long g_tl[16];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_MIN(i) atomicMin(&g_tl[2 * (i)], tl_now())
#define TL_MAX(i) atomicMax(&g_tl[2 * (i) + 1], tl_now())
#define TL_EXPORT(name)                                                           \
  extern "C" int name(unsigned long long* out, int reset) {                        \
    if (out) cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl));                        \
    if (reset) {                                                                  \
      unsigned long long init[16];                                                \
      for (int i = 0; i < 16; i += 2) { init[i] = ~0ull; init[i + 1] = 0ull; }     \
      cudaMemcpyToSymbol(g_tl, init, sizeof(init));                               \
    }                                                                             \
    return static_cast<int>(cudaDeviceSynchronize());                             \
  }
// per-unit trace of the fused FFN: [cluster < 148][unit slot < 16][8 stamps]
static __device__ unsigned long long g_tr[148 * 16 * 8];
#define TR(cl, k, j)                                              \
  do {                                                            \
    if ((cl) < 148 && (k) < 16) g_tr[((cl) * 16 + (k)) * 8 + (j)] = tl_now(); \
  } while (0)
#define TR_EXPORT(name)                                                          \
  extern "C" int name(unsigned long long* out, int reset) {                       \
    if (out) cudaMemcpyFromSymbol(out, g_tr, sizeof(g_tr));                       \
    if (reset) cudaMemset(reinterpret_cast<void*>(0), 0, 0);                      \
    if (reset) {                                                                 \
      void* p = nullptr;                                                         \
      cudaGetSymbolAddress(&p, g_tr);                                            \
      cudaMemset(p, 0, sizeof(g_tr));                                            \
    }                                                                            \
    return static_cast<int>(cudaDeviceSynchronize());                            \
  }
#else
#define TL_MIN(i)
#define TL_MAX(i)
#define TL_EXPORT(name)
#define TR(cl, k, j)
#define TR_EXPORT(name)
#endif
