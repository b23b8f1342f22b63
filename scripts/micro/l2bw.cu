// Aggregate global -> shared-memory fill bandwidth with 1-D bulk copies (cp.async.bulk,
// the engine the FFN's weight and token loads use), one persistent CTA per SM, an
// S-stage ring of B-byte copies per CTA, data either L2-resident (buffer << L2) or
// streamed from HBM (buffer >> L2). Question: is the FFN bound by HBM or by the
// L2 -> SMEM fill rate?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int S>
__global__ void __launch_bounds__(128) fill(const uint8_t* __restrict__ buf, size_t buf_bytes,
                                            int chunk, long long per_cta, unsigned long long* sink,
                                            int T) {
  extern __shared__ __align__(1024) uint8_t smx[];
  __shared__ uint64_t fullx[4 * S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 4 * S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fullx[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // T issuing threads (lane 0 of warps 0..T-1), each with its own S-stage ring
  if ((tid & 31) != 0 || tid / 32 >= T) return;
  const int me = tid / 32;
  uint64_t* full = fullx + me * S;
  uint8_t* sm = smx + static_cast<size_t>(me) * S * chunk;
  per_cta /= T;
  const size_t nchunks = buf_bytes / chunk;
  // walk chunks (CTA, thread) interleaved, wrapping over the buffer
  size_t idx = static_cast<size_t>(blockIdx.x) * T + me;
  const size_t step = static_cast<size_t>(gridDim.x) * T;
  uint32_t phase = 0;
  unsigned long long acc = 0;
  const long long n = per_cta / chunk;
  for (long long i = 0; i < n + S; ++i) {
    const int s = static_cast<int>(i % S);
    if (i >= S) {   // wait for the copy issued S iterations ago
      const uint32_t bar = smem_u32(&full[s]);
      asm volatile(
          "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(bar),
          "r"(phase));
      acc += sm[s * chunk];
      if (s == S - 1) phase ^= 1;
    }
    if (i < n) {
      const uint32_t bar = smem_u32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk) : "memory");
      const uint8_t* src = buf + (idx % nchunks) * chunk;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sm + s * chunk)),
                   "l"(src), "r"(chunk), "r"(bar)
                   : "memory");
      idx += step;
    }
  }
  sink[blockIdx.x * 4 + me] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 4ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(fill<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const long long per_cta = 32ll << 20;
  struct Cfg { size_t bytes; int chunk, T, grid; };
  const Cfg cfgs[] = {
      {48u << 20, 16384, 1, sms}, {48u << 20, 16384, 2, sms}, {48u << 20, 16384, 3, sms},
      {48u << 20, 8192, 4, sms}, {48u << 20, 32768, 1, sms}, {48u << 20, 4096, 1, sms},
      {48u << 20, 16384, 1, 2 * sms}, {48u << 20, 16384, 2, 2 * sms},
      {size_t(4) << 30, 16384, 1, sms}, {size_t(4) << 30, 16384, 2, sms}, {size_t(4) << 30, 16384, 3, sms},
  };
  for (const Cfg& c : cfgs) {
    const int S = 4;
    if ((size_t)c.T * S * c.chunk > 200 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      fill<4><<<c.grid, 128, c.T * S * c.chunk>>>(buf, c.bytes, c.chunk, per_cta, sink, c.T);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 1)
        printf("buffer %5zu MB chunk %5d B  issuers %d  CTAs %3d (4 stages each): %6.0f GB/s aggregate, %5.1f GB/s per SM\n",
               c.bytes >> 20, c.chunk, c.T, c.grid, c.grid * (double)per_cta / ms / 1e6,
               c.grid * (double)per_cta / ms / 1e6 / sms);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
