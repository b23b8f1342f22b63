// gemm_simt.cu - CUDA-core (FFMA) grouped GEMMs over all experts' shards in
// one launch per projection (Sec. 3.3 fusion).
//
// Used for the fp32 validation mode (BASELINE.json: max-abs-rel <= 1e-4,
// which plain TF32 tensor-core math cannot meet; R16) and, behind
// MOESHARD_FLAG_SIMT_GEMM, as a bf16 ablation of the tcgen05 path.
//
//   up:   H[j, f]          = relu( sum_k Xp[j, k] * WiT[e][f][k] )        (Step 4, 1st product)
//   down: out[perm[j], c]  = gate[perm[j]] * sum_f H[j, f] * WoT[e][c][f] (2nd product, gate,
//                                                                         un-permute scatter)
// j runs over expert e's segment [pos[e], pos[e] + counts[e]) of the
// expert-contiguous (32-row padded) internal token order; perm = perm_pad.
// Tiles: 64 tokens x 64 outputs x 32 K, 256 threads each owning a 4x4 fp32
// accumulator block; persistent
// grid-stride loop over (expert, token-chunk, output-tile) units.
#include "common.cuh"

namespace moeshard {
namespace {

constexpr int BM = kSimtTokTile;   // tokens
constexpr int BN = kSimtFeatTile;  // outputs
constexpr int BK = 32;

template <typename T> __device__ __forceinline__ void load8(const T* p, float* v);
template <> __device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(b[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <> __device__ __forceinline__ void load8<float>(const float* p, float* v) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <typename T, bool kDown>
__global__ void __launch_bounds__(256) simt_grouped_gemm(const T* __restrict__ A,   // [N][K]
                                                         const T* __restrict__ Wt,  // [E][NOUT][K]
                                                         int K, int NOUT, int E, Tables tb,
                                                         const int32_t* __restrict__ perm,
                                                         const RouteRec* __restrict__ route,
                                                         T* __restrict__ out) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  __shared__ int32_t s_pref[kMaxExperts + 1];
  __shared__ int32_t s_off[kMaxExperts + 1];   // internal (padded) segment starts
  __shared__ int32_t s_cnt[kMaxExperts];
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    s_pref[e] = tb.simt_chunk_pref[e];
    s_off[e] = tb.pos[e];
    if (e < E) s_cnt[e] = tb.counts[e];
  }
  __syncthreads();
  const int n_nt = NOUT / BN;
  const int total = s_pref[E] * n_nt;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int lr = tid >> 2, lc = (tid & 3) * 8;  // tile-load coordinates

  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    // decode unit -> (expert, chunk, output tile); units are chunk-major per expert
    const int q = u / n_nt;
    int lo = 0, hi = E;  // find e: s_pref[e] <= q < s_pref[e+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pref[mid] <= q) lo = mid; else hi = mid;
    }
    const int e = lo;
    const int c = q - s_pref[e];
    const int nt = u - q * n_nt;
    const int row0 = s_off[e] + c * BM;
    const int rows = min(BM, s_cnt[e] - c * BM);
    const int n0 = nt * BN;
    const T* Wte = Wt + (size_t)e * NOUT * K;

    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < K; k0 += BK) {
      float va[8], vb[8];
      if (lr < rows) load8<T>(A + (size_t)(row0 + lr) * K + k0 + lc, va);
      else {
#pragma unroll
        for (int i = 0; i < 8; ++i) va[i] = 0.f;
      }
      load8<T>(Wte + (size_t)(n0 + lr) * K + k0 + lc, vb);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        As[lc + i][lr] = va[i];
        Bs[lc + i][lr] = vb[i];
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], bb[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      if (r >= rows) continue;
      const int j = row0 + r;
      if (!kDown) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          out[(size_t)j * NOUT + n0 + tx * 4 + jj] = from_f32<T>(fmaxf(acc[i][jj], 0.f));
      } else {
        const int t = perm[j];
        const float g = route[t].gate;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          out[(size_t)t * NOUT + n0 + tx * 4 + jj] = from_f32<T>(g * acc[i][jj]);
      }
    }
  }
}

template <typename T, bool kDown>
void launch(const void* A, const void* Wt, int K, int NOUT, int E, Tables tb, const int32_t* perm,
            const RouteRec* route, void* out, int num_sms, cudaStream_t s) {
  simt_grouped_gemm<T, kDown><<<num_sms * 4, 256, 0, s>>>(
      static_cast<const T*>(A), static_cast<const T*>(Wt), K, NOUT, E, tb, perm, route,
      static_cast<T*>(out));
}

}  // namespace

void launch_simt_up(int dtype, const void* x_perm, const void* wt_in, int K, int F, int E, Tables tb,
                    void* H, int num_sms, cudaStream_t s) {
  if (dtype == 0)
    launch<__nv_bfloat16, false>(x_perm, wt_in, K, F, E, tb, nullptr, nullptr, H, num_sms, s);
  else
    launch<float, false>(x_perm, wt_in, K, F, E, tb, nullptr, nullptr, H, num_sms, s);
}

void launch_simt_down(int dtype, const void* H, const void* wt_out, int K, int h, int E, Tables tb,
                      const int32_t* perm, const RouteRec* route, void* out, int num_sms,
                      cudaStream_t s) {
  if (dtype == 0)
    launch<__nv_bfloat16, true>(H, wt_out, K, h, E, tb, perm, route, out, num_sms, s);
  else
    launch<float, true>(H, wt_out, K, h, E, tb, perm, route, out, num_sms, s);
}

}  // namespace moeshard
