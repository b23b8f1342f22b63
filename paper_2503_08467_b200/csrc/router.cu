// router.cu - Step 1 token routing (Alg. 1 line "m_expert <- router(x)",
// PAPER.md:187-188, 261-263): logits = x W_r (fp32 accumulation), softmax,
// top-1 argmax with lowest-index tie-break (R4), gate = softmax
// probability of the chosen expert (R2). Optional forced expert ids (the
// paper's replaced router).
//
// Layout: x [n][h] row-major (bf16 or fp32), W_r [h][E] row-major.
// One CTA = 64 tokens x all E experts. 256 threads = 16 token groups (ty) x
// 16 expert lanes (tx); thread (ty, tx) owns tokens ty*4+i and experts
// tx + 16*j (j < EPT). The per-token max / sum-exp reductions over the 16
// expert lanes are xor warp shuffles (the 16 lanes sit in one half-warp).
#include "common.cuh"

namespace moeshard {
namespace {

constexpr int RT_TOK = 64;
constexpr int RT_KC = 32;

template <typename T> struct Load8;
template <> struct Load8<__nv_bfloat16> {
  __device__ static void run(const __nv_bfloat16* p, float* v) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(b[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
};
template <> struct Load8<float> {
  __device__ static void run(const float* p, float* v) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

template <typename T, int EPT>
__global__ void __launch_bounds__(256) router_kernel(const T* __restrict__ x, int n, int h,
                                                     const T* __restrict__ w_r, int E,
                                                     const int32_t* __restrict__ forced,
                                                     RouteRec* __restrict__ out,
                                                     int32_t* __restrict__ err_flag) {
  constexpr int EP = EPT * 16;                 // padded expert count handled by this instantiation
  __shared__ __align__(16) float xs[RT_KC][RT_TOK + 4];
  __shared__ __align__(16) float ws[RT_KC][EP];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int tok0 = blockIdx.x * RT_TOK;

  float acc[4][EPT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < EPT; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < h; k0 += RT_KC) {
    // x tile: 64 tokens x 32 k -> 2048 elements, 8 per thread (one 16/32-B vector)
    {
      const int r = tid >> 2, c = (tid & 3) * 8;
      float v[8];
      if (tok0 + r < n) {
        Load8<T>::run(x + (size_t)(tok0 + r) * h + k0 + c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) xs[c + i][r] = v[i];
    }
    // W_r chunk: 32 rows x E (pad to EP with zeros)
    for (int idx = tid; idx < RT_KC * EP; idx += 256) {
      const int kk = idx / EP, e = idx - kk * EP;
      ws[kk][e] = (e < E) ? to_f32(w_r[(size_t)(k0 + kk) * E + e]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < RT_KC; ++kk) {
      const float4 xv = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
      const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const float w = ws[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(xa[i], w, acc[i][j]);
      }
    }
    __syncthreads();
  }

  // softmax + top-1 per token; reductions over the 16 expert lanes
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = tok0 + ty * 4 + i;
    float best = -INFINITY;
    int best_e = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tx + 16 * j;
      if (e < E && (acc[i][j] > best || (acc[i][j] == best && e < best_e))) {
        best = acc[i][j];
        best_e = e;
      }
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oe = __shfl_xor_sync(0xffffffffu, best_e, off);
      if (ob > best || (ob == best && oe < best_e)) {
        best = ob;
        best_e = oe;
      }
    }
    int sel = best_e;
    bool bad = false;
    if (forced != nullptr && t < n) {
      sel = forced[t];
      if (sel < 0 || sel >= E) {
        bad = true;
        sel = sel < 0 ? 0 : E - 1;
      }
    }
    float sum = 0.f, lsel = 0.f;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tx + 16 * j;
      if (e < E) sum += expf(acc[i][j] - best);
      if (e == sel) lsel = acc[i][j];
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, off);
      lsel += __shfl_xor_sync(0xffffffffu, lsel, off);
    }
    if (tx == 0 && t < n) {
      RouteRec r;
      r.expert = sel;
      r.gate = expf(lsel - best) / sum;
      out[t] = r;
      if (bad) atomicExch(err_flag, 1);
    }
  }
}

template <typename T>
void launch_router_t(const T* x, int n, int h, const T* w_r, int E, const int32_t* forced,
                     RouteRec* out, int32_t* err, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid(ceil_div(n, RT_TOK));
  if (E <= 16) router_kernel<T, 1><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, err);
  else if (E <= 32) router_kernel<T, 2><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, err);
  else if (E <= 64) router_kernel<T, 4><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, err);
  else if (E <= 128) router_kernel<T, 8><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, err);
  else router_kernel<T, 16><<<grid, 256, 0, s>>>(x, n, h, w_r, E, forced, out, err);
}

}  // namespace

void launch_router(int dtype, const void* x, int n, int h, const void* w_r, int E,
                   const int32_t* forced, RouteRec* out, int32_t* err_flag, cudaStream_t s) {
  if (dtype == 0)
    launch_router_t(static_cast<const __nv_bfloat16*>(x), n, h,
                    static_cast<const __nv_bfloat16*>(w_r), E, forced, out, err_flag, s);
  else
    launch_router_t(static_cast<const float*>(x), n, h, static_cast<const float*>(w_r), E, forced,
                    out, err_flag, s);
}

}  // namespace moeshard
