// gemm_tc.cuh - host interface of the tcgen05 grouped GEMM (gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace moeshard {

struct TcParams {
  int K;              // reduction length: h (up) or F = d_ff/G (down); multiple of 64
  int n_mt;           // output tiles of 128 features: F/128 (up) or h/128 (down)
  int rows_per_e;     // weight rows per expert in the A tensor map (= n_mt * 128)
  int E;              // experts
  Tables tb;          // device segment tables of the current forward
  __nv_bfloat16* out; // up: H [N][F]; down: out [N or n][h] in global token order
  int ld_out;         // F (up) or h (down)
  const int32_t* perm;     // down: perm[j] = global token id of expert-ordered row j
  const RouteRec* route;   // down: gate per global token
};

// grid = number of persistent CTAs (normally the SM count).
cudaError_t launch_tc_gemm(bool down, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const TcParams& p, int grid, cudaStream_t s);

}  // namespace moeshard
