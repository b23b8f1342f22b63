// p2p.cu - the two exchange steps of Alg. 1 done with device-initiated stores
// into peer GPU memory instead of NCCL (MOESHARD_FLAG_P2P; SURVEY.md §8(f)
// NEXT(1)): Step 3 "scatter tokens" and Step 5
// "gather + aggregate".
//
// Every rank owns an exchange region (one cudaMalloc, mapped by every peer
// through CUDA IPC or, for ranks sharing a process, directly):
//   header: [0] epoch (forwards completed), [1] push CTA counter,
//           flags_ag[g] at int 32*(1+g), flags_rs[g] at int 32*(1+G+g)
//   x_all [G*n_max][h] bf16, route [G*n_max] RouteRec, hist [G*nbr_max][E] int32,
//   recv [G][n_max][h] bf16 (slot g = rank g's partial output for this rank's tokens)
// Step 3: push_tokens copies this rank's tokens, route records and block
// histograms into slot r of every region (its own included), then its last CTA
// publishes flags_ag[r] = epoch + 1 everywhere (release, system scope). The
// grouping launch acquires all G flags before it reads x_all.
// Step 5: the fused FFN's down-projection epilogue stores each partial row
// straight into recv[r] of the row's owner (no partial buffer, no separate
// collective); rs_signal then publishes flags_rs[r] = epoch + 1 everywhere and
// reduce_partials sums the G slots in ascending rank order (fp32, so the
// aggregate is bit-reproducible) into hidden_out and advances the epoch.
// Waits are bounded: a peer that never arrives sets error bit 4 (reported by
// moeshard_check) instead of hanging the GPU.
#include "common.cuh"
#include "group.cuh"
#include "p2p.cuh"
#include "ptx.cuh"

#include <algorithm>

namespace moeshard {
namespace {

__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// all G flags >= target, bounded (~2^24 polls of >= 256 ns); on timeout raise error bit 4
__device__ __forceinline__ void wait_flags(const int32_t* flags, int world, int target,
                                           int32_t* err) {
  for (int g = 0; g < world; ++g) {
    const int32_t* f = flags + 32 * g;
    uint32_t it = 0;
    while (ld_acquire_sys(f) < target) {
      if (++it > (1u << 24)) {
        atomicOr(err, 4);
        return;
      }
      __nanosleep(256);
    }
  }
}

// Step 3 push: this rank's n rows / records / block histograms into slot `rank`
// of every peer region. 16-B vectors, grid-stride.
__global__ void __launch_bounds__(256) push_tokens(P2PArgs a, const uint4* __restrict__ x, int n,
                                                   int ns, int row_vecs, int nbr, int E) {
  ptx::griddep_wait();   // x / route / hist come from the router
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  const size_t nx = static_cast<size_t>(n) * row_vecs;    // this rank's rows
  const size_t sx = static_cast<size_t>(ns) * row_vecs;   // slot stride (ns >= n)
  const size_t nrec = static_cast<size_t>(ns);            // the whole slot (tail marked invalid)
  const size_t nh = static_cast<size_t>(nbr) * E;          // int32
  const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const RouteRec* my_route = reinterpret_cast<const RouteRec*>(a.self + a.off_route) + a.rank * nrec;
  const int32_t* my_hist = reinterpret_cast<const int32_t*>(a.self + a.off_hist) + a.rank * nh;
  // token rows: 8 vectors per thread in flight, each read once and stored to every rank
  constexpr int kU = 8;
  for (size_t i0 = tid; i0 < nx; i0 += kU * stride) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * stride < nx) v[u] = __ldg(x + i0 + u * stride);
    for (int g = 0; g < a.world; ++g) {
      uint4* dx = reinterpret_cast<uint4*>(a.peers[g] + a.off_x) + a.rank * sx;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i0 + u * stride < nx) dx[i0 + u * stride] = v[u];
    }
  }
  for (int g = 0; g < a.world; ++g) {
    char* peer = a.peers[g];
    if (g != a.rank) {   // the router already wrote its own slot of route / hist
      RouteRec* dr = reinterpret_cast<RouteRec*>(peer + a.off_route) + a.rank * nrec;
      for (size_t i = tid; i < nrec; i += stride) dr[i] = my_route[i];
      int32_t* dh = reinterpret_cast<int32_t*>(peer + a.off_hist) + a.rank * nh;
      for (size_t i = tid; i < nh; i += stride) dh[i] = my_hist[i];
    }
  }
  (void)epoch;   // the flags are published by push_publish, the next launch
}

// Step 3 publish (one thread, right after push_tokens in stream order): the push grid has
// completed, one system-scope fence makes its stores visible to every peer, then flags_ag
// are released. System-scope operations cost microseconds each on B200 (one-GPU ncu: a
// one-thread fence + release kernel 5.3 us; a system-scope atomic per push CTA made the push
// 18-22 us for 12.6 MB), so the push grid itself carries none.
__global__ void push_publish(P2PArgs a) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  __threadfence_system();
  const int g = threadIdx.x;
  if (g < a.world)
    st_release_sys(reinterpret_cast<int32_t*>(a.peers[g]) + 32 * (1 + a.rank), epoch + 1);
}

// Step 5 signal: after the FFN's remote partial-row stores (stream order): the FFN grid has
// completed, one system-scope fence, then flags_rs are released to every peer.
__global__ void rs_signal(P2PArgs a) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  __threadfence_system();
  const int g = threadIdx.x;
  if (g < a.world)
    st_release_sys(reinterpret_cast<int32_t*>(a.peers[g]) + 32 * (1 + a.world + a.rank), epoch + 1);
}

// Step 5 aggregate: out[i] = sum_g recv[g][i] (fp32, ascending g), then epoch += 1
// (every rank's partials for this rank's rows have landed: wait_partials, one CTA, just
// before - the flags are acquired once instead of by every CTA of the reduce)
__global__ void wait_partials(P2PArgs a, int32_t* err) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  if (threadIdx.x == 0)
    wait_flags(reinterpret_cast<const int32_t*>(a.self) + 32 * (1 + a.world), a.world, epoch + 1,
               err);
}
__global__ void __launch_bounds__(256) reduce_partials(P2PArgs a, int n, int row_vecs,
                                                       uint4* __restrict__ out, int32_t* err) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  const size_t nv = static_cast<size_t>(n) * row_vecs;
  const size_t slot = static_cast<size_t>(a.n_max) * row_vecs;
  const uint4* recv = reinterpret_cast<const uint4*>(a.self + a.off_recv);
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  constexpr int kU = 4;   // vectors per thread per pass; all G slots' loads of a pass in flight
  for (size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i0 < nv;
       i0 += kU * stride) {
    float acc[kU][8];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[u][k] = 0.f;
    for (int g = 0; g < a.world; ++g) {   // ascending rank: a fixed summation order
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i0 + u * stride < nv) v[u] = __ldcg(recv + g * slot + i0 + u * stride);   // peers' writes: L2
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (i0 + u * stride >= nv) continue;
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(b[k]);
          acc[u][2 * k] += f.x;
          acc[u][2 * k + 1] += f.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (i0 + u * stride >= nv) continue;
      uint4 o;
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) ob[k] = __floats2bfloat162_rn(acc[u][2 * k], acc[u][2 * k + 1]);
      out[i0 + u * stride] = o;
    }
  }
  // the last CTA out advances the epoch (every CTA has read it by now)
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* ctr = reinterpret_cast<int32_t*>(a.self) + 2;
    __threadfence();
    if (atomicAdd(ctr, 1) == static_cast<int>(gridDim.x) - 1) {
      *ctr = 0;
      *reinterpret_cast<volatile int32_t*>(a.self) = epoch + 1;
      __threadfence();
    }
  }
}

// grouping-side wait for Step 3 (one CTA; launched just before the grouping kernels)
__global__ void wait_tokens(P2PArgs a, int32_t* err) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  if (threadIdx.x == 0)
    wait_flags(reinterpret_cast<const int32_t*>(a.self) + 32, a.world, epoch + 1, err);
}

// ===========================================================================
// Expert-parallel baseline (MOESHARD_FLAG_EXPERT_PARALLEL, the
// comparison system of Sec. 4, with the DeepSpeed capacity of PAPER.md:393-398).
// Rank o hosts whole experts [o*E_loc, (o+1)*E_loc). The all-to-all scatter is a
// routed push: each admitted token row goes only to its expert's host, into the
// same rank-major x_all slot MoEShard uses (row r*n_max + i), with a route record
// carrying the LOCAL expert id (-1 in every other host's copy) and per-block
// histograms over the host's experts - so the host runs the unchanged Step-2
// grouping and fused FFN (F = d_ff) on what it received, and its down epilogue
// stores each result row into the source rank's receive slot (the all-to-all
// gather). Admission is first-come inside the source rank's minibatch: token i of
// expert e is kept iff fewer than `cap` earlier tokens of this rank chose e.
// ===========================================================================

// One group of kSplit CTAs per 128-token block of this rank's slot (n_max rows).
template <int kSplit>
__global__ void __launch_bounds__(256) ep_dispatch(P2PArgs a, const uint4* __restrict__ x, int n,
                                                   int row_vecs, const RouteRec* __restrict__ rec,
                                                   const int32_t* __restrict__ hist, int E,
                                                   int E_loc, int cap, int32_t* __restrict__ owner) {
  constexpr int kThreads = 256, kRows = 128 / kSplit;
  __shared__ int32_t s_pre[kMaxExperts];      // this rank's tokens of e in earlier blocks
  __shared__ int32_t s_kept[kMaxExperts];     // admitted tokens of e in this block
  __shared__ int32_t whist[4][kMaxExperts];
  __shared__ int32_t s_own[128];              // host rank of each token of the block, -1 dropped
  __shared__ int32_t s_el[128];               // local expert id at the host
  ptx::griddep_wait();   // route records / histograms come from the router
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  const int b = blockIdx.x / kSplit, part = blockIdx.x % kSplit;
  const int nbr = (a.n_max + 127) / 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb_own = (n + 127) / 128;   // blocks holding tokens (the router's histograms)
  for (int e = threadIdx.x; e < E; e += kThreads) {
    int sum = 0;
    for (int bb = 0; bb < min(b, nb_own); ++bb) sum += __ldg(hist + static_cast<size_t>(bb) * E + e);
    s_pre[e] = sum;
    s_kept[e] = 0;
  }
  for (int k = threadIdx.x; k < 4 * E; k += kThreads) whist[k / E][k % E] = 0;
  __syncthreads();
  int e = -1, rank_w = 0;
  const int t = b * 128 + threadIdx.x;
  float gate = 0.f;
  if (warp < 4) {
    if (t < n) {
      const RouteRec r = rec[t];
      e = r.expert;
      gate = r.gate;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    rank_w = __popc(peers & lanemask_lt());
    if (e >= 0 && rank_w == 0) whist[warp][e] = __popc(peers);
  }
  __syncthreads();
  if (warp < 4) {
    int own = -1, el = -1;
    if (e >= 0) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += whist[w][e];
      if (s_pre[e] + before + rank_w < cap) {   // first-come admission (R20)
        own = e / E_loc;
        el = e - own * E_loc;
        atomicAdd(&s_kept[e], 1);
      }
    }
    s_own[threadIdx.x] = own;
    s_el[threadIdx.x] = el;
    if (part == 0 && t < a.n_max) {
      if (t < n) owner[t] = own;
      for (int g = 0; g < a.world; ++g) {   // every host's copy of this rank's slot
        RouteRec r;
        r.expert = g == own ? el : -1;
        r.gate = g == own ? gate : 0.f;
        reinterpret_cast<RouteRec*>(a.peers[g] + a.off_route)[static_cast<size_t>(a.rank) * a.n_max + t] = r;
      }
    }
  }
  __syncthreads();
  if (part == 0 && b < nbr) {   // admitted-token histograms over each host's experts
    for (int k = threadIdx.x; k < a.world * E_loc; k += kThreads) {
      const int g = k / E_loc, el = k - g * E_loc;
      int32_t* dh = reinterpret_cast<int32_t*>(a.peers[g] + a.off_hist);
      dh[(static_cast<size_t>(a.rank) * nbr + b) * E_loc + el] = s_kept[g * E_loc + el];
    }
  }
  // admitted rows to their host's x_all slot (8 warps x kRows / 8 rows, 16-B vectors)
  for (int rr = warp; rr < kRows; rr += kThreads / 32) {
    const int j = part * kRows + rr;
    const int own = s_own[j];
    const int tt = b * 128 + j;
    if (own < 0) continue;
    const uint4* src = x + static_cast<size_t>(tt) * row_vecs;
    uint4* dst = reinterpret_cast<uint4*>(a.peers[own] + a.off_x) +
                 (static_cast<size_t>(a.rank) * a.n_max + tt) * row_vecs;
    for (int c = lane; c < row_vecs; c += 32) dst[c] = __ldg(src + c);
  }
  // publish: every CTA's stores fenced at system scope, then the last CTA raises
  // flags_ag[rank] on every host (as push_tokens)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    int32_t* ctr = reinterpret_cast<int32_t*>(a.self) + 1;
    if (atomicAdd(ctr, 1) == static_cast<int>(gridDim.x) - 1) {
      *ctr = 0;
      __threadfence_system();
      for (int g = 0; g < a.world; ++g)
        st_release_sys(reinterpret_cast<int32_t*>(a.peers[g]) + 32 * (1 + a.rank), epoch + 1);
    }
  }
}

// EP all-to-all gather: out[i] = recv[owner[i]][i] (the host's gate-scaled row), 0 for a
// dropped token; waits for every host's signal, then advances the epoch.
__global__ void __launch_bounds__(256) ep_combine(P2PArgs a, int n, int row_vecs,
                                                  const int32_t* __restrict__ owner,
                                                  uint4* __restrict__ out, int32_t* err) {
  const int32_t epoch = *reinterpret_cast<volatile int32_t*>(a.self);
  if (threadIdx.x == 0)
    wait_flags(reinterpret_cast<const int32_t*>(a.self) + 32 * (1 + a.world), a.world, epoch + 1,
               err);
  __syncthreads();
  const uint4* recv = reinterpret_cast<const uint4*>(a.self + a.off_recv);
  const size_t slot = static_cast<size_t>(a.n_max) * row_vecs;
  const int warps = gridDim.x * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const int o = __ldg(owner + i);
    uint4* dst = out + static_cast<size_t>(i) * row_vecs;
    if (o < 0) {
      for (int c = lane; c < row_vecs; c += 32) dst[c] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      const uint4* src = recv + o * slot + static_cast<size_t>(i) * row_vecs;
      for (int c = lane; c < row_vecs; c += 32) dst[c] = __ldcg(src + c);   // peers' writes: L2
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* ctr = reinterpret_cast<int32_t*>(a.self) + 2;
    __threadfence();
    if (atomicAdd(ctr, 1) == static_cast<int>(gridDim.x) - 1) {
      *ctr = 0;
      *reinterpret_cast<volatile int32_t*>(a.self) = epoch + 1;
      __threadfence();
    }
  }
}

}  // namespace

P2PLayout p2p_layout(int world, int n_max, int h, int E, int nbr_max) {
  auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  P2PLayout L{};
  size_t off = al(static_cast<size_t>(32) * 4 * (1 + 2 * world));
  L.off_x = off;
  off += al(static_cast<size_t>(world) * n_max * h * 2);
  L.off_route = off;
  off += al(static_cast<size_t>(world) * n_max * sizeof(RouteRec));
  L.off_hist = off;
  off += al(static_cast<size_t>(world) * nbr_max * E * 4);
  L.off_recv = off;
  off += al(static_cast<size_t>(world) * n_max * h * 2);
  L.total = off;
  return L;
}

cudaError_t launch_p2p_push(const P2PArgs& a, const void* x, int n, int ns, int row_vecs, int nbr,
                            int E, int num_sms, cudaStream_t s) {
  if (ns <= 0) return cudaSuccess;
  const size_t work = static_cast<size_t>(std::max(n, 1)) * row_vecs;
  // 4 CTAs x 256 threads x 8 vectors = 128 KB of rows in flight per SM (ncu: 2 CTAs per SM
  // left the push latency-bound at 18 % of DRAM bandwidth)
  const int grid = static_cast<int>(std::min<size_t>(4 * num_sms, (work + 2047) / 2048));
  cudaError_t e = launch_pdl(push_tokens, dim3(std::max(grid, 1)), dim3(256), 0, s, a,
                             static_cast<const uint4*>(x), n, ns, row_vecs, nbr, E);
  if (e != cudaSuccess) return e;
  push_publish<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ep_dispatch(const P2PArgs& a, const void* x, int n, int row_vecs,
                               const RouteRec* rec, const int32_t* hist, int E, int E_loc, int cap,
                               int32_t* owner, cudaStream_t s) {
  const int nbr = (a.n_max + 127) / 128;
  return launch_pdl(ep_dispatch<4>, dim3(nbr * 4), dim3(256), 0, s, a, static_cast<const uint4*>(x),
                    n, row_vecs, rec, hist, E, E_loc, cap, owner);
}

cudaError_t launch_ep_combine(const P2PArgs& a, int n, int row_vecs, const int32_t* owner, void* out,
                              int32_t* err, int num_sms, cudaStream_t s) {
  const int grid = std::max(1, std::min(4 * num_sms, (n + 7) / 8));
  ep_combine<<<grid, 256, 0, s>>>(a, n, row_vecs, owner, static_cast<uint4*>(out), err);
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait_tokens(const P2PArgs& a, int32_t* err, cudaStream_t s) {
  wait_tokens<<<1, 32, 0, s>>>(a, err);
  return cudaGetLastError();
}

cudaError_t launch_p2p_signal_partials(const P2PArgs& a, cudaStream_t s) {
  rs_signal<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_p2p_reduce(const P2PArgs& a, int n, int row_vecs, void* out, int32_t* err,
                              int num_sms, cudaStream_t s) {
  // runs even for n = 0 (uneven token counts): it consumes the flags and advances the epoch
  const size_t work = static_cast<size_t>(n) * row_vecs;
  const int grid = static_cast<int>(std::min<size_t>(3 * num_sms, (work + 1023) / 1024));
  wait_partials<<<1, 32, 0, s>>>(a, err);
  reduce_partials<<<std::max(grid, 1), 256, 0, s>>>(a, n, row_vecs, static_cast<uint4*>(out), err);
  return cudaGetLastError();
}

}  // namespace moeshard
