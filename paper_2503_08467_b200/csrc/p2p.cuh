// p2p.cuh - host interface of the peer-memory exchange (p2p.cu, MOESHARD_FLAG_P2P).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace moeshard {

struct P2PLayout {
  size_t off_x, off_route, off_hist, off_recv, total;
};

// Region of one rank for `world` ranks of at most n_max tokens, d_model h, E experts,
// nbr_max hist-blocks per rank.
P2PLayout p2p_layout(int world, int n_max, int h, int E, int nbr_max);

struct P2PArgs {
  char* self;                 // this rank's region (device pointer)
  char* peers[kMaxWorld];     // every rank's region as mapped in this process (peers[rank] == self)
  int rank, world, n_max;
  size_t off_x, off_route, off_hist, off_recv;
};

// Step 3: copy x [n][row_vecs x 16 B], this rank's route records and block histograms
// (already in its own region slot) into slot `rank` of every region; publish flags_ag.
cudaError_t launch_p2p_push(const P2PArgs& a, const void* x, int n, int ns, int row_vecs, int nbr,
                            int E, int num_sms, cudaStream_t s);
// wait until every rank's Step-3 data has landed in this rank's region (bounded; err bit 4)
cudaError_t launch_p2p_wait_tokens(const P2PArgs& a, int32_t* err, cudaStream_t s);
// after the FFN wrote its partial rows into the owners' recv slots: publish flags_rs
cudaError_t launch_p2p_signal_partials(const P2PArgs& a, cudaStream_t s);
// Step 5: wait for every rank's partials, out = sum over ranks (fp32, ascending rank), epoch++
cudaError_t launch_p2p_reduce(const P2PArgs& a, int n, int row_vecs, void* out, int32_t* err,
                              int num_sms, cudaStream_t s);

// Expert-parallel baseline (MOESHARD_FLAG_EXPERT_PARALLEL): routed push of this rank's
// admitted tokens (rec / hist: its router's output for n tokens over E experts) to the
// hosts of their experts (E_loc per rank), capacity `cap` per expert (first-come);
// owner[i] = host of token i or -1 (dropped). Publishes flags_ag like launch_p2p_push.
cudaError_t launch_ep_dispatch(const P2PArgs& a, const void* x, int n, int row_vecs,
                               const RouteRec* rec, const int32_t* hist, int E, int E_loc, int cap,
                               int32_t* owner, cudaStream_t s);
// EP gather: out[i] = the host's result row for token i (recv[owner[i]][i]), 0 if dropped.
cudaError_t launch_ep_combine(const P2PArgs& a, int n, int row_vecs, const int32_t* owner, void* out,
                              int32_t* err, int num_sms, cudaStream_t s);

}  // namespace moeshard
