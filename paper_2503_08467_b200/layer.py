"""Torch-facing wrapper of the C ABI: one object per rank serving n_layers MoE layers.

Marshalling only - buffers are torch tensors, pointers and the current CUDA
stream are passed through to libmoeshard.so. For world > 1 rank 0 creates
the NCCL unique id and it is broadcast with torch.distributed (CS3 in
SURVEY.md §3; collective contract of moeshard_init).
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch

from . import moeshard as C

_DTYPES = {torch.bfloat16: C.MOESHARD_BF16, torch.float32: C.MOESHARD_FP32}


def shard_columns(d_ff: int, world: int, rank: int) -> Tuple[int, int]:
    """This rank's contiguous slice of W_i's columns / W_o's rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} not in [0, {world})")
    if d_ff % world:
        raise ValueError(f"d_ff={d_ff} is not divisible by world={world} (PAPER.md:169)")
    F = d_ff // world
    return rank * F, (rank + 1) * F


def local_token_range(n_global: int, world: int, rank: int) -> Tuple[int, int]:
    """Tokens of rank r in the global rank-major order t = r*n + i (equal split, v1)."""
    if n_global % world:
        raise ValueError(f"global token count {n_global} not divisible by world {world}")
    n = n_global // world
    return rank * n, (rank + 1) * n


def broadcast_uid(uid: Optional[bytes], rank: int, group=None) -> bytes:
    """Rank 0's 128-byte NCCL id to every rank over torch.distributed (any backend)."""
    import torch.distributed as dist
    obj: List[Optional[bytes]] = [uid if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    assert obj[0] is not None and len(obj[0]) == 128
    return obj[0]


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class MoEShardLayer:
    """Sharded Switch-MoE FFN layers on one GPU of a `world`-GPU job."""

    def __init__(self, d_model: int, d_ff: int, n_experts: int, *, n_layers: int = 1,
                 max_tokens_per_rank: int, dtype=torch.bfloat16, rank: int = 0, world: int = 1,
                 device: Optional[int] = None, flags: int = 0, group=None,
                 ep_capacity_factor: float = 0.0, top_k: int = 1):
        """flags & MOESHARD_FLAG_EXPERT_PARALLEL builds the paper's expert-parallel baseline
        instead (needs MOESHARD_FLAG_P2P): this rank then hosts experts
        [rank*E/world, (rank+1)*E/world) whole, and load_expert_shards takes
        [E/world, h, d_ff] / [E/world, d_ff, h]; ep_capacity_factor <= 0 means min(E, 50).
        top_k = 2: two experts per token (R21); routing tables then have one entry per
        (token, choice) assignment and forced_expert is int32 [n, 2]."""
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be bf16 or fp32, got {dtype}")
        self.device = torch.cuda.current_device() if device is None else device
        self.dtype, self.rank, self.world = dtype, rank, world
        self.h, self.d_ff, self.E = d_model, d_ff, n_experts
        self.ep = bool(flags & C.MOESHARD_FLAG_EXPERT_PARALLEL)
        self.F = d_ff if self.ep else d_ff // world
        self.E_host = n_experts // world if self.ep else n_experts   # experts computed here
        self.top_k = max(1, top_k)
        self.cfg = C.moeshard_config(d_model, d_ff, n_experts, n_layers, max_tokens_per_rank,
                                     _DTYPES[dtype], flags, ep_capacity_factor, top_k)
        ws = C.moeshard_workspace_size(self.cfg, world)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._wbytes = C.moeshard_weight_storage_size(self.cfg, world)
        self._storage: List[Optional[torch.Tensor]] = [None] * n_layers
        uid = None
        p2p = bool(flags & C.MOESHARD_FLAG_P2P)
        if not p2p and (world > 1 or (flags & C.MOESHARD_FLAG_FORCE_COLLECTIVES)):
            uid = C.moeshard_get_unique_id() if rank == 0 else None
            if world > 1:
                uid = broadcast_uid(uid, rank, group)
        self.ctx = C.moeshard_init(self.cfg, rank, world, uid, self.workspace.data_ptr(), ws,
                                   self.device)
        if p2p and world > 1:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                self.p2p_connect_group(group)     # one process per rank
        elif p2p:
            self.p2p_connect([self.p2p_region()])

    def _stream(self) -> int:
        """The current stream of this layer's device (not of the current device)."""
        return torch.cuda.current_stream(self.device).cuda_stream

    def load_expert_shards(self, layer: int, w_in_shard: torch.Tensor, w_out_shard: torch.Tensor):
        """w_in_shard [E, h, d_ff/world], w_out_shard [E, d_ff/world, h] (this rank's slices);
        expert-parallel baseline: [E/world, h, d_ff] / [E/world, d_ff, h] (this rank's experts)."""
        exp_in, exp_out = (self.E_host, self.h, self.F), (self.E_host, self.F, self.h)
        if tuple(w_in_shard.shape) != exp_in or tuple(w_out_shard.shape) != exp_out:
            raise C.MoEShardError(-2, f"shards {tuple(w_in_shard.shape)}/{tuple(w_out_shard.shape)}"
                                      f" vs expected {exp_in}/{exp_out}")
        w_in_shard = w_in_shard.to(device=f"cuda:{self.device}", dtype=self.dtype).contiguous()
        w_out_shard = w_out_shard.to(device=f"cuda:{self.device}", dtype=self.dtype).contiguous()
        st = torch.empty(self._wbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        C.moeshard_load_expert_shards(self.ctx, layer, w_in_shard.data_ptr(),
                                      w_out_shard.data_ptr(), st.data_ptr(), self._wbytes,
                                      self._stream())
        torch.cuda.current_stream(self.device).synchronize()  # inputs may be freed afterwards
        self._storage[layer] = st

    # ---------------------------------------------------------- peer-memory exchange
    def p2p_region(self) -> int:
        """Device pointer of this rank's exchange region (MOESHARD_FLAG_P2P)."""
        return C.moeshard_p2p_region(self.ctx)[0]

    def p2p_connect(self, regions):
        """regions[g] = rank g's exchange region as mapped in this process."""
        C.moeshard_p2p_connect(self.ctx, list(regions))

    def p2p_connect_group(self, group=None):
        """One process per rank: exchange CUDA IPC handles over torch.distributed
        (host bytes only), map every peer's region, connect."""
        import torch.distributed as dist
        mine = C.moeshard_p2p_export(self.ctx)
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        regions = [self.p2p_region() if g == self.rank else C.moeshard_p2p_open(self.ctx, handles[g])
                   for g in range(self.world)]
        self.p2p_connect(regions)

    @staticmethod
    def p2p_connect_local(layers):
        """Ranks that share one process (and GPU): connect their regions directly."""
        regions = [l.p2p_region() for l in layers]
        for l in layers:
            l.p2p_connect(regions)

    def forward(self, layer: int, hidden: torch.Tensor, router_w: torch.Tensor,
                forced_expert: Optional[torch.Tensor] = None,
                out: Optional[torch.Tensor] = None, stages: int = C.MOESHARD_STAGE_ALL) -> torch.Tensor:
        n = hidden.shape[0]
        if hidden.device != torch.device("cuda", self.device):
            raise C.MoEShardError(-1, f"hidden is on {hidden.device}, the layer on cuda:{self.device}")
        if hidden.dtype != self.dtype or router_w.dtype != self.dtype:
            raise C.MoEShardError(-1, f"hidden/router_w must be {self.dtype}")
        if hidden.dim() != 2 or hidden.shape[1] != self.h or tuple(router_w.shape) != (self.h, self.E):
            raise C.MoEShardError(-2, f"hidden {tuple(hidden.shape)} / router_w {tuple(router_w.shape)}"
                                      f" vs expected [n, {self.h}] / [{self.h}, {self.E}]")
        if not (hidden.is_contiguous() and router_w.is_contiguous()):
            raise C.MoEShardError(-1, "hidden and router_w must be contiguous")
        if out is None:
            out = torch.empty_like(hidden)
        if forced_expert is not None:
            shape = (n,) if self.top_k == 1 else (n, self.top_k)
            if forced_expert.dtype != torch.int32 or tuple(forced_expert.shape) != shape:
                raise C.MoEShardError(-2, f"forced_expert must be int32 {list(shape)}")
        if stages == C.MOESHARD_STAGE_ALL:
            C.moeshard_forward(self.ctx, layer, hidden.data_ptr(), n, router_w.data_ptr(),
                               out.data_ptr(), _ptr(forced_expert), self._stream())
        else:
            C.moeshard_forward_stages(self.ctx, layer, hidden.data_ptr(), n, router_w.data_ptr(),
                                      out.data_ptr(), _ptr(forced_expert), stages, self._stream())
        return out

    __call__ = forward

    def routing(self, n_local: int) -> dict:
        """Routing tables of the last forward. With MOESHARD_FLAG_UNEVEN_TOKENS the token
        index space is world slots of max_tokens_per_rank (unused slot entries: expert -1)."""
        if self._collective() and (self.cfg.flags & (C.MOESHARD_FLAG_UNEVEN_TOKENS |
                                                     C.MOESHARD_FLAG_EXPERT_PARALLEL)):
            n_local = self.cfg.max_tokens_per_rank
        N = n_local * (self.world if self._collective() else 1) * self.top_k   # assignments
        dev = f"cuda:{self.device}"
        r = {
            "expert": torch.empty(N, dtype=torch.int32, device=dev),
            "gate": torch.empty(N, dtype=torch.float32, device=dev),
            "counts": torch.empty(self.E_host, dtype=torch.int32, device=dev),
            "offsets": torch.empty(self.E_host + 1, dtype=torch.int32, device=dev),
            "perm": torch.empty(N, dtype=torch.int32, device=dev),
        }
        C.moeshard_get_routing(self.ctx, r["expert"].data_ptr(), r["gate"].data_ptr(),
                               r["counts"].data_ptr(), r["offsets"].data_ptr(),
                               r["perm"].data_ptr(), self._stream())
        return r

    def ep_admission(self, n_local: int) -> dict:
        """Expert-parallel baseline: this rank's admission of its last forward - owner (host
        rank, -1 = dropped), expert, gate per local token, and the tokens its experts received."""
        dev = f"cuda:{self.device}"
        r = {"owner": torch.empty(n_local, dtype=torch.int32, device=dev),
             "expert": torch.empty(n_local, dtype=torch.int32, device=dev),
             "gate": torch.empty(n_local, dtype=torch.float32, device=dev),
             "received": torch.empty(self.E_host, dtype=torch.int32, device=dev)}
        C.moeshard_get_ep_admission(self.ctx, r["owner"].data_ptr(), r["expert"].data_ptr(),
                                    r["gate"].data_ptr(), r["received"].data_ptr(), self._stream())
        return r

    def _collective(self) -> bool:
        return self.world > 1 or bool(self.cfg.flags & (C.MOESHARD_FLAG_FORCE_COLLECTIVES |
                                                         C.MOESHARD_FLAG_P2P))

    def stats(self) -> dict:
        return C.moeshard_get_stats(self.ctx, self._stream())

    def profile(self, enable: bool = True):
        C.moeshard_profile(self.ctx, enable)

    def phase_ms(self):
        return C.moeshard_get_phase_ms(self.ctx)

    def forward_host(self, layer: int, hidden_host: torch.Tensor, router_w: torch.Tensor,
                     dev_in: torch.Tensor, dev_out: torch.Tensor, host_out: torch.Tensor,
                     forced_expert: Optional[torch.Tensor] = None) -> torch.Tensor:
        """End-to-end call with HOST buffers: H2D copy of the tokens (pinned),
        the forward, D2H copy of the result - all enqueued on the current stream."""
        dev_in.copy_(hidden_host, non_blocking=True)
        self.forward(layer, dev_in, router_w, forced_expert=forced_expert, out=dev_out)
        host_out.copy_(dev_out, non_blocking=True)
        return host_out

    def host_streamer(self, n_local: int) -> "HostStreamer":
        """Streaming inference from/to pinned host memory (see HostStreamer)."""
        return HostStreamer(self, n_local)

    def check(self):
        C.moeshard_check(self.ctx, self._stream())

    def close(self):
        if getattr(self, "ctx", None) is not None:
            C.moeshard_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostStreamer:
    """Streams batches of tokens between pinned host memory and the layer.

    A three-stage software pipeline in lock step: step(k) issues the H2D copy of
    batch k (copy stream), the forward of batch k-1 (the caller's stream) and the
    D2H copy of batch k-2's output (second copy stream) together, then joins the
    three into the caller's stream, so a step costs max(H2D || D2H, forward) and
    both PCIe directions stay busy. (The former per-batch event chain, with NBUF
    buffers and cross-stream waits per copy, left the copy engines idle between
    batches: 304 us vs 258 us per c2 step, scripts/e2e_probe.py.) Two device
    buffers per direction suffice: a buffer is rewritten two steps after it was
    filled, one join after its reader ran.

    Host-buffer contract (the copies are asynchronous DMAs; nothing here blocks the
    host): step() returns the batch index k. host_in of batch k may be refilled only
    after input_done(k) (its H2D has completed; a CUDA event, wait with
    .synchronize()). host_out of batch k holds the result only after output_done(k)
    has completed; that event exists once the D2H was issued, by step(k+2) or join().
    router_w and forced_expert of batch k must stay unchanged until output_done(k).
    join() drains the pipeline (issues the last forward and copies) and makes the
    caller's stream wait for them. Marshalling only: the forward is the library's."""

    NBUF = 2
    KEEP = 8   # events kept per direction (batches older than k - KEEP are long complete)

    def __init__(self, layer: MoEShardLayer, n_local: int):
        self.layer = layer
        dev = f"cuda:{layer.device}"
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        nb = self.NBUF
        self.din = [torch.empty(n_local, layer.h, dtype=layer.dtype, device=dev) for _ in range(nb)]
        self.dout = [torch.empty_like(self.din[0]) for _ in range(nb)]
        self.k = 0
        self.to_forward = None   # (buffer, batch, layer_idx, router_w, forced) of batch k-1
        self.to_copy = None      # (buffer, batch) of batch k-2
        self.host_out = {}       # batch -> pinned host output tensor
        self.in_ev = {}          # batch -> event after its H2D
        self.out_ev = {}         # batch -> event after its D2H

    def _prune(self):
        for d in (self.in_ev, self.out_ev, self.host_out):
            for b in [b for b in d if b < self.k - self.KEEP]:
                if d is not self.host_out or b in self.out_ev:
                    del d[b]

    def _advance(self, new_in) -> None:
        comp = torch.cuda.current_stream(self.layer.device)
        self.h2d.wait_stream(comp)
        self.d2h.wait_stream(comp)
        if new_in is not None:
            b, batch, host_in = new_in
            with torch.cuda.stream(self.h2d):
                self.din[b].copy_(host_in, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.h2d)
                self.in_ev[batch] = ev
        if self.to_copy is not None:
            b, batch = self.to_copy
            with torch.cuda.stream(self.d2h):
                self.host_out[batch].copy_(self.dout[b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.d2h)
                self.out_ev[batch] = ev
        self.to_copy = None
        if self.to_forward is not None:
            b, batch, layer_idx, router_w, forced = self.to_forward
            self.layer.forward(layer_idx, self.din[b], router_w, forced_expert=forced,
                               out=self.dout[b])
            self.to_copy = (b, batch)
        comp.wait_stream(self.h2d)
        comp.wait_stream(self.d2h)

    def step(self, layer_idx: int, host_in: torch.Tensor, router_w: torch.Tensor,
             host_out: torch.Tensor, forced_expert: Optional[torch.Tensor] = None) -> int:
        k = self.k
        b = k % self.NBUF
        self.host_out[k] = host_out
        self._advance((b, k, host_in))
        self.to_forward = (b, k, layer_idx, router_w, forced_expert)
        self.k += 1
        self._prune()
        return k

    def input_done(self, k: int) -> torch.cuda.Event:
        """Event after the H2D copy of batch k (host_in of k may be refilled once it completes)."""
        return self.in_ev[k]

    def output_done(self, k: int) -> torch.cuda.Event:
        """Event after the D2H copy of batch k (issued by step(k+2) or join())."""
        if k not in self.out_ev:
            raise RuntimeError(f"batch {k}: D2H not issued yet (call step() twice more or join())")
        return self.out_ev[k]

    def join(self):
        while self.to_forward is not None or self.to_copy is not None:
            self._advance(None)
            self.to_forward = None
