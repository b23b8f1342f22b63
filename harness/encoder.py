"""Switch-style encoder stack for the TTFT measurement.

Measurement harness, not the product: the non-MoE blocks (RMSNorm, multi-head
self-attention, dense FFN) are plain torch (cuBLAS / SDPA library kernels) and
are replicated data-parallel on every rank; every
other FFN is an MoE FFN executed by the library (libmoeshard via
MoEShardLayer, all ranks collectively). TTFT = one forward of the whole
encoder over the batch. Synthetic random-init weights of the
Switch-Base / Switch-Large shapes; T5 relative position bias is omitted (it
does not touch the studied mechanism).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.nn.functional as Fn

import workload as W


@dataclass
class EncoderConfig:
    d_model: int = 768
    d_ff: int = 3072
    n_heads: int = 12
    n_layers: int = 12
    n_experts: int = 128
    moe_every: int = 2        # MoE at odd layer indices 1, 3, ... (R18)
    seq: int = 512
    batch: int = 32           # global batch; each rank holds batch / world sequences


class SwitchEncoder:
    def __init__(self, cfg: EncoderConfig, *, seed: int, rank: int = 0, world: int = 1,
                 device="cuda", moe_layer_factory=None):
        self.cfg = cfg
        self.rank, self.world = rank, world
        h, dt = cfg.d_model, torch.bfloat16
        self.moe_ids = [i for i in range(cfg.n_layers) if i % cfg.moe_every == 1]
        n_local = (cfg.batch // world) * cfg.seq
        self.moe = moe_layer_factory(len(self.moe_ids), n_local) if moe_layer_factory else None
        self.layers = []
        c0, c1 = rank * (cfg.d_ff // world), (rank + 1) * (cfg.d_ff // world)
        for i in range(cfg.n_layers):
            s = seed * 1000 + i
            L = {
                "ln1": torch.ones(h, dtype=dt, device=device),
                "ln2": torch.ones(h, dtype=dt, device=device),
                "wqkv": W.normal_tensor(s, 101, (h, 3 * h), scale=1 / math.sqrt(h), dtype=dt, device=device),
                "wo": W.normal_tensor(s, 102, (h, h), scale=1 / math.sqrt(h), dtype=dt, device=device),
            }
            if i in self.moe_ids:
                j = self.moe_ids.index(i)
                L["w_r"] = W.make_router_weight(s, h, cfg.n_experts, device=device, layer=0)
                wi, wo = W.make_expert_weights(s, cfg.n_experts, h, cfg.d_ff, cols=(c0, c1),
                                               device=device)
                self.moe.load_expert_shards(j, wi, wo)
                del wi, wo
                L["moe_slot"] = j
            else:
                L["wi"] = W.normal_tensor(s, 103, (h, cfg.d_ff), scale=1 / math.sqrt(h), dtype=dt, device=device)
                L["wf"] = W.normal_tensor(s, 104, (cfg.d_ff, h), scale=1 / math.sqrt(cfg.d_ff), dtype=dt, device=device)
            self.layers.append(L)
        self.moe_out = None

    def forward(self, x: torch.Tensor, forced: Optional[List[torch.Tensor]] = None,
                capture: Optional[list] = None) -> torch.Tensor:
        """x [b_local, seq, h] -> [b_local, seq, h]. capture (test hook): a list that receives,
        per MoE layer, {slot, input, output, routing} copies for teacher-forced parity."""
        cfg = self.cfg
        b, s, h = x.shape
        nh, hd = cfg.n_heads, h // cfg.n_heads
        for L in self.layers:
            y = Fn.rms_norm(x, (h,), L["ln1"], 1e-6)
            qkv = (y.view(-1, h) @ L["wqkv"]).view(b, s, 3, nh, hd).permute(2, 0, 3, 1, 4)
            a = Fn.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])
            x = x + (a.transpose(1, 2).reshape(-1, h) @ L["wo"]).view(b, s, h)
            y = Fn.rms_norm(x, (h,), L["ln2"], 1e-6).view(-1, h).contiguous()
            if "moe_slot" in L:
                if self.moe_out is None or self.moe_out.shape != y.shape:
                    self.moe_out = torch.empty_like(y)
                f = None if forced is None else forced[L["moe_slot"]]
                z = self.moe.forward(L["moe_slot"], y, L["w_r"], forced_expert=f, out=self.moe_out)
                if capture is not None:
                    capture.append({"slot": L["moe_slot"], "input": y.clone(), "output": z.clone(),
                                    "routing": self.moe.routing(y.shape[0])})
            else:
                z = torch.relu(y @ L["wi"]) @ L["wf"]
            x = x + z.view(b, s, h)
        return x
