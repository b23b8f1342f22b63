"""Seeded synthetic workload generator shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no routing, no expert
FFN, no grouping): it only produces input tensors and, for the paper's
replaced-router experiments (§4.1), the per-token expert
draws that are handed to the layer as ``forced_expert``.

Every element is a pure function of ``(seed, stream, flat_index)`` through a
counter-based generator (two rounds of the 32-bit ``lowbias32`` integer hash,
then Box-Muller), so

* any slice of a tensor (e.g. rank r's column shard of W_i)
  can be generated without materialising the rest, and
* the same values come out on CPU and on CUDA (integer hashing is exact; the
  Box-Muller transform is evaluated in float64 and rounded once to the
  requested dtype).

Input recipe:
  x   ~ N(0, 1)                 tokens, post-attention hidden states
  W_r ~ N(0, 1/h)               router weight [h, E]
  W_i ~ N(0, 1/h)               expert up-projection  [E, h, d_ff]
  W_o ~ N(0, 1/d_ff)            expert down-projection [E, d_ff, h]
(scale 1/sqrt(fan-in)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

__all__ = [
    "STREAM_X", "STREAM_WR", "STREAM_WI", "STREAM_WO", "STREAM_ROUTE",
    "hash32_int", "uniform_at", "normal_at", "normal_tensor", "LayerInputs",
    "make_layer_inputs", "make_tokens", "make_router_weight", "make_expert_weights",
    "skew_probabilities", "zipf_probabilities", "draw_experts", "round_to",
]

STREAM_X, STREAM_WR, STREAM_WI, STREAM_WO, STREAM_ROUTE, STREAM_PERM = 1, 2, 3, 4, 5, 6

_M32 = 0xFFFFFFFF


# --------------------------------------------------------------------------
# counter-based generator
# --------------------------------------------------------------------------
def hash32_int(x: int) -> int:
    """lowbias32 on a Python int (scalar key derivation)."""
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & _M32
    x ^= x >> 16
    return x


def _mul32(a: torch.Tensor, b: int) -> torch.Tensor:
    """(a * b) mod 2^32 for int64 tensors holding values in [0, 2^32).

    Split into 16-bit halves of b so no intermediate exceeds 2^49 (no
    signed-overflow reliance on any device)."""
    b_lo, b_hi = b & 0xFFFF, b >> 16
    return (a * b_lo + (((a * b_hi) & 0xFFFF) << 16)) & _M32


def _hash32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _keys(seed: int, stream: int, salt: int):
    k1 = hash32_int(hash32_int(seed * 0x9E3779B1 + 0x632BE5AB) ^ (stream * 0x85EBCA77) ^ salt)
    k2 = hash32_int(k1 ^ 0x27D4EB2F ^ (seed >> 32))
    return k1, k2


def _bits_at(seed: int, stream: int, salt: int, idx: torch.Tensor) -> torch.Tensor:
    k1, k2 = _keys(seed, stream, salt)
    lo = idx & _M32
    hi = idx >> 32
    return _hash32(_hash32(lo ^ k1) ^ ((hi * 0x9E3779B1) & _M32) ^ k2)


def uniform_at(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """U(0,1) float64 (open interval) at flat int64 indices ``idx``."""
    b = _bits_at(seed, stream, 0x1234567, idx.to(torch.int64))
    return (b.to(torch.float64) + 0.5) * (1.0 / 4294967296.0)


def normal_at(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """N(0,1) float64 at flat int64 indices (Box-Muller on two uniforms)."""
    idx = idx.to(torch.int64)
    b1 = _bits_at(seed, stream, 0x0BADF00D, idx)
    b2 = _bits_at(seed, stream, 0x5EED5EED, idx)
    u1 = (b1.to(torch.float64) + 0.5) * (1.0 / 4294967296.0)
    u2 = (b2.to(torch.float64) + 0.5) * (1.0 / 4294967296.0)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * math.pi) * u2)


def normal_tensor(seed: int, stream: int, shape: Sequence[int], *, scale: float = 1.0,
                  dtype=torch.float32, device="cpu", offset: int = 0,
                  chunk: int = 1 << 24) -> torch.Tensor:
    """Dense tensor whose element at row-major flat index i is normal_at(offset + i)."""
    numel = 1
    for s in shape:
        numel *= int(s)
    out = torch.empty(numel, dtype=dtype, device=device)
    for s in range(0, numel, chunk):
        e = min(numel, s + chunk)
        idx = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device)
        out[s:e] = (normal_at(seed, stream, idx) * scale).to(dtype)
    return out.view(*shape)


def round_to(t: torch.Tensor, dtype) -> torch.Tensor:
    """Round to the storage dtype the GPU consumes (bf16 / fp32)."""
    return t.to(dtype)


# --------------------------------------------------------------------------
# layer inputs
# --------------------------------------------------------------------------
def make_tokens(seed: int, n_tokens: int, h: int, *, dtype=torch.bfloat16, device="cpu",
                layer: int = 0, token_offset: int = 0) -> torch.Tensor:
    """Tokens x[t, k] for global token ids token_offset .. token_offset+n_tokens-1."""
    return normal_tensor(seed, STREAM_X + 16 * layer, (n_tokens, h), dtype=dtype,
                         device=device, offset=token_offset * h)


def make_router_weight(seed: int, h: int, E: int, *, dtype=torch.bfloat16, device="cpu",
                       layer: int = 0) -> torch.Tensor:
    return normal_tensor(seed, STREAM_WR + 16 * layer, (h, E), scale=1.0 / math.sqrt(h),
                         dtype=dtype, device=device)


def make_expert_weights(seed: int, E: int, h: int, d_ff: int, *, cols: Optional[tuple] = None,
                        dtype=torch.bfloat16, device="cpu", layer: int = 0,
                        experts: Optional[Sequence[int]] = None):
    """(W_i [E', h, F], W_o [E', F, h]) with F the d_ff slice ``cols=(c0, c1)``.

    Element (e, k, j) of the FULL W_i is normal_at(e*h*d_ff + k*d_ff + j) and
    element (e, j, k) of the full W_o is normal_at(e*d_ff*h + j*h + k), so a
    rank's column/row shard is generated on its own."""
    c0, c1 = cols if cols is not None else (0, d_ff)
    ex = list(range(E)) if experts is None else list(experts)
    F = c1 - c0
    wi = torch.empty((len(ex), h, F), dtype=dtype, device=device)
    wo = torch.empty((len(ex), F, h), dtype=dtype, device=device)
    k = torch.arange(h, dtype=torch.int64, device=device)
    j = torch.arange(c0, c1, dtype=torch.int64, device=device)
    for n, e in enumerate(ex):
        idx_i = e * h * d_ff + k[:, None] * d_ff + j[None, :]
        wi[n] = (normal_at(seed, STREAM_WI + 16 * layer, idx_i) / math.sqrt(h)).to(dtype)
        idx_o = e * d_ff * h + j[:, None] * h + k[None, :]
        wo[n] = (normal_at(seed, STREAM_WO + 16 * layer, idx_o) / math.sqrt(d_ff)).to(dtype)
    return wi, wo


@dataclass
class LayerInputs:
    x: torch.Tensor          # [N, h] all ranks' tokens, rank-major (global t = r*n + i)
    w_r: torch.Tensor        # [h, E]
    w_i: torch.Tensor        # [E, h, d_ff]
    w_o: torch.Tensor        # [E, d_ff, h]
    forced: Optional[torch.Tensor]  # [N] int32 or None (natural routing)


def make_layer_inputs(seed: int, N: int, h: int, d_ff: int, E: int, *, dtype=torch.bfloat16,
                      device="cpu", routing: str = "natural", layer: int = 0,
                      **routing_kw) -> LayerInputs:
    x = make_tokens(seed, N, h, dtype=dtype, device=device, layer=layer)
    w_r = make_router_weight(seed, h, E, dtype=dtype, device=device, layer=layer)
    w_i, w_o = make_expert_weights(seed, E, h, d_ff, dtype=dtype, device=device, layer=layer)
    forced = None if routing == "natural" else draw_experts(seed, N, E, routing, device=device,
                                                            layer=layer, **routing_kw)
    return LayerInputs(x, w_r, w_i, w_o, forced)


# --------------------------------------------------------------------------
# replaced-router draws (the paper's §4.1 experiments and our skewed configs)
# --------------------------------------------------------------------------
def skew_probabilities(E: int, alpha_r: float, k_r: int) -> list:
    """p_i proportional to 1/|E| + alpha_r for the first k_r experts, else 1/|E|.

    PAPER.md:379-385 (§4.1 custom router); the index set "i <= k_r" is read
    1-based, i.e. the first k_r experts (reading R14)."""
    if E < 1 or k_r < 0 or k_r > E or alpha_r < 0:
        raise ValueError(f"skew_probabilities: need E>=1, 0<=k_r<=E, alpha_r>=0 (E={E}, k_r={k_r}, alpha_r={alpha_r})")
    w = [1.0 / E + (alpha_r if i < k_r else 0.0) for i in range(E)]
    s = sum(w)
    return [v / s for v in w]


def zipf_probabilities(E: int, s: float) -> list:
    """p_rank proportional to rank^-s, rank = 1..E (BASELINE.json configs[1])."""
    w = [(r + 1) ** (-s) for r in range(E)]
    tot = sum(w)
    return [v / tot for v in w]


def _expert_permutation(seed: int, E: int, layer: int, device) -> torch.Tensor:
    """Seeded rank->expert-id permutation (reading R15)."""
    keys = _bits_at(seed, STREAM_PERM + 16 * layer, 0x77, torch.arange(E, dtype=torch.int64, device=device))
    return torch.argsort(keys * E + torch.arange(E, device=device))


def draw_experts(seed: int, N: int, E: int, routing: str, *, device="cpu", layer: int = 0,
                 s: float = 1.2, k: int = 1, alpha_r: float = 0.6, k_r: Optional[int] = None,
                 token_offset: int = 0) -> torch.Tensor:
    """Per-token expert ids [N] int32 drawn i.i.d. from the named distribution.

    routing: 'uniform' (iid U{0..E-1}), 'balanced' (exactly N/E per expert,
    seeded shuffle), 'zipf' (Zipf(s) over a seeded permutation of experts),
    'patho' (uniform over k seeded experts), 'skew' (paper §4.1 with alpha_r,
    k_r; default k_r = 10% of E)."""
    idx = torch.arange(token_offset, token_offset + N, dtype=torch.int64, device=device)
    u = uniform_at(seed, STREAM_ROUTE + 16 * layer, idx)
    if routing == "uniform":
        e = torch.clamp((u * E).floor().to(torch.int64), max=E - 1)
        return e.to(torch.int32)
    if routing == "balanced":
        order = torch.argsort(u)
        e = torch.empty(N, dtype=torch.int64, device=device)
        e[order] = torch.arange(N, device=device) % E
        return e.to(torch.int32)
    perm = _expert_permutation(seed, E, layer, device)
    if routing == "patho":
        if not 1 <= k <= E:
            raise ValueError("patho routing needs 1 <= k <= E")
        r = torch.clamp((u * k).floor().to(torch.int64), max=k - 1)
        return perm[r].to(torch.int32)
    if routing == "zipf":
        p = zipf_probabilities(E, s)
    elif routing == "skew":
        p = skew_probabilities(E, alpha_r, k_r if k_r is not None else max(1, round(0.1 * E)))
        perm = torch.arange(E, device=device)  # the paper skews the first k_r experts
    else:
        raise ValueError(f"unknown routing {routing!r}")
    cdf = torch.tensor(p, dtype=torch.float64, device=device).cumsum(0)
    cdf[-1] = 1.0
    r = torch.clamp(torch.searchsorted(cdf, u, right=True), max=E - 1)
    return perm[r].to(torch.int32)
