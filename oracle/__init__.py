"""CPU oracle for MoEShard's sharded Switch-MoE layer (arXiv 2503.08467).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product path (``paper_2503_08467_b200``) never imports it and
shares no code with it.

Plain, slow, obviously-correct float64 numpy. Each function cites the
PAPER.md (or SPEC.md) passage it follows. Library primitives used as single
steps: ``np.matmul`` (a dense product), ``np.argsort(kind="stable")`` (a
stable sort), ``np.exp``.

The method reaches exactly - up to rounding
order - the unsharded Switch MoE FFN, so :func:`moe_layer` is that plain
definition written out; :func:`moe_layer_sharded` follows Algorithm 1
 step by step in the paper's notation and is pinned
against :func:`moe_layer` and the pure-Python brute force
:func:`brute_force_layer`.

Readings of the paper (R1-R19) used here:
  R1  activation between W_i and W_o is ReLU;
  R2  y = g_t * FFN(x_t), g_t = softmax(logits_t)[e_t];
  R3  no router bias / temperature / jitter, no expert biases;
  R4  argmax ties -> lowest expert index;
  R12 error metric max|y - y_ref| / max|y_ref|;
  R20 expert-parallel baseline: capacity ceil(CF n / |E|), CF = min(|E|, 50),
      first-come admission per GPU, dropped tokens give a zero MoE output;
  R21 top-k routing ("typically one or two" experts per token): the k
      largest logits, ordered by logit then lowest index, gate g_tj = softmax(l_t)[e_tj]
      (not renormalised: k = 1 is R2), y_t = sum_j g_tj FFN_{e_tj}(x_t).

Parity status: every function below is pinned by a ``-m "not gpu"`` test in
tests/test_oracle.py (worked examples under tests/golden/, closed forms,
invariants, brute force). None is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "route", "group_per_expert", "expert_ffn", "moe_layer", "moe_layer_tokens",
    "moe_layer_sharded", "brute_force_layer", "shard_plan", "extract_shard",
    "transfer_entries", "shard_storage_entries", "scatter_payload_bytes",
    "macs_per_rank", "max_abs_rel", "routing_margin", "Routing",
    "ep_capacity", "ep_admit", "moe_layer_ep",
    "route_topk", "routing_margin_topk", "moe_layer_topk", "brute_force_layer_topk",
]


def _f64(a) -> np.ndarray:
    if hasattr(a, "detach"):  # torch tensor -> exact widening to float64
        a = a.detach().cpu()
        if a.is_floating_point():
            a = a.double()
        a = a.numpy()
    return np.asarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# Step 1: token routing
# ---------------------------------------------------------------------------
@dataclass
class Routing:
    expert: np.ndarray   # m_expert, int64 [T]
    gate: np.ndarray     # g_t = softmax(l_t)[e_t], float64 [T]
    logits: np.ndarray   # l_t, float64 [T, E]


def route(x, w_r, forced: Optional[Sequence[int]] = None) -> Routing:
    """m_expert <- router(x).

    l_t[e] = sum_k x[t,k] W_r[k,e]; e_t = lowest index attaining max_e l_t[e]
    (R4); g_t = 1 / sum_e exp(l_t[e] - l_t[e_t]) = softmax(l_t)[e_t] (R2).
    With ``forced`` (the paper's replaced router) e_t is
    taken from the input and g_t is still softmax(l_t)[e_t]."""
    x = _f64(x)
    w_r = _f64(w_r)
    if x.ndim != 2 or w_r.ndim != 2 or x.shape[1] != w_r.shape[0]:
        raise ValueError(f"route: shape mismatch x{tuple(x.shape)} vs W_r{tuple(w_r.shape)}")
    logits = x @ w_r
    E = w_r.shape[1]
    if forced is None:
        expert = np.argmax(logits, axis=1).astype(np.int64)  # first maximal index
    else:
        expert = np.asarray(forced, dtype=np.int64).reshape(-1)
        if expert.shape[0] != x.shape[0]:
            raise ValueError("route: forced expert length != token count")
        if expert.size and (expert.min() < 0 or expert.max() >= E):
            raise IndexError("route: forced expert id out of range")
    T = x.shape[0]
    l_e = logits[np.arange(T), expert] if T else np.zeros(0)
    gate = 1.0 / np.exp(logits - l_e[:, None]).sum(axis=1) if T else np.zeros(0)
    return Routing(expert, gate, logits)


def routing_margin(logits: np.ndarray) -> np.ndarray:
    """Gap between the largest and second-largest logit per token (inf if E=1)."""
    if logits.shape[1] < 2:
        return np.full(logits.shape[0], np.inf)
    s = np.sort(logits, axis=1)
    return s[:, -1] - s[:, -2]


# ---------------------------------------------------------------------------
# Step 2: groupPerExpert / countPerExpert
# ---------------------------------------------------------------------------
def group_per_expert(expert, E: int):
    """I_exp and m_sizes.

    Returns (counts [E], offsets [E+1], perm [T]) where perm lists token ids
    grouped by expert, ascending token id inside each group (stable), so
    tokens perm[offsets[e]:offsets[e+1]] are I_exp[e] and counts = m_sizes."""
    expert = np.asarray(expert, dtype=np.int64).reshape(-1)
    if expert.size and (expert.min() < 0 or expert.max() >= E):
        raise IndexError("group_per_expert: expert id out of range")
    counts = np.bincount(expert, minlength=E).astype(np.int64)
    offsets = np.zeros(E + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    perm = np.argsort(expert, kind="stable").astype(np.int64)
    return counts, offsets, perm


# ---------------------------------------------------------------------------
# Expert FFN and expert sharding
# ---------------------------------------------------------------------------
def expert_ffn(x, w_i, w_o) -> np.ndarray:
    """x . W_i -> ReLU (R1) -> . W_o  (Fig. 2a)."""
    x, w_i, w_o = _f64(x), _f64(w_i), _f64(w_o)
    if x.shape[1] != w_i.shape[0] or w_i.shape[1] != w_o.shape[0] or w_o.shape[1] != x.shape[1]:
        raise ValueError(f"expert_ffn: shape mismatch x{x.shape} W_i{w_i.shape} W_o{w_o.shape}")
    return np.maximum(x @ w_i, 0.0) @ w_o


def shard_plan(d_ff: int, G: int) -> List[tuple]:
    """Contiguous equal column ranges of W_i (= row ranges of W_o) per GPU.

    PAPER.md:302-308 ("GPU 0 loads the first two columns ..."), divisibility
    assumption PAPER.md:169, 329-330."""
    if G < 1:
        raise ValueError("shard_plan: G must be >= 1")
    if d_ff % G:
        raise ValueError(f"shard_plan: d_ff={d_ff} not divisible by G={G}")
    F = d_ff // G
    return [(g * F, (g + 1) * F) for g in range(G)]


def extract_shard(w_i, w_o, g: int, G: int):
    """(W_i^g, W_o^g): columns of W_i and rows of W_o in GPU g's range."""
    w_i, w_o = _f64(w_i), _f64(w_o)
    plan = shard_plan(w_i.shape[-1], G)
    if not 0 <= g < G:
        raise IndexError(f"extract_shard: rank {g} out of range for G={G}")
    c0, c1 = plan[g]
    return w_i[..., :, c0:c1], w_o[..., c0:c1, :]


def transfer_entries(c: int, h: int, G: int, split: str) -> int:
    """Entries each GPU sends in the first exchange.

    column-wise W_i: c*h*(G-1); row-wise W_i: c*h*(G-1)/G."""
    if split == "column":
        return c * h * (G - 1)
    if split == "row":
        return c * h * (G - 1) // G
    raise ValueError(split)


def shard_storage_entries(h: int, d_ff: int, G: int) -> int:
    """Entries of W_i (and of W_o) stored per GPU: h*d_ff/G."""
    shard_plan(d_ff, G)
    return h * d_ff // G


def scatter_payload_bytes(b: int, s: int, h: int, bytes_per_elt: int) -> int:
    """Bytes one GPU sends to one peer in Step 3: b*s*h*bytes."""
    return b * s * h * bytes_per_elt


def macs_per_rank(n_tokens_total: int, h: int, d_ff: int, G: int) -> int:
    """Expert MACs executed by each GPU (both products): 2*N*h*d_ff/G.

    Every GPU runs every token through its shard,
    independent of the routing."""
    shard_plan(d_ff, G)
    return 2 * n_tokens_total * h * (d_ff // G)


# ---------------------------------------------------------------------------
# the whole layer, unsharded (the plain definition)
# ---------------------------------------------------------------------------
def moe_layer(x, w_r, w_i, w_o, forced=None, return_routing: bool = False):
    """Top-1 Switch MoE FFN, y_t = g_t * relu(x_t W_i^{e_t}) W_o^{e_t}.

    x [T,h]; W_r [h,E]; W_i [E,h,d_ff]; W_o [E,d_ff,h]. Experts are applied
    to their token groups (Step 2's I_exp) with one product per expert."""
    x = _f64(x)
    w_i, w_o = _f64(w_i), _f64(w_o)
    E = w_i.shape[0]
    rt = route(x, w_r, forced)
    counts, offsets, perm = group_per_expert(rt.expert, E)
    y = np.zeros_like(x)
    for e in range(E):
        rows = perm[offsets[e]:offsets[e + 1]]
        if rows.size == 0:
            continue
        y[rows] = rt.gate[rows, None] * expert_ffn(x[rows], w_i[e], w_o[e])
    if return_routing:
        return y, rt, counts, offsets, perm
    return y


def moe_layer_tokens(x_rows, w_r, expert_weights, forced_rows=None):
    """The layer on a sample of tokens only (full-size parity checks).

    ``expert_weights(e) -> (W_i^e [h,d_ff], W_o^e [d_ff,h])`` supplies the
    weights of one expert on demand, so only the experts the sample routes
    to are materialised."""
    x = _f64(x_rows)
    rt = route(x, w_r, forced_rows)
    y = np.zeros_like(x)
    for e in np.unique(rt.expert):
        rows = np.nonzero(rt.expert == e)[0]
        wi, wo = expert_weights(int(e))
        y[rows] = rt.gate[rows, None] * expert_ffn(x[rows], wi, wo)
    return y, rt


# ---------------------------------------------------------------------------
# top-k routing (R21)                    PAPER.md:85 ("typically one or two")
# ---------------------------------------------------------------------------
def route_topk(x, w_r, k: int, forced=None) -> Routing:
    """Step 1 with k experts per token (R21): expert [T,k] = the k largest logits in
    descending order (ties: lowest index first), gate [T,k] = softmax(l_t)[e_tj]. With
    ``forced`` [T,k] the experts are taken from the input (gates still softmax(l_t)[e])."""
    x, w_r = _f64(x), _f64(w_r)
    if x.ndim != 2 or w_r.ndim != 2 or x.shape[1] != w_r.shape[0]:
        raise ValueError(f"route_topk: shape mismatch x{tuple(x.shape)} vs W_r{tuple(w_r.shape)}")
    E = w_r.shape[1]
    if not 1 <= k <= E:
        raise ValueError(f"route_topk: k={k} not in [1, E={E}]")
    logits = x @ w_r
    T = x.shape[0]
    if forced is None:
        # stable sort of -logit: equal logits keep ascending expert order
        order = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int64)
    else:
        order = np.asarray(forced, dtype=np.int64).reshape(T, k)
        if order.size and (order.min() < 0 or order.max() >= E):
            raise IndexError("route_topk: forced expert id out of range")
    top = np.take_along_axis(logits, order, axis=1)
    m = logits.max(axis=1, keepdims=True) if T else np.zeros((0, 1))
    z = np.exp(logits - m).sum(axis=1, keepdims=True) if T else np.ones((0, 1))
    gate = np.exp(top - m) / z
    return Routing(order, gate, logits)


def routing_margin_topk(logits: np.ndarray, k: int) -> np.ndarray:
    """Smallest gap between consecutive logits among the k + 1 largest of each token (the
    expert set and its order are decided at these gaps; inf when E <= 1)."""
    E = logits.shape[1]
    if E < 2:
        return np.full(logits.shape[0], np.inf)
    s = -np.sort(-logits, axis=1)[:, :min(k + 1, E)]
    return np.min(s[:, :-1] - s[:, 1:], axis=1)


def moe_layer_topk(x, w_r, w_i, w_o, k: int, return_routing: bool = False, forced=None):
    """Top-k MoE FFN (R21): y_t = sum_j g_tj relu(x_t W_i^{e_tj}) W_o^{e_tj}.

    The k (token, expert) assignments of token t are numbered a = t k + j; Step 2 groups
    the assignments per expert (stable in a), each expert runs once over its group, and the
    results are summed per token. Returns (y, routing, counts, offsets, perm over a)."""
    x = _f64(x)
    w_i, w_o = _f64(w_i), _f64(w_o)
    E = w_i.shape[0]
    rt = route_topk(x, w_r, k, forced)
    counts, offsets, perm = group_per_expert(rt.expert.reshape(-1), E)
    y = np.zeros_like(x)
    g = rt.gate.reshape(-1)
    for e in range(E):
        a = perm[offsets[e]:offsets[e + 1]]
        if a.size == 0:
            continue
        t = a // k
        np.add.at(y, t, g[a, None] * expert_ffn(x[t], w_i[e], w_o[e]))
    if return_routing:
        return y, rt, counts, offsets, perm
    return y


def brute_force_layer_topk(x, w_r, w_i, w_o, k: int):
    """Per token, pure Python: logits by explicit sums, the k largest by repeated scans
    (strictly larger wins, so ties keep the lowest index), explicit FFN loops, summed."""
    import math
    x = _f64(x).tolist()
    w_r = _f64(w_r).tolist()
    w_i = _f64(w_i).tolist()
    w_o = _f64(w_o).tolist()
    T, h = len(x), len(x[0]) if x else 0
    E = len(w_i)
    d_ff = len(w_i[0][0]) if E else 0
    out = []
    for t in range(T):
        logits = [sum(x[t][kk] * w_r[kk][e] for kk in range(h)) for e in range(E)]
        chosen = []
        for _ in range(k):
            best = -1
            for e in range(E):
                if e in chosen:
                    continue
                if best < 0 or logits[e] > logits[best]:
                    best = e
            chosen.append(best)
        m = logits[chosen[0]]
        z = sum(math.exp(logits[e] - m) for e in range(E))
        row = [0.0] * h
        for e in chosen:
            g = math.exp(logits[e] - m) / z
            hid = [max(0.0, sum(x[t][kk] * w_i[e][kk][j] for kk in range(h))) for j in range(d_ff)]
            for c in range(h):
                row[c] += g * sum(hid[j] * w_o[e][j][c] for j in range(d_ff))
        out.append(row)
    return np.array(out, dtype=np.float64).reshape(T, h)


# ---------------------------------------------------------------------------
# Algorithm 1, step by step, with G simulated GPUs
# ---------------------------------------------------------------------------
def moe_layer_sharded(x_per_gpu: Sequence, w_r, w_i, w_o, forced_per_gpu=None, stats=None):
    """MoEShard forward for all GPUs g in G; returns the list of per-GPU outputs.

    x_per_gpu[g] is GPU g's [n_g, h] input. Each GPU g holds (W_i^g, W_o^g)
    for all experts. ``stats`` (dict) receives per-GPU MAC
    counts and token counts for the invariance pins."""
    G = len(x_per_gpu)
    xs = [_f64(x) for x in x_per_gpu]
    w_i, w_o = _f64(w_i), _f64(w_o)
    E = w_i.shape[0]
    shard_plan(w_i.shape[2], G)

    # Step 1: token routing (router replicated, run locally)
    routings = [route(xs[g], w_r, None if forced_per_gpu is None else forced_per_gpu[g])
                for g in range(G)]
    # Step 2: I_exp <- groupPerExpert; m_sizes <- countPerExpert; exchange
    I_exp, m_sizes = [], []
    for g in range(G):
        counts, offsets, perm = group_per_expert(routings[g].expert, E)
        I_exp.append((offsets, perm))
        m_sizes.append(counts)
    m_sizes_recv = np.stack(m_sizes)                       # m'_sizes[g][e], same on every GPU
    # Step 3: scatter tokens: every GPU receives W[g][e] from every GPU g
    def inbox(g, e):
        offsets, perm = I_exp[g]
        rows = perm[offsets[e]:offsets[e + 1]]
        assert rows.size == m_sizes_recv[g, e]
        return rows, xs[g][rows]
    # Step 4: expert computation on every GPU r with its shard (W_i^r, W_o^r)
    partial = [[np.zeros_like(xs[g]) for g in range(G)] for _r in range(G)]  # partial[r][g]
    macs = [0] * G
    for r in range(G):
        wi_r, wo_r = extract_shard(w_i, w_o, r, G)
        for g in range(G):
            for e in range(E):
                rows, tokens = inbox(g, e)
                if rows.size == 0:
                    continue
                out = np.maximum(tokens @ wi_r[e], 0.0) @ wo_r[e]
                macs[r] += 2 * rows.size * wi_r.shape[1] * wi_r.shape[2]
                partial[r][g][rows] = routings[g].gate[rows, None] * out
    # Step 5: gather tokens: GPU g receives y[g] from every r and aggregates
    outputs = []
    for g in range(G):
        acc = np.zeros_like(xs[g])
        for r in range(G):           # ascending rank
            acc = acc + partial[r][g]
        outputs.append(acc)
    if stats is not None:
        stats["macs_per_rank"] = macs
        stats["m_sizes"] = m_sizes_recv
        stats["tokens_per_rank"] = [sum(int(m_sizes_recv[g].sum()) for g in range(G))] * G
    return outputs


# ---------------------------------------------------------------------------
# Expert-parallel baseline (the paper's comparison system)
#   PAPER.md:153-161 (EP forward), 393-398 (DeepSpeed baseline, CF = min(|E|, 50))
# ---------------------------------------------------------------------------
def ep_capacity(n_tokens: int, E: int, capacity_factor=None) -> int:
    """Tokens each expert admits from one GPU's minibatch: ceil(CF * n / |E|), with the
    paper's CF = min(|E|, 50) by default (reading R20)."""
    cf = min(E, 50) if capacity_factor is None else capacity_factor
    return int(np.ceil(cf * n_tokens / E))


def ep_admit(expert, E: int, capacity: int) -> np.ndarray:
    """First-come admission inside one GPU's minibatch: token t is kept iff fewer than
    `capacity` earlier tokens (in token order) chose the same expert (R20)."""
    expert = np.asarray(expert, dtype=np.int64).reshape(-1)
    seen = np.zeros(E, dtype=np.int64)
    keep = np.zeros(expert.shape[0], dtype=bool)
    for t, e in enumerate(expert.tolist()):
        keep[t] = seen[e] < capacity
        seen[e] += 1
    return keep


def moe_layer_ep(x_per_gpu: Sequence, w_r, w_i, w_o, capacity_factor=None, forced_per_gpu=None,
                 stats=None):
    """Expert parallelism, step by step: the router is replicated and each
    GPU routes its own minibatch; GPU o hosts the |E|/|G| whole experts
    [o*|E|/|G|, (o+1)*|E|/|G|); an all-to-all scatter sends every admitted token to the GPU
    hosting its expert, which computes it with the full expert; an all-to-all gather returns
    the results, scaled by the gate. A token beyond its expert's capacity (first-come per
    GPU, ep_admit) is dropped: its MoE output is zero (the residual carries it, R20).

    Returns the per-GPU outputs; ``stats`` receives per-GPU received-token counts, MACs and
    the dropped-token count."""
    G = len(x_per_gpu)
    xs = [_f64(x) for x in x_per_gpu]
    w_i, w_o = _f64(w_i), _f64(w_o)
    E = w_i.shape[0]
    if E % G:
        raise ValueError(f"moe_layer_ep: |E|={E} not divisible by |G|={G}")
    E_loc = E // G
    routings = [route(xs[g], w_r, None if forced_per_gpu is None else forced_per_gpu[g])
                for g in range(G)]
    keeps = [ep_admit(routings[g].expert, E, ep_capacity(xs[g].shape[0], E, capacity_factor))
             for g in range(G)]
    # all-to-all scatter: inbox[o] = (source GPU, token index) pairs of o's experts
    inbox = [[] for _ in range(G)]
    for g in range(G):
        for t in np.nonzero(keeps[g])[0].tolist():
            inbox[int(routings[g].expert[t]) // E_loc].append((g, t))
    outputs = [np.zeros_like(xs[g]) for g in range(G)]
    macs = [0] * G
    for o in range(G):                     # expert computation on the hosting GPU
        for g, t in inbox[o]:
            e = int(routings[g].expert[t])
            y = expert_ffn(xs[g][t:t + 1], w_i[e], w_o[e])[0]
            outputs[g][t] = routings[g].gate[t] * y   # all-to-all gather back to GPU g
            macs[o] += 2 * w_i.shape[1] * w_i.shape[2]
    if stats is not None:
        stats["tokens_per_rank"] = [len(inbox[o]) for o in range(G)]
        stats["macs_per_rank"] = macs
        stats["dropped"] = int(sum((~k).sum() for k in keeps))
        stats["keep"] = keeps
    return outputs


# ---------------------------------------------------------------------------
# brute force: a dense per-token loop with no grouping (pure Python, tiny only)
# ---------------------------------------------------------------------------
def brute_force_layer(x, w_r, w_i, w_o, forced=None):
    """Per token: logits by explicit sums, argmax by scan, FFN by explicit loops."""
    x = _f64(x).tolist()
    w_r = _f64(w_r).tolist()
    w_i = _f64(w_i).tolist()
    w_o = _f64(w_o).tolist()
    T, h = len(x), len(x[0]) if x else 0
    E = len(w_i)
    d_ff = len(w_i[0][0]) if E else 0
    out = []
    import math
    for t in range(T):
        logits = [sum(x[t][k] * w_r[k][e] for k in range(h)) for e in range(E)]
        if forced is None:
            best = 0
            for e in range(1, E):
                if logits[e] > logits[best]:
                    best = e
        else:
            best = int(forced[t])
        z = sum(math.exp(logits[e] - logits[best]) for e in range(E))
        g = 1.0 / z
        hid = [max(0.0, sum(x[t][k] * w_i[best][k][j] for k in range(h))) for j in range(d_ff)]
        out.append([g * sum(hid[j] * w_o[best][j][c] for j in range(d_ff)) for c in range(h)])
    return np.array(out, dtype=np.float64).reshape(T, h)


def max_abs_rel(y, y_ref) -> float:
    """R12: max_{t,j} |y - y_ref| / max_{t,j} |y_ref| (0 if both empty/zero)."""
    y, y_ref = _f64(y), _f64(y_ref)
    if y.shape != y_ref.shape:
        raise ValueError(f"max_abs_rel: shape mismatch {y.shape} vs {y_ref.shape}")
    if y.size == 0:
        return 0.0
    den = float(np.max(np.abs(y_ref)))
    num = float(np.max(np.abs(y - y_ref)))
    if den == 0.0:
        return num
    return num / den
