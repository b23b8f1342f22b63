"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test names the passage or property it checks. Chosen so that a
plausible slip in the oracle (dropped gate factor, wrong softmax sign,
transposed operand, unstable grouping, wrong shard slice, missing ReLU,
wrong tie-break) fails at least one of them.
"""
import math

import numpy as np
import pytest

import oracle as O

rng = np.random.default_rng(12345)


def _rand_layer(T, h, d_ff, E, seed=0):
    r = np.random.default_rng(seed)
    x = r.standard_normal((T, h))
    w_r = r.standard_normal((h, E)) / math.sqrt(h)
    w_i = r.standard_normal((E, h, d_ff)) / math.sqrt(h)
    w_o = r.standard_normal((E, d_ff, h)) / math.sqrt(d_ff)
    return x, w_r, w_i, w_o


# ----------------------------------------------------------------- Step 1 router
def test_router_worked_example(golden):
    g = golden("router_worked_example.json")
    rt = O.route(np.array(g["x"]), np.array(g["w_r"]))
    assert rt.expert.tolist() == g["expert"]
    assert rt.gate[0] == pytest.approx(g["gate"][0], abs=1e-15)
    # independent closed form: logistic(5)
    assert rt.gate[0] == pytest.approx(1.0 / (1.0 + math.exp(-5.0)), abs=1e-15)


def test_router_all_zero_gate_goes_to_expert0_with_gate_1_over_E():
    # tie everywhere -> lowest index, softmax uniform
    E = 7
    rt = O.route(rng.standard_normal((11, 5)), np.zeros((5, E)))
    assert (rt.expert == 0).all()
    np.testing.assert_allclose(rt.gate, 1.0 / E, rtol=0, atol=1e-15)


def test_router_single_expert_gate_is_one():
    # SPEC.md:132
    rt = O.route(rng.standard_normal((9, 4)), rng.standard_normal((4, 1)))
    assert (rt.expert == 0).all()
    np.testing.assert_array_equal(rt.gate, 1.0)


def test_router_tie_break_lowest_index():
    # R4: columns 1 and 3 identical and maximal -> expert 1
    w_r = np.array([[0.0, 2.0, -1.0, 2.0], [0.0, 1.0, 0.5, 1.0]])
    x = np.array([[1.0, 1.0], [3.0, -1.0]])
    rt = O.route(x, w_r)
    assert rt.expert.tolist() == [1, 1]


def test_router_argmax_invariant_to_positive_scaling():
    # SPEC.md:153 (softmax argmax invariance)
    x, w_r, _, _ = _rand_layer(200, 8, 4, 6, seed=3)
    a = O.route(x, w_r).expert
    b = O.route(x, 3.7 * w_r).expert
    np.testing.assert_array_equal(a, b)


def test_router_gate_is_softmax_probability_of_chosen_expert():
    # independent: softmax by explicit normalisation, not the oracle's formula
    x, w_r, _, _ = _rand_layer(50, 6, 4, 5, seed=4)
    rt = O.route(x, w_r)
    for t in range(50):
        l = [sum(x[t, k] * w_r[k, e] for k in range(6)) for e in range(5)]
        z = [math.exp(v) for v in l]
        p = [v / sum(z) for v in z]
        best = max(range(5), key=lambda e: (l[e], -e))
        assert rt.expert[t] == best
        assert rt.gate[t] == pytest.approx(p[best], rel=1e-12)
    forced = [(t * 3) % 5 for t in range(50)]
    rf = O.route(x, w_r, forced)
    for t in range(50):
        l = [sum(x[t, k] * w_r[k, e] for k in range(6)) for e in range(5)]
        z = [math.exp(v) for v in l]
        assert rf.gate[t] == pytest.approx(z[forced[t]] / sum(z), rel=1e-12)


def test_routing_margin_worked_cases(golden):
    g = golden("routing_margin.json")
    for c in g["cases"]:
        want = [np.inf if v == "inf" else v for v in c["margin"]]
        np.testing.assert_array_equal(O.routing_margin(np.array(c["logits"])), want)
    # SPEC.md:130 example: two experts, gate g printed -> margin = log(g / (1 - g)) = 5
    gate = g["spec_gate"]
    rt = O.route(np.array([[5.0, 0.0]]), np.eye(2))
    assert abs(O.routing_margin(rt.logits)[0] - np.log(gate / (1 - gate))) < 1e-12


def test_routing_margin_brute_force_and_invariances():
    """Against a pure-Python pairwise definition (max over e of l_e minus max over the
    others), and invariant to permuting experts and to a common shift of the logits."""
    rng = np.random.default_rng(3)
    L = rng.normal(size=(50, 9))
    top = L.max(axis=1)[::7] + 1.0
    L[::7, 2] = top                             # exact ties for the maximum on some rows
    L[::7, 4] = top
    want = []
    for row in L.tolist():
        best = max(range(len(row)), key=lambda e: (row[e], -e))
        want.append(row[best] - max(v for e, v in enumerate(row) if e != best))
    np.testing.assert_array_equal(O.routing_margin(L), np.array(want))
    perm = rng.permutation(9)
    np.testing.assert_array_equal(O.routing_margin(L[:, perm]), O.routing_margin(L))
    np.testing.assert_allclose(O.routing_margin(L + 3.5), O.routing_margin(L), atol=1e-12)
    assert (O.routing_margin(L)[::7] == 0).all()


def test_router_shape_and_bounds_errors():
    with pytest.raises(ValueError):
        O.route(np.zeros((3, 4)), np.zeros((5, 2)))
    with pytest.raises(IndexError):
        O.route(np.zeros((2, 4)), np.zeros((4, 2)), forced=[0, 2])


# ----------------------------------------------------------------- Step 2 grouping
def test_grouping_worked_example(golden):
    g = golden("grouping_example.json")
    counts, offsets, perm = O.group_per_expert(g["m_expert"], g["E"])
    assert counts.tolist() == g["counts"]
    assert perm.tolist() == g["perm"]
    assert offsets.tolist() == [0, 3, 3, 4, 4]


def test_grouping_is_stable_permutation_and_inverts():
    e = rng.integers(0, 9, size=1000)
    counts, offsets, perm = O.group_per_expert(e, 9)
    assert counts.sum() == 1000
    assert sorted(perm.tolist()) == list(range(1000))           # bijection
    for k in range(9):
        seg = perm[offsets[k]:offsets[k + 1]]
        assert (e[seg] == k).all()
        assert (np.diff(seg) > 0).all()                          # stable: ascending token id
    x = rng.standard_normal((1000, 3))
    grouped = x[perm]
    back = np.empty_like(grouped)
    back[perm] = grouped                                         # ungroup(group(x)) == x
    np.testing.assert_array_equal(back, x)


def test_grouping_bounds_error():
    with pytest.raises(IndexError):
        O.group_per_expert([0, 4], 4)


# ----------------------------------------------------------------- expert FFN
def test_identity_expert(golden):
    g = golden("identity_expert.json")
    y = O.expert_ffn(np.array(g["x"]), np.array(g["w_i"]), np.array(g["w_o"]))
    np.testing.assert_array_equal(y, np.array(g["y"]))
    np.testing.assert_array_equal(O.expert_ffn(np.zeros((3, 2)), np.eye(2), np.eye(2)), 0.0)


def test_expert_ffn_matches_explicit_loops_and_uses_relu():
    x, _, w_i, w_o = _rand_layer(5, 4, 6, 1, seed=5)
    y = O.expert_ffn(x, w_i[0], w_o[0])
    for t in range(5):
        hid = [max(0.0, sum(x[t, k] * w_i[0, k, j] for k in range(4))) for j in range(6)]
        for c in range(4):
            assert y[t, c] == pytest.approx(sum(hid[j] * w_o[0, j, c] for j in range(6)), abs=1e-12)
    # without the ReLU the answer differs (guards a dropped activation)
    assert not np.allclose(y, x @ w_i[0] @ w_o[0])


# ----------------------------------------------------------------- sharding plan
def test_shard_plan_examples(golden):
    for case in golden("shard_plan_examples.json")["cases"]:
        if "error" in case:
            with pytest.raises(ValueError):
                O.shard_plan(case["d_ff"], case["G"])
        else:
            assert [list(r) for r in O.shard_plan(case["d_ff"], case["G"])] == case["ranges"]


def test_extract_shard_reassembles_exactly():
    _, _, w_i, w_o = _rand_layer(1, 6, 8, 3, seed=6)
    for G in (1, 2, 4, 8):
        parts = [O.extract_shard(w_i, w_o, g, G) for g in range(G)]
        np.testing.assert_array_equal(np.concatenate([p[0] for p in parts], axis=2), w_i)
        np.testing.assert_array_equal(np.concatenate([p[1] for p in parts], axis=1), w_o)
    # Fig. 2b: GPU 1 of 2 holds the second half of W_i's columns / W_o's rows
    wi1, wo1 = O.extract_shard(w_i, w_o, 1, 2)
    np.testing.assert_array_equal(wi1, w_i[:, :, 4:8])
    np.testing.assert_array_equal(wo1, w_o[:, 4:8, :])
    with pytest.raises(IndexError):
        O.extract_shard(w_i, w_o, 2, 2)


def test_byte_and_entry_counts(golden):
    g = golden("byte_counts.json")
    s = g["scatter"]
    nbytes = O.scatter_payload_bytes(s["b"], s["s"], s["h"], s["bytes_per_elt"])
    assert nbytes == s["payload_bytes"]
    assert round(nbytes / 2**20) == s["payload_mib_approx"]
    for c in g["transfer"]:
        assert O.transfer_entries(c["c"], c["h"], c["G"], c["split"]) == c["entries"]
    for G in (1, 2, 4, 8):          # column split = G x row split
        assert O.transfer_entries(16, 8, G, "column") == G * O.transfer_entries(16, 8, G, "row")
    st = g["storage"]
    assert O.shard_storage_entries(st["h"], st["d_ff"], st["G"]) == st["entries"]
    assert O.shard_storage_entries(st["h"], st["d_ff"], st["G"]) * st["G"] == st["h"] * st["d_ff"]
    t = g["time"]
    ms = t["mib"] * 2**20 / (t["gib_per_s"] * 2**30) * 1e3
    assert abs(ms - t["ms_approx"]) < 0.01


# ----------------------------------------------------------------- whole layer
@pytest.mark.parametrize("T,h,d_ff,E", [(1, 3, 4, 1), (17, 8, 12, 3), (40, 16, 64, 8), (64, 12, 32, 5)])
def test_layer_matches_brute_force(T, h, d_ff, E):
    x, w_r, w_i, w_o = _rand_layer(T, h, d_ff, E, seed=T + E)
    y = O.moe_layer(x, w_r, w_i, w_o)
    yb = O.brute_force_layer(x, w_r, w_i, w_o)
    np.testing.assert_allclose(y, yb, rtol=0, atol=1e-12 * max(1.0, np.abs(yb).max()))
    forced = [(3 * t + 1) % E for t in range(T)]
    yf = O.moe_layer(x, w_r, w_i, w_o, forced=forced)
    ybf = O.brute_force_layer(x, w_r, w_i, w_o, forced=forced)
    np.testing.assert_allclose(yf, ybf, rtol=0, atol=1e-12 * max(1.0, np.abs(ybf).max()))


def test_single_expert_reduces_to_dense_t5_ffn():
    # E=1 -> gate 1, the layer is relu(x W_i) W_o (textbook T5 v1.0 FFN)
    x, w_r, w_i, w_o = _rand_layer(30, 8, 16, 1, seed=9)
    y = O.moe_layer(x, w_r, w_i, w_o)
    dense = O.brute_force_layer(x, w_r, w_i, w_o)
    np.testing.assert_allclose(y, dense, atol=1e-12)


def test_layer_zero_experts_give_zero_and_all_tokens_kept():
    x, w_r, w_i, w_o = _rand_layer(50, 8, 16, 4, seed=10)
    np.testing.assert_array_equal(O.moe_layer(x, w_r, 0 * w_i, w_o), 0.0)
    y, rt, counts, offsets, perm = O.moe_layer(x, w_r, w_i, w_o, return_routing=True)
    assert counts.sum() == 50                                   # droplessness
    assert (np.abs(y).sum(axis=1) > 0).all()                    # every token got its expert output


def test_layer_token_permutation_equivariance_and_expert_relabelling():
    x, w_r, w_i, w_o = _rand_layer(60, 8, 16, 6, seed=11)
    y = O.moe_layer(x, w_r, w_i, w_o)
    p = rng.permutation(60)
    np.testing.assert_allclose(O.moe_layer(x[p], w_r, w_i, w_o), y[p], atol=1e-13)
    q = rng.permutation(6)
    np.testing.assert_allclose(O.moe_layer(x, w_r[:, q], w_i[q], w_o[q]), y, atol=1e-13)


def test_layer_tokens_sample_matches_full_layer():
    x, w_r, w_i, w_o = _rand_layer(80, 8, 16, 5, seed=12)
    y = O.moe_layer(x, w_r, w_i, w_o)
    rows = np.array([0, 7, 33, 79])
    ys, rt = O.moe_layer_tokens(x[rows], w_r, lambda e: (w_i[e], w_o[e]))
    np.testing.assert_allclose(ys, y[rows], atol=1e-14)


# ----------------------------------------------------------------- Algorithm 1 sharded
@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("routing", ["natural", "skewed"])
def test_sharded_alg1_equals_unsharded(G, routing):
    # summing y_g over GPUs yields the unsharded output
    n, h, d_ff, E = 24, 12, 32, 8
    x, w_r, w_i, w_o = _rand_layer(n * G, h, d_ff, E, seed=20 + G)
    forced = None
    if routing == "skewed":
        forced = np.where(rng.random(n * G) < 0.9, 2, rng.integers(0, E, n * G))
    y = O.moe_layer(x, w_r, w_i, w_o, forced=forced)
    stats = {}
    outs = O.moe_layer_sharded([x[g * n:(g + 1) * n] for g in range(G)], w_r, w_i, w_o,
                               None if forced is None else [forced[g * n:(g + 1) * n] for g in range(G)],
                               stats=stats)
    got = np.concatenate(outs)
    assert O.max_abs_rel(got, y) <= 1e-12
    # per-GPU work identical whatever the routing
    assert stats["macs_per_rank"] == [O.macs_per_rank(n * G, h, d_ff, G)] * G
    # metadata table: row g is GPU g's m_sizes; column sums are global counts
    np.testing.assert_array_equal(stats["m_sizes"].sum(axis=0),
                                  np.bincount(O.route(x, w_r, forced).expert, minlength=E))


def test_sharded_partials_are_not_individually_the_answer():
    # guards an oracle that would forget to sum partials (Step 5)
    n, h, d_ff, E = 16, 8, 16, 2
    x, w_r, w_i, w_o = _rand_layer(2 * n, h, d_ff, E, seed=30)
    wi0, wo0 = O.extract_shard(w_i, w_o, 0, 2)
    half = O.moe_layer(x, w_r, wi0, wo0)
    assert O.max_abs_rel(half, O.moe_layer(x, w_r, w_i, w_o)) > 1e-3


def test_sharded_divisibility_error():
    x, w_r, w_i, w_o = _rand_layer(8, 4, 6, 2, seed=31)
    with pytest.raises(ValueError):
        O.moe_layer_sharded([x[:2], x[2:4], x[4:6], x[6:]], w_r, w_i, w_o)


def test_max_abs_rel_definition():
    ref = np.array([[1.0, -4.0], [2.0, 0.0]])
    y = ref + np.array([[0.1, 0.0], [0.0, -0.2]])
    assert O.max_abs_rel(y, ref) == pytest.approx(0.2 / 4.0)


# ---------------------------------------------------------------------------
# expert-parallel baseline
# ---------------------------------------------------------------------------
def test_ep_admission_worked_cases(golden):
    for c in golden("ep_admission.json")["cases"]:
        cap = O.ep_capacity(c["n"], c["E"], c["cf"])
        assert cap == c["capacity"]
        np.testing.assert_array_equal(O.ep_admit(c["expert"], c["E"], cap), c["keep"])


def test_ep_paper_cf_never_drops_up_to_50_experts():
    """CF = min(|E|, 50): capacity = n for |E| <= 50, so no routing drops a
    token; above 50 experts the pathological routing drops n - ceil(50 n / |E|)."""
    rng = np.random.default_rng(0)
    for E in (1, 8, 50):
        n = 37
        for expert in (np.zeros(n, int), rng.integers(0, E, n)):
            assert O.ep_admit(expert, E, O.ep_capacity(n, E)).all()
    for E in (64, 128, 256):
        n = 1000
        keep = O.ep_admit(np.zeros(n, int), E, O.ep_capacity(n, E))
        assert (~keep).sum() == n - math.ceil(50 * n / E)


@pytest.mark.parametrize("G,E,routing", [(1, 8, "uniform"), (2, 8, "skew"), (4, 16, "zipf")])
def test_ep_without_drops_equals_unsharded_layer(G, E, routing):
    """With capacity >= n nothing is dropped and EP computes exactly the Switch layer:
    the concatenated per-GPU outputs equal moe_layer (fp64, rounding order only)."""
    import torch
    import workload as W
    n, h, d_ff = 40, 16, 24
    inp = W.make_layer_inputs(5, G * n, h, d_ff, E, dtype=torch.float64, routing=routing, k_r=2)
    xs = [inp.x[g * n:(g + 1) * n] for g in range(G)]
    fs = [inp.forced[g * n:(g + 1) * n].numpy() for g in range(G)]
    st = {}
    ys = O.moe_layer_ep(xs, inp.w_r, inp.w_i, inp.w_o, capacity_factor=E, forced_per_gpu=fs, stats=st)
    y_ref = O.moe_layer(inp.x, inp.w_r, inp.w_i, inp.w_o, forced=inp.forced.numpy())
    np.testing.assert_allclose(np.concatenate(ys), y_ref, rtol=1e-12, atol=1e-12)
    assert st["dropped"] == 0 and sum(st["tokens_per_rank"]) == G * n


def test_ep_matches_brute_force_with_drops():
    """Tiny inputs with a capacity that bites: kept tokens equal the dense per-token brute
    force, dropped tokens are exactly zero, and the kept set is first-come per GPU."""
    import torch
    import workload as W
    G, n, h, d_ff, E = 2, 12, 8, 16, 4
    inp = W.make_layer_inputs(9, G * n, h, d_ff, E, dtype=torch.float64, routing="patho", k=2)
    xs = [inp.x[g * n:(g + 1) * n] for g in range(G)]
    fs = [inp.forced[g * n:(g + 1) * n].numpy() for g in range(G)]
    st = {}
    ys = O.moe_layer_ep(xs, inp.w_r, inp.w_i, inp.w_o, capacity_factor=1.0, forced_per_gpu=fs, stats=st)
    dense = O.brute_force_layer(inp.x, inp.w_r, inp.w_i, inp.w_o, forced=inp.forced.numpy())
    cap = math.ceil(n / E)
    for g in range(G):
        seen = {}
        for t in range(n):
            e = int(fs[g][t])
            kept = seen.get(e, 0) < cap
            seen[e] = seen.get(e, 0) + 1
            assert st["keep"][g][t] == kept
            if kept:
                np.testing.assert_allclose(ys[g][t], dense[g * n + t], rtol=1e-12, atol=1e-12)
            else:
                assert (ys[g][t] == 0).all()
    assert st["dropped"] > 0


def test_ep_per_rank_load_under_pathological_routing():
    """SPEC.md:474-482 contrast: under EP all tokens routed to one expert land on one GPU
    (max/mean load = G), while MoEShard's per-GPU MACs are identical whatever the routing."""
    import torch
    import workload as W
    G, n, h, d_ff, E = 4, 30, 8, 16, 8
    inp = W.make_layer_inputs(11, G * n, h, d_ff, E, dtype=torch.float64, routing="patho", k=1)
    xs = [inp.x[g * n:(g + 1) * n] for g in range(G)]
    fs = [inp.forced[g * n:(g + 1) * n].numpy() for g in range(G)]
    st = {}
    O.moe_layer_ep(xs, inp.w_r, inp.w_i, inp.w_o, capacity_factor=E, forced_per_gpu=fs, stats=st)
    load = np.array(st["tokens_per_rank"])
    assert load.max() == G * n and load.sum() == G * n and load.max() / load.mean() == G
    st2 = {}
    O.moe_layer_sharded(xs, inp.w_r, inp.w_i, inp.w_o, forced_per_gpu=fs, stats=st2)
    assert len(set(st2["macs_per_rank"])) == 1


# ------------------------------------------------------------------ top-k routing (R21)
def test_topk_k1_is_the_top1_layer():
    x, w_r, w_i, w_o = _rand_layer(37, 6, 10, 5, seed=21)
    y1 = O.moe_layer(x, w_r, w_i, w_o)
    yk, rt, counts, offsets, perm = O.moe_layer_topk(x, w_r, w_i, w_o, 1, return_routing=True)
    assert np.max(np.abs(y1 - yk)) <= 1e-12 * max(1.0, np.max(np.abs(y1)))
    r1 = O.route(x, w_r)
    assert np.array_equal(rt.expert[:, 0], r1.expert)
    assert np.allclose(rt.gate[:, 0], r1.gate, rtol=0, atol=1e-15)


def test_topk_all_experts_is_the_dense_softmax_mixture():
    # k = E: every expert, weighted by its softmax probability (a closed form with no routing)
    x, w_r, w_i, w_o = _rand_layer(9, 5, 7, 4, seed=22)
    y = O.moe_layer_topk(x, w_r, w_i, w_o, 4)
    logits = x @ w_r
    p = np.exp(logits - logits.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    ref = np.zeros_like(x)
    for e in range(4):
        ref += p[:, e:e + 1] * (np.maximum(x @ w_i[e], 0.0) @ w_o[e])
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("k", [2, 3])
def test_topk_layer_matches_brute_force(k):
    x, w_r, w_i, w_o = _rand_layer(7, 4, 6, 5, seed=23 + k)
    y = O.moe_layer_topk(x, w_r, w_i, w_o, k)
    ref = O.brute_force_layer_topk(x, w_r, w_i, w_o, k)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_topk_routing_order_ties_gates_and_droplessness():
    # planted logits: token 0 ties experts 1 and 3 at the top, token 1 has a clear order
    x = np.eye(2)
    w_r = np.array([[0.0, 2.0, 1.0, 2.0], [0.5, 3.0, 4.0, -1.0]])
    rt = O.route_topk(x, w_r, 2)
    assert rt.expert.tolist() == [[1, 3], [2, 1]]
    rf = O.route_topk(x, w_r, 2, forced=rt.expert)     # the replaced-router hook
    assert np.array_equal(rf.gate, rt.gate) and np.array_equal(rf.expert, rt.expert)
    for t in range(2):
        l = x[t] @ w_r
        p = np.exp(l - l.max()) / np.exp(l - l.max()).sum()
        assert np.allclose(rt.gate[t], p[rt.expert[t]], rtol=0, atol=1e-15)
        assert rt.gate[t, 0] >= rt.gate[t, 1] and rt.gate[t].sum() <= 1.0
    # every token keeps all k assignments (no capacity): counts sum to T k
    x2, w_r2, w_i2, w_o2 = _rand_layer(50, 6, 8, 6, seed=31)
    _, rt2, counts, _, perm = O.moe_layer_topk(x2, w_r2, w_i2, w_o2, 2, return_routing=True)
    assert counts.sum() == 100 and sorted(perm.tolist()) == list(range(100))
    assert all(len(set(r)) == 2 for r in rt2.expert.tolist())
    m = O.routing_margin_topk(rt2.logits, 2)
    s = -np.sort(-rt2.logits, axis=1)
    assert np.allclose(m, np.minimum(s[:, 0] - s[:, 1], s[:, 1] - s[:, 2]))


def test_topk_expert_shards_sum_to_the_unsharded_layer():
    # the MoEShard identity does not depend on the routing: the layer on
    # each GPU's column / row shard of every expert sums to the unsharded top-2 layer
    x, w_r, w_i, w_o = _rand_layer(40, 8, 16, 6, seed=41)
    full = O.moe_layer_topk(x, w_r, w_i, w_o, 2)
    for G in (2, 4):
        acc = np.zeros_like(full)
        for g in range(G):
            wi_g, wo_g = O.extract_shard(w_i, w_o, g, G)
            acc += O.moe_layer_topk(x, w_r, wi_g, wo_g, 2)
        assert np.max(np.abs(acc - full)) <= 1e-12 * np.max(np.abs(full))
