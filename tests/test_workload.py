"""The seeded input generator (workload/): determinism, slicing, statistics."""
import math

import pytest
import torch

import workload as W


def test_hash_scalar_matches_tensor_path():
    xs = [0, 1, 2, 12345, 0xFFFFFFFF, 0x80000000]
    t = W._hash32(torch.tensor(xs, dtype=torch.int64))
    assert t.tolist() == [W.hash32_int(x) for x in xs]


def test_deterministic_and_slice_consistent():
    a = W.normal_tensor(7, W.STREAM_X, (64, 48))
    b = W.normal_tensor(7, W.STREAM_X, (64, 48))
    assert torch.equal(a, b)
    # generating rows 10..20 on their own gives the same values
    c = W.normal_tensor(7, W.STREAM_X, (10, 48), offset=10 * 48)
    assert torch.equal(c, a[10:20])
    # token generation for a rank's slice equals the slice of the global tensor
    x_all = W.make_tokens(3, 32, 16)
    x_r1 = W.make_tokens(3, 16, 16, token_offset=16)
    assert torch.equal(x_all[16:], x_r1)
    # other seeds / streams differ
    assert not torch.equal(a, W.normal_tensor(8, W.STREAM_X, (64, 48)))
    assert not torch.equal(a, W.normal_tensor(7, W.STREAM_WR, (64, 48)))


def test_expert_weight_shards_are_slices_of_full():
    wi, wo = W.make_expert_weights(5, 3, 8, 16, dtype=torch.float32)
    wi1, wo1 = W.make_expert_weights(5, 3, 8, 16, cols=(8, 16), dtype=torch.float32)
    assert torch.equal(wi[:, :, 8:16], wi1)
    assert torch.equal(wo[:, 8:16, :], wo1)
    wie, woe = W.make_expert_weights(5, 3, 8, 16, dtype=torch.float32, experts=[2])
    assert torch.equal(wie[0], wi[2]) and torch.equal(woe[0], wo[2])


def test_normal_statistics():
    z = W.normal_tensor(1, 9, (200000,), dtype=torch.float64)
    assert abs(z.mean().item()) < 0.01
    assert abs(z.std().item() - 1.0) < 0.01
    # tails behave (Box-Muller on (0,1) open uniforms never yields inf)
    assert torch.isfinite(z).all()
    assert 0.002 < (z.abs() > 3).double().mean().item() < 0.0035   # 2*(1-Phi(3)) = 0.0027


def test_skew_probabilities_golden(golden):
    g = golden("skew_probabilities.json")
    p = W.skew_probabilities(g["E"], g["alpha_r"], g["k_r"])
    assert p == pytest.approx(g["p"], abs=1e-15)
    assert W.skew_probabilities(8, 0.0, 3) == pytest.approx([1 / 8] * 8)
    assert W.skew_probabilities(8, 0.6, 8) == pytest.approx([1 / 8] * 8)
    with pytest.raises(ValueError):
        W.skew_probabilities(4, 0.6, 5)


def test_draw_distributions():
    N, E = 200000, 8
    u = W.draw_experts(1, N, E, "uniform")
    cnt = torch.bincount(u.long(), minlength=E).double() / N
    sigma = math.sqrt((1 / E) * (1 - 1 / E) / N)
    assert (cnt - 1 / E).abs().max().item() < 4 * sigma
    z = W.draw_experts(1, N, 64, "zipf", s=1.2)
    top = torch.bincount(z.long(), minlength=64).max().item() / N
    assert top == pytest.approx(W.zipf_probabilities(64, 1.2)[0], abs=0.005)  # ~0.2925
    p = W.draw_experts(1, 1000, 256, "patho", k=3)
    assert len(set(p.tolist())) == 3
    b = W.draw_experts(1, 1024, 64, "balanced")
    assert torch.bincount(b.long(), minlength=64).tolist() == [16] * 64
    s = W.draw_experts(2, N, 128, "skew", alpha_r=0.6, k_r=13)
    share = (s < 13).double().mean().item()
    p_sk = sum(W.skew_probabilities(128, 0.6, 13)[:13])
    assert abs(share - p_sk) < 4 * math.sqrt(p_sk * (1 - p_sk) / N)
