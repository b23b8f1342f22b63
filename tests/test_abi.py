"""The C-ABI library loads and exports every symbol include/moeshard.h declares;
host-side validation works without a GPU (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moeshard.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moeshard_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2503_08467_b200 import moeshard as C
    lib = ctypes.CDLL(C.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), f"libmoeshard.so does not export {name}"
    assert sorted(C.EXPORTS) == declared


def test_no_torch_types_in_abi():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for bad in ("torch", "at::", "c10", "Tensor", "cudaStream_t", "#include <cuda"):
        assert bad not in src


def test_version_and_status_strings():
    from paper_2503_08467_b200 import moeshard as C
    assert "sm_100a" in C.moeshard_version()
    for code, name in C.STATUS.items():
        assert C._lib.moeshard_status_string(code).decode() == name


def _cfg(**kw):
    from paper_2503_08467_b200 import moeshard as C
    d = dict(d_model=768, d_ff=3072, n_experts=64, n_layers=1, max_tokens_per_rank=1024,
             dtype=C.MOESHARD_BF16, flags=0)
    d.update(kw)
    return C.moeshard_config(**d)


def test_config_validation_errors():
    from paper_2503_08467_b200 import moeshard as C
    with pytest.raises(C.MoEShardError) as ei:
        C.moeshard_workspace_size(_cfg(d_ff=3072), 5)        # 3072 % 5 != 0
    assert ei.value.code == -3 and "divisible" in str(ei.value)
    with pytest.raises(C.MoEShardError) as ei:
        C.moeshard_workspace_size(_cfg(n_experts=0), 1)
    assert ei.value.code == -5
    with pytest.raises(C.MoEShardError) as ei:
        C.moeshard_workspace_size(_cfg(d_model=100), 1)
    assert ei.value.code == -5
    with pytest.raises(C.MoEShardError) as ei:
        C.moeshard_workspace_size(_cfg(dtype=7), 1)
    assert ei.value.code == -1
    with pytest.raises(C.MoEShardError):
        C.moeshard_workspace_size(_cfg(), 0)
    for removed in (0x8, 0x10, 0x20, 0x40, 0x100, 0x400, 0x800, 1 << 20):   # unknown flag bits
        with pytest.raises(C.MoEShardError) as ei:
            C.moeshard_workspace_size(_cfg(flags=removed), 1)
        assert ei.value.code == -1 and "unknown" in str(ei.value)


def test_sizes():
    from paper_2503_08467_b200 import moeshard as C
    for G in (1, 2, 4, 8):
        # 2 * E * h * d_ff/G elements of storage per rank
        assert C.moeshard_weight_storage_size(_cfg(), G) == 2 * 64 * 768 * (3072 // G) * 2
        assert C.moeshard_weight_storage_size(_cfg(dtype=C.MOESHARD_FP32), G) == 2 * 64 * 768 * (3072 // G) * 4
    w1 = C.moeshard_workspace_size(_cfg(), 1)
    w8 = C.moeshard_workspace_size(_cfg(), 8)
    assert w1 > 1024 * 768 * 2 * 2 and w8 > w1   # world 8 holds 8x the tokens


def test_init_fails_loudly_without_device_or_bad_args():
    from paper_2503_08467_b200 import moeshard as C
    with pytest.raises(C.MoEShardError):
        C.moeshard_init(_cfg(), 2, 2, None, 0, 0, 0)          # rank out of range
    with pytest.raises(C.MoEShardError):
        C.moeshard_init(_cfg(), 0, 1, None, 0, 0, 0)          # NULL workspace
    with pytest.raises(C.MoEShardError):
        C.moeshard_forward(None, 0, None, 0, None, None, None, None)


def test_shard_and_token_helpers():
    from paper_2503_08467_b200 import local_token_range, shard_columns
    assert [shard_columns(4, 2, g) for g in range(2)] == [(0, 2), (2, 4)]
    with pytest.raises(ValueError):
        shard_columns(6, 4, 0)
    assert local_token_range(8192, 4, 3) == (6144, 8192)


def test_top_k_config_validation():
    # top_k (R21): 0 / 1 = top-1, 2 = top-2 on the bf16 fused tcgen05 path only
    from paper_2503_08467_b200 import moeshard as C
    w1 = C.moeshard_workspace_size(_cfg(top_k=1), 1)
    assert C.moeshard_workspace_size(_cfg(top_k=0), 1) == w1
    w2 = C.moeshard_workspace_size(_cfg(top_k=2), 1)
    assert w2 > w1 + 1024 * 768 * 2 * 2        # assignment rows: X_perm, H, y_assign grow
    for bad in (dict(top_k=3), dict(top_k=-1), dict(top_k=2, n_experts=1),
                dict(top_k=2, dtype=C.MOESHARD_FP32), dict(top_k=2, flags=C.MOESHARD_FLAG_P2P),
                dict(top_k=2, flags=C.MOESHARD_FLAG_UNFUSED_GEMM),
                dict(top_k=2, flags=C.MOESHARD_FLAG_SIMT_GEMM),
                dict(top_k=2, flags=C.MOESHARD_FLAG_LAUNCH_PER_EXPERT),
                dict(top_k=2, flags=C.MOESHARD_FLAG_ONCHIP_H)):
        with pytest.raises(C.MoEShardError) as ei:
            C.moeshard_workspace_size(_cfg(**bad), 1)
        assert ei.value.code == -5, bad
