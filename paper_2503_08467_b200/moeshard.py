"""Thin ctypes binding over libmoeshard.so (include/moeshard.h).

Argument marshalling only: every step of the layer runs in the library's
CUDA kernels. PyTorch supplies device memory (workspace, weight storage,
activations), the stream, and - for world > 1 - the process group used to
broadcast the NCCL unique id. There is no fallback: if the shared library is
missing the import of this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libmoeshard.so")

MOESHARD_OK = 0
MOESHARD_BF16 = 0
MOESHARD_FP32 = 1
MOESHARD_FLAG_FORCE_COLLECTIVES = 0x1
MOESHARD_FLAG_SIMT_GEMM = 0x2
MOESHARD_FLAG_UNFUSED_GEMM = 0x4
MOESHARD_FLAG_NO_L2_PERSIST = 0x80
MOESHARD_FLAG_P2P = 0x200
MOESHARD_FLAG_DYNAMIC_SCHED = 0x1000
MOESHARD_FLAG_UNEVEN_TOKENS = 0x2000
MOESHARD_FLAG_SERIAL_AG = 0x4000
MOESHARD_FLAG_EXPERT_PARALLEL = 0x8000
MOESHARD_FLAG_LAUNCH_PER_EXPERT = 0x10000
MOESHARD_FLAG_LAUNCH_PER_SOURCE = 0x20000
MOESHARD_FLAG_ONCHIP_H = 0x40000
MOESHARD_STAGE_ROUTE = 0x1
MOESHARD_STAGE_COMPUTE = 0x2
MOESHARD_STAGE_REDUCE = 0x4
MOESHARD_STAGE_ALL = 0x7
MOESHARD_P2P_HANDLE_BYTES = 64

STATUS = {
    0: "MOESHARD_OK", -1: "MOESHARD_ERR_INVALID_ARG", -2: "MOESHARD_ERR_SHAPE",
    -3: "MOESHARD_ERR_DIVISIBILITY", -4: "MOESHARD_ERR_BOUNDS", -5: "MOESHARD_ERR_CONFIG",
    -6: "MOESHARD_ERR_NOT_LOADED", -7: "MOESHARD_ERR_PROTOCOL", -8: "MOESHARD_ERR_CUDA",
    -9: "MOESHARD_ERR_NCCL",
}

# every entry point include/moeshard.h declares
EXPORTS = [
    "moeshard_get_unique_id", "moeshard_workspace_size", "moeshard_weight_storage_size",
    "moeshard_init", "moeshard_load_expert_shards", "moeshard_forward", "moeshard_get_routing",
    "moeshard_get_stats", "moeshard_check", "moeshard_last_error", "moeshard_status_string",
    "moeshard_destroy", "moeshard_version", "moeshard_profile", "moeshard_get_phase_ms",
    "moeshard_forward_stages", "moeshard_p2p_region", "moeshard_p2p_export", "moeshard_p2p_open",
    "moeshard_p2p_connect", "moeshard_get_ep_admission",
]
PHASES = ["router", "allgather", "grouping", "gemm_up", "gemm_down", "reduce_scatter"]


class MoEShardError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class moeshard_config(ctypes.Structure):
    _fields_ = [
        ("d_model", ctypes.c_int32), ("d_ff", ctypes.c_int32), ("n_experts", ctypes.c_int32),
        ("n_layers", ctypes.c_int32), ("max_tokens_per_rank", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("flags", ctypes.c_uint32),
        ("ep_capacity_factor", ctypes.c_float), ("top_k", ctypes.c_int32),
    ]


class moeshard_stats(ctypes.Structure):
    _fields_ = [("n_tokens_global", ctypes.c_int64), ("tiles_up", ctypes.c_int64),
                ("tiles_down", ctypes.c_int64), ("rows_executed_up", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64)]


def _nccl_lib_path() -> Optional[str]:
    try:
        import nvidia.nccl as nn
        p = os.path.join(list(nn.__path__)[0], "lib", "libnccl.so.2")
        return p if os.path.exists(p) else None
    except Exception:
        return None


def load_library() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU or eager fallback)")
    if "MOESHARD_NCCL_LIB" not in os.environ:
        p = _nccl_lib_path()
        if p:
            os.environ["MOESHARD_NCCL_LIB"] = p
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    cfgp = ctypes.POINTER(moeshard_config)
    sig = {
        "moeshard_get_unique_id": ([ctypes.c_char_p], i32),
        "moeshard_workspace_size": ([cfgp, i32, ctypes.POINTER(sz)], i32),
        "moeshard_weight_storage_size": ([cfgp, i32, ctypes.POINTER(sz)], i32),
        "moeshard_init": ([ctypes.POINTER(vp), cfgp, i32, i32, ctypes.c_char_p, vp, sz, i32], i32),
        "moeshard_load_expert_shards": ([vp, i32, vp, vp, vp, sz, vp], i32),
        "moeshard_forward": ([vp, i32, vp, i32, vp, vp, vp, vp], i32),
        "moeshard_get_routing": ([vp, vp, vp, vp, vp, vp, vp], i32),
        "moeshard_get_stats": ([vp, ctypes.POINTER(moeshard_stats), vp], i32),
        "moeshard_check": ([vp, vp], i32),
        "moeshard_last_error": ([vp], ctypes.c_char_p),
        "moeshard_status_string": ([i32], ctypes.c_char_p),
        "moeshard_destroy": ([vp], i32),
        "moeshard_version": ([], ctypes.c_char_p),
        "moeshard_profile": ([vp, i32], i32),
        "moeshard_get_phase_ms": ([vp, ctypes.POINTER(ctypes.c_float), i32,
                                   ctypes.POINTER(ctypes.c_int)], i32),
        "moeshard_forward_stages": ([vp, i32, vp, i32, vp, vp, vp, i32, vp], i32),
        "moeshard_p2p_region": ([vp, ctypes.POINTER(vp), ctypes.POINTER(sz)], i32),
        "moeshard_p2p_export": ([vp, ctypes.c_char_p], i32),
        "moeshard_p2p_open": ([vp, ctypes.c_char_p, ctypes.POINTER(vp)], i32),
        "moeshard_p2p_connect": ([vp, ctypes.POINTER(vp)], i32),
        "moeshard_get_ep_admission": ([vp, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = load_library()


def _check(code: int, ctx=None):
    if code != MOESHARD_OK:
        raise MoEShardError(code, _lib.moeshard_last_error(ctx).decode())


# ---------------------------------------------------------------- raw C-ABI mirrors
def moeshard_version() -> str:
    return _lib.moeshard_version().decode()


def moeshard_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.moeshard_get_unique_id(buf))
    return buf.raw


def moeshard_workspace_size(cfg: moeshard_config, world: int) -> int:
    out = ctypes.c_size_t()
    _check(_lib.moeshard_workspace_size(ctypes.byref(cfg), world, ctypes.byref(out)))
    return out.value


def moeshard_weight_storage_size(cfg: moeshard_config, world: int) -> int:
    out = ctypes.c_size_t()
    _check(_lib.moeshard_weight_storage_size(ctypes.byref(cfg), world, ctypes.byref(out)))
    return out.value


def moeshard_init(cfg: moeshard_config, rank: int, world: int, uid: Optional[bytes],
                  workspace_ptr: int, ws_bytes: int, device: int) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    _check(_lib.moeshard_init(ctypes.byref(ctx), ctypes.byref(cfg), rank, world, uid,
                              ctypes.c_void_p(workspace_ptr), ws_bytes, device))
    return ctx


def moeshard_load_expert_shards(ctx, layer, w_in_ptr, w_out_ptr, storage_ptr, nbytes, stream):
    _check(_lib.moeshard_load_expert_shards(ctx, layer, w_in_ptr, w_out_ptr, storage_ptr, nbytes,
                                            stream), ctx)


def moeshard_forward(ctx, layer, hidden_ptr, n_local, router_ptr, out_ptr, forced_ptr, stream):
    _check(_lib.moeshard_forward(ctx, layer, hidden_ptr, n_local, router_ptr, out_ptr, forced_ptr,
                                 stream), ctx)


def moeshard_forward_stages(ctx, layer, hidden_ptr, n_local, router_ptr, out_ptr, forced_ptr,
                            stages, stream):
    _check(_lib.moeshard_forward_stages(ctx, layer, hidden_ptr, n_local, router_ptr, out_ptr,
                                        forced_ptr, stages, stream), ctx)


def moeshard_p2p_region(ctx):
    """(device pointer, bytes) of this context's exchange region."""
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(_lib.moeshard_p2p_region(ctx, ctypes.byref(p), ctypes.byref(n)), ctx)
    return p.value, n.value


def moeshard_p2p_export(ctx) -> bytes:
    buf = ctypes.create_string_buffer(MOESHARD_P2P_HANDLE_BYTES)
    _check(_lib.moeshard_p2p_export(ctx, buf), ctx)
    return buf.raw


def moeshard_p2p_open(ctx, handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(_lib.moeshard_p2p_open(ctx, handle, ctypes.byref(p)), ctx)
    return p.value


def moeshard_p2p_connect(ctx, regions):
    arr = (ctypes.c_void_p * len(regions))(*regions)
    _check(_lib.moeshard_p2p_connect(ctx, arr), ctx)


def moeshard_get_routing(ctx, expert_ptr, gate_ptr, counts_ptr, offsets_ptr, perm_ptr, stream):
    _check(_lib.moeshard_get_routing(ctx, expert_ptr, gate_ptr, counts_ptr, offsets_ptr, perm_ptr,
                                     stream), ctx)


def moeshard_get_ep_admission(ctx, owner_ptr, expert_ptr, gate_ptr, received_ptr, stream):
    _check(_lib.moeshard_get_ep_admission(ctx, owner_ptr, expert_ptr, gate_ptr, received_ptr,
                                          stream), ctx)


def moeshard_get_stats(ctx, stream) -> dict:
    st = moeshard_stats()
    _check(_lib.moeshard_get_stats(ctx, ctypes.byref(st), stream), ctx)
    return {k: getattr(st, k) for k, _ in st._fields_}


def moeshard_check(ctx, stream):
    _check(_lib.moeshard_check(ctx, stream), ctx)


def moeshard_destroy(ctx):
    _check(_lib.moeshard_destroy(ctx))


def moeshard_last_error(ctx=None) -> str:
    return _lib.moeshard_last_error(ctx).decode()


def moeshard_profile(ctx, enable: bool):
    _check(_lib.moeshard_profile(ctx, 1 if enable else 0), ctx)


def moeshard_get_phase_ms(ctx):
    """({phase: total ms}, number of forwards) since profiling was enabled."""
    buf = (ctypes.c_float * len(PHASES))()
    cnt = ctypes.c_int()
    _check(_lib.moeshard_get_phase_ms(ctx, buf, len(PHASES), ctypes.byref(cnt)), ctx)
    return {k: float(buf[i]) for i, k in enumerate(PHASES)}, cnt.value
