"""world_size-2 multi-process tests on CPU (gloo): the rank-side host logic of
the N>1 path - uid broadcast, shard slicing, rank-major token split - and
Algorithm 1 run with real collectives (all_gather for Step 3, a summing
collective for Step 5) against the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        import workload as W
        from paper_2503_08467_b200 import broadcast_uid, local_token_range, shard_columns

        # uid broadcast (moeshard_init's collective contract)
        uid = bytes(range(128)) if rank == 0 else None
        got = broadcast_uid(uid, rank)
        assert got == bytes(range(128))

        N, h, d_ff, E, seed = 64, 16, 32, 4, 7
        t0, t1 = local_token_range(N, world, rank)
        x_local = W.make_tokens(seed, t1 - t0, h, dtype=torch.float64, token_offset=t0)
        w_r = W.make_router_weight(seed, h, E, dtype=torch.float64)
        c0, c1 = shard_columns(d_ff, world, rank)
        wi_r, wo_r = W.make_expert_weights(seed, E, h, d_ff, cols=(c0, c1), dtype=torch.float64)

        # Step 1: route local tokens; Steps 2-3: all-gather tokens and routing
        rt = O.route(x_local, w_r)
        xs = [torch.empty_like(x_local) for _ in range(world)]
        dist.all_gather(xs, x_local)
        ex = [torch.empty(t1 - t0, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ex, torch.from_numpy(rt.expert))
        gs = [torch.empty(t1 - t0, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gs, torch.from_numpy(rt.gate))
        x_all = torch.cat(xs).numpy()
        e_all = torch.cat(ex).numpy()
        g_all = torch.cat(gs).numpy()
        # Step 4: this rank's shard on ALL tokens, grouped per expert across GPUs (Sec. 3.3)
        counts, offsets, perm = O.group_per_expert(e_all, E)
        partial = np.zeros_like(x_all)
        for e in range(E):
            rows = perm[offsets[e]:offsets[e + 1]]
            partial[rows] = g_all[rows, None] * (np.maximum(x_all[rows] @ wi_r[e].numpy(), 0) @ wo_r[e].numpy())
        # Step 5: sum partials; this rank keeps its own tokens (reduce-scatter semantics)
        p = torch.from_numpy(partial)
        dist.all_reduce(p)
        y_local = p[t0:t1].numpy()

        x_full = W.make_tokens(seed, N, h, dtype=torch.float64)
        wi, wo = W.make_expert_weights(seed, E, h, d_ff, dtype=torch.float64)
        y_ref = O.moe_layer(x_full, w_r, wi, wo)[t0:t1]
        err = O.max_abs_rel(y_local, y_ref)
        q.put((rank, err, None))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.timeout(300)
def test_alg1_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, tb in res:
        assert tb is None, tb
        assert err <= 1e-12, f"rank {rank}: {err}"
