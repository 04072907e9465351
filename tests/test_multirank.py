"""World-size-2 `gloo` tests of the multi-GPU host logic (no GPU): the NCCL-style state
broadcast used by bench.py and the sample sharding across ranks."""
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


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from tninputs import lattices as L
    from tninputs import synthetic as S
    lat = L.square(2, 3)
    st = S.vidal_like(lat, 3, seed=bench.STATE_SEED) if rank == 0 else None
    got = bench.broadcast_state(st, lat, 3, rank, dist, torch, torch.device("cpu"))
    ref = S.vidal_like(lat, 3, seed=bench.STATE_SEED)
    same = all(np.array_equal(a, b) for a, b in zip(got["tensors"], ref["tensors"]))
    u_all = np.random.default_rng(1).random((4 * world * 5, lat.n))
    mine = bench.shard_uniforms(u_all, 4, world, rank, 5)
    t = torch.from_numpy(mine.reshape(-1, lat.n).copy())
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    if rank == 0:
        rows = torch.cat(gathered).numpy()
        # every global sample exactly once
        keys = {tuple(r) for r in rows}
        out.put((same, len(keys) == u_all.shape[0], rows.shape[0] == u_all.shape[0]))
    else:
        out.put((same, True, True))
    dist.destroy_process_group()


def test_broadcast_and_sharding_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(all(r) for r in res), res


def test_shard_is_rank_count_invariant():
    import bench
    u = np.random.default_rng(0).random((48, 4))
    one = bench.shard_uniforms(u, 6, 1, 0, 8).reshape(-1, 4)
    two = np.concatenate([bench.shard_uniforms(u, 6, 2, r, 4) for r in range(2)], axis=1).reshape(-1, 4)
    assert sorted(map(tuple, one)) == sorted(map(tuple, two))
