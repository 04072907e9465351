"""World-size-2/3 `gloo` tests of the multi-GPU host logic (no GPU): the state broadcast, the
contiguous sample shards and the gather of paper_2507_11424_b200/dist.py,
which bench.py and users drive over NCCL on GPUs."""
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


# ------------------------------------------------------------ the product driver (dist.py)
def _stub_sampler(u, offset):
    """Deterministic stand-in for the GPU sampler (no oracle, no method): bits = u >= 1/2,
    ln q = sum ln u, plus the global index of the first row (checks the offsets)."""
    bits = torch.from_numpy((u >= 0.5).astype(np.uint8))
    logq = torch.from_numpy(np.log(u).sum(axis=1) + offset)
    return bits, logq


def _dist_worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_11424_b200.dist import DistSampler, shard_range
    from tninputs import lattices as L
    from tninputs import synthetic as S
    lat = L.square(2, 3)
    st = S.vidal_like(lat, 3, seed=5) if rank == 0 else None
    ds = DistSampler(st, lat.rows, 8, dist, torch.device("cpu"), sampler=_stub_sampler)
    ref = S.vidal_like(lat, 3, seed=5)
    same_state = all(np.array_equal(a, b) for a, b in zip(ds.state["tensors"], ref["tensors"])) and \
        np.array_equal(ds.state["edges"], ref["edges"]) and np.array_equal(ds.state["bond_dims"], ref["bond_dims"])
    bits, logq = ds.sample(n, seed=99)
    u = S.uniforms(n, lat.n, 99)
    want_b = (u >= 0.5).astype(np.uint8)
    offs = np.concatenate([[shard_range(n, world, r)[0]] * (shard_range(n, world, r)[1] - shard_range(n, world, r)[0])
                           for r in range(world)])
    want_l = np.log(u).sum(axis=1) + offs
    out.put((rank, same_state, np.array_equal(bits.numpy(), want_b), np.array_equal(logq.numpy(), want_l)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 11), (3, 10), (2, 1)])
def test_dist_sampler_gather_global_order(world, n):
    """DistSampler over gloo: state broadcast from rank 0, contiguous shards of the global
    sample index, all_gather_into_tensor of bits and ln q -> every rank holds
    all n samples in global order, equal to the unsharded run (ragged shards, an empty one)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(all(r[1:]) for r in res), res


def test_uniform_rows_equal_full_matrix():
    from paper_2507_11424_b200.dist import shard_range, uniforms_rows
    from tninputs import synthetic as S
    full = S.uniforms(23, 7, 1234)
    for world in (1, 2, 3, 8):
        parts = [uniforms_rows(1234, 7, *shard_range(23, world, r)) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)
