"""GPU tests of the multi-GPU product driver (paper_2507_11424_b200/dist.py) on one B200.

Only one GPU is available per test box, so the N > 1 collectives are covered by the gloo
tests in test_multirank.py; here (i) the whole DistSampler pipeline runs over NCCL at world
size 1 (broadcast, tn_prepare, tn_sample_dev, all_gather_into_tensor), and (ii) the shards
that ranks 0..G-1 of a G-GPU run would draw (contiguous global index ranges, uniforms of the
global index) are drawn one after another on this GPU and must equal the unsharded run
bitwise (SURVEY 8(e) determinism: bits and ln q identical for G in {1, 2, 3, 8})."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2507_11424_b200 import TNState  # noqa: E402
from paper_2507_11424_b200.dist import DistSampler, shard_range, uniforms_rows  # noqa: E402
from tninputs import lattices as L  # noqa: E402
from tninputs import synthetic as S  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dev_sample(g, rows, R, u):
    dev = torch.device("cuda", 0)
    ud = torch.from_numpy(np.ascontiguousarray(u)).to(dev)
    b = torch.empty((u.shape[0], u.shape[1]), dtype=torch.uint8, device=dev)
    lq = torch.empty(u.shape[0], dtype=torch.float64, device=dev)
    g.sample_dev(rows, R, u.shape[0], ud.data_ptr(), b.data_ptr(), lq.data_ptr(), 0, 0,
                 torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize()
    return b.cpu().numpy(), lq.cpu().numpy()


@pytest.mark.parametrize("lat_name,chi,R", [("square3x3", 2, 16), ("willow105", 4, 16)])
def test_shards_bitwise_equal_unsharded(lat_name, chi, R):
    lat = L.by_name(lat_name)
    st = S.vidal_like(lat, chi, seed=8, xi=2.0)
    n, seed = 37, 77
    g = TNState(st)
    g.prepare(lat.rows, R)
    full_b, full_l = _dev_sample(g, lat.rows, R, S.uniforms(n, lat.n, seed))
    for world in (2, 3, 8):
        bs, ls = [], []
        for r in range(world):
            k0, k1 = shard_range(n, world, r)
            if k1 > k0:
                b, lq = _dev_sample(g, lat.rows, R, uniforms_rows(seed, lat.n, k0, k1))
                bs.append(b)
                ls.append(lq)
        assert np.array_equal(np.concatenate(bs), full_b), world
        assert np.array_equal(np.concatenate(ls), full_l), world


def test_dist_sampler_nccl_world1():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        lat = L.square(3, 3)
        st = S.vidal_like(lat, 2, seed=3, xi=2.0)
        dev = torch.device("cuda", 0)
        ds = DistSampler(st, lat.rows, 16, dist, dev).prepare()
        bits, logq = ds.sample(24, seed=5)
        g = TNState(st)
        ref_b, ref_l, _, _ = g.sample(lat.rows, 16, S.uniforms(24, lat.n, 5))
        assert np.array_equal(bits.cpu().numpy(), ref_b)
        assert np.array_equal(logq.cpu().numpy(), ref_l)
        assert ds.gather_ms >= 0
    finally:
        dist.destroy_process_group()


def test_sharded_precompute_world1_bitwise():
    """NEXT-2: tn_prepare through the sharded chunk loops (an NCCL communicator of one rank,
    every chunk broadcast from its owner, assembled in chunk order) gives bitwise the same
    norm environments -- hence samples, ln q and ln <psi|psi> -- as the one-GPU path with the
    same chunking; small chunks (option chunk_elems) make every double-layer fit span
    several chunks."""
    from paper_2507_11424_b200._lib import comm_unique_id
    lat = L.by_name("willow105")
    st = S.vidal_like(lat, 4, seed=12, xi=3.0)
    R = 16
    u = S.uniforms(8, lat.n, 3)
    ref = TNState(st)
    ref.set_option("chunk_elems", 20000)
    rb, rl, rc, _ = ref.sample(lat.rows, R, u, want_cond=True)
    g = TNState(st)
    g.set_option("chunk_elems", 20000)
    g.set_comm(comm_unique_id(), 0, 1)
    b, lq, cd, _ = g.sample(lat.rows, R, u, want_cond=True)
    assert (b == rb).all() and np.array_equal(lq, rl) and np.array_equal(cd, rc)
    assert g.log_norm(R) == ref.log_norm(R)
    # default chunking: the same samples up to the summation order of the chunk partials
    d = TNState(st)
    db, dl, _, _ = d.sample(lat.rows, R, u, want_cond=True)
    assert np.allclose(dl, rl, rtol=1e-4, atol=1e-6)
