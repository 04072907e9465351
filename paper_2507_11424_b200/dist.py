"""Multi-GPU sampling driver: one process per GPU, torch.distributed for the
plumbing, every step of the method in libtnsample's kernels.

Samples are independent given the state and its norm environments (the norm
network is contracted "once (independent of the number of samples)"), so the path shards
without a data-path collective:

1. ``broadcast_state``  -- the TNS (graph + complex128 tensors) is broadcast from rank 0
   (NCCL over NVLink on GPUs; gloo in the CPU tests).
2. ``tn_prepare`` (a1) runs on every rank; by default the ranks share it (NEXT-2): the
   double-layer fits split their chunk loops over the ranks inside libtnsample (NCCL
   broadcast of each chunk from its owner, assembly in the same order as one GPU, so the
   environments are bitwise the same on every rank); without sharing every rank computes all
   of it (deterministic kernels, no communication);
3. rank g of G draws the global samples [floor(g n / G), floor((g+1) n / G)) -- its contiguous
   shard -- reading uniforms[k] of the global sample index k (so results do not depend on G);
4. ``all_gather_into_tensor`` of the bits (uint8) and ln q (float64), padded to the largest
   shard and trimmed, gives every rank the n samples in global order.

The sampler is injectable (``sampler(u_shard, offset) -> (bits, logq)``) so the sharding
and the collectives are tested on CPU with gloo and a deterministic stub; the product
sampler is ``TNState.sample_dev`` (device buffers, the caller's CUDA stream).
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int):
    """Contiguous shard [floor(rank n / world), floor((rank+1) n / world))."""
    return (rank * n) // world, ((rank + 1) * n) // world


def uniforms_rows(seed: int, n_vertices: int, k0: int, k1: int) -> np.ndarray:
    """Rows k0..k1-1 of tninputs.synthetic.uniforms(n, n_vertices, seed) without drawing the
    rows before them: numpy's PCG64 produces one 64-bit draw per float64, so the stream is
    advanced by k0 * n_vertices draws (bit-identical to slicing the full matrix)."""
    bg = np.random.PCG64(np.random.SeedSequence(seed))
    bg.advance(k0 * n_vertices)
    return np.random.Generator(bg).random((k1 - k0, n_vertices))


def broadcast_state(st, dist, device, src: int = 0):
    """Broadcast a TNS dict (n, edges, bond_dims, chi, tensors) from rank ``src``; the other
    ranks pass st=None and receive an equal dict (complex128 tensors on the host)."""
    import torch
    rank = dist.get_rank()
    if rank == src:
        n = int(st["n"])
        edges = np.asarray(st["edges"], dtype=np.int64).reshape(-1, 2)
        bd = np.asarray(st["bond_dims"], dtype=np.int64)
        head = np.array([n, len(bd), int(st["chi"])], dtype=np.int64)
        meta = torch.from_numpy(np.concatenate([head, edges.reshape(-1), bd])).to(device)
        ln = torch.tensor([meta.numel()], dtype=torch.int64, device=device)
    else:
        ln = torch.zeros(1, dtype=torch.int64, device=device)
    dist.broadcast(ln, src)
    if rank != src:
        meta = torch.zeros(int(ln.item()), dtype=torch.int64, device=device)
    dist.broadcast(meta, src)
    m = meta.cpu().numpy()
    n, ne, chi = int(m[0]), int(m[1]), int(m[2])
    edges = m[3:3 + 2 * ne].reshape(ne, 2)
    bd = m[3 + 2 * ne:3 + 3 * ne]
    inc = [[] for _ in range(n)]
    for e, (u, v) in enumerate(edges):
        inc[u].append(e)
        inc[v].append(e)
    shapes = [(2,) + tuple(int(bd[e]) for e in inc[v]) for v in range(n)]
    sizes = [int(np.prod(s)) for s in shapes]
    if rank == src:
        flat = np.concatenate([np.ascontiguousarray(t, dtype=np.complex128).reshape(-1).view(np.float64)
                               for t in st["tensors"]])
        buf = torch.from_numpy(flat).to(device)
    else:
        buf = torch.zeros(2 * sum(sizes), dtype=torch.float64, device=device)
    dist.broadcast(buf, src)
    if rank == src:
        return st
    host = buf.cpu().numpy()
    tensors, off = [], 0
    for s, z in zip(shapes, sizes):
        tensors.append(host[off:off + 2 * z].view(np.complex128).reshape(s).copy())
        off += 2 * z
    return {"n": n, "edges": edges.astype(np.int32), "bond_dims": bd.astype(np.int32), "chi": chi,
            "tensors": tensors, "meta": {}}


def gather_samples(bits, logq, n: int, dist, device):
    """all_gather_into_tensor of this rank's shard (bits [m][N] uint8, logq [m] float64, m =
    its shard size) into the n samples in global order, on every rank (torch tensors)."""
    import torch
    world = dist.get_world_size()
    N = bits.shape[1]
    mx = max(shard_range(n, world, r)[1] - shard_range(n, world, r)[0] for r in range(world))
    pb = torch.zeros((mx, N), dtype=torch.uint8, device=device)
    pl = torch.zeros(mx, dtype=torch.float64, device=device)
    m = bits.shape[0]
    pb[:m] = bits
    pl[:m] = logq
    gb = torch.empty((world * mx, N), dtype=torch.uint8, device=device)
    gl = torch.empty(world * mx, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(gb, pb)
    dist.all_gather_into_tensor(gl, pl)
    keep = np.concatenate([np.arange(r * mx, r * mx + (shard_range(n, world, r)[1] - shard_range(n, world, r)[0]))
                           for r in range(world)])
    idx = torch.from_numpy(keep).to(device)
    return gb.index_select(0, idx), gl.index_select(0, idx)


class DistSampler:
    """Data-parallel boundary-MPS sampling over the ranks of a torch.distributed group.

    state: the TNS dict on rank 0 (None elsewhere); rows: the row partition (all ranks);
    chi_env: the boundary bond R. ``sample(n, seed)`` returns (bits [n][N] uint8, ln q [n]
    float64) as torch tensors on ``device``, identical on every rank and bitwise equal to a
    one-GPU run over the same uniforms."""

    def __init__(self, state, rows, chi_env: int, dist, device, sampler=None, tn=None):
        self.dist = dist
        self.device = device
        self.rows = rows
        self.R = int(chi_env)
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.state = broadcast_state(state, dist, device) if tn is None else state
        self.n_vertices = int(self.state["n"])
        self._tn = tn  # an already prepared TNState of this state may be passed in
        self.sampler = sampler if sampler is not None else self._gpu_sampler
        self.gather_ms = 0.0

    def prepare(self, shard_precompute: bool = True, chunk_elems: int = 0):
        """a1 (tn_prepare) on every rank. With shard_precompute and more than one rank, the
        double-layer fits are split over the ranks (NEXT-2: chunk ci computed by rank
        ci % world, NCCL broadcast; bitwise the same environments on every rank); else every
        rank computes all of it (deterministic, no communication)."""
        import torch
        from ._lib import TNState, comm_unique_id
        self._tn = TNState(self.state)
        if chunk_elems:
            self._tn.set_option("chunk_elems", chunk_elems)
        if shard_precompute and self.world > 1:
            uid = torch.zeros(128, dtype=torch.uint8)
            if self.rank == 0:
                uid = torch.frombuffer(bytearray(comm_unique_id()), dtype=torch.uint8).clone()
            uid = uid.to(self.device)
            self.dist.broadcast(uid, 0)
            self._tn.set_comm(uid.cpu().numpy().tobytes(), self.rank, self.world)
        self._tn.prepare(self.rows, self.R)
        return self

    def _gpu_sampler(self, u_shard, offset):
        import torch
        if self._tn is None:
            self.prepare()
        m = u_shard.shape[0]
        u = torch.from_numpy(np.ascontiguousarray(u_shard)).pin_memory().to(self.device, non_blocking=True)
        bits = torch.empty((m, self.n_vertices), dtype=torch.uint8, device=self.device)
        logq = torch.empty(m, dtype=torch.float64, device=self.device)
        if m:
            stream = torch.cuda.current_stream(self.device)
            self._tn.sample_dev(self.rows, self.R, m, u.data_ptr(), bits.data_ptr(), logq.data_ptr(), 0, 0,
                                stream.cuda_stream)
        return bits, logq

    def sample(self, n: int, seed: int):
        k0, k1 = shard_range(n, self.world, self.rank)
        u = uniforms_rows(seed, self.n_vertices, k0, k1)
        bits, logq = self.sampler(u, k0)
        import time

        import torch
        cuda = getattr(self.device, "type", str(self.device)) == "cuda"
        if cuda:
            torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        out = gather_samples(bits, logq, n, self.dist, self.device)
        if cuda:
            torch.cuda.synchronize(self.device)
        self.gather_ms = 1e3 * (time.perf_counter() - t0)
        return out
