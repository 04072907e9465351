#!/usr/bin/env python
"""bench.py -- bitstring samples/s of generalised boundary-MPS sampling on B200 (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload NAME]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole per-sample hot path (row fit, right
ladder, left pass + draw, project/merge, over every row) for one batch of samples per GPU,
inputs (state, norm environments, uniforms) resident in HBM. The norm-environment
precompute (a1) runs once before timing and is reported separately, as in the paper
("following a pre-computed contraction of the norm network").
Multi-GPU: weak scaling, samples sharded by rank; the state is NCCL-broadcast from rank 0,
every rank recomputes the (deterministic) environments; no collective in the timed region.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bitstring samples/sec at 1/2/4/8 B200 (Willow-105, χ_env=128); TC-pipe util"

# name: lattice, chi, chi_env, samples per GPU per step
WORKLOADS = {
    # the metric configuration: Willow-105 shapes of config 4 (chi = 32, chi_env = 128)
    "willow105_chi32_env128": ("willow105", 32, 128, 4),
    # parity / smaller shapes (not the metric)
    "willow105_chi16_env64": ("willow105", 16, 64, 16),
    "willow105_chi8_env32": ("willow105", 8, 32, 256),
    "eagle127_chi16_env64": ("eagle127", 16, 64, 64),
    "square6x6_chi8_env32": ("square6x6", 8, 32, 512),
    # the paper's literal order is meant for chi_env <= chi (R <= 20 with chi >= 20)
    "willow105_chi8_env8": ("willow105", 8, 8, 256),
    # config 5 shapes (LUCJ-like two-register ladders, rows = rung pairs, chi = 64, chi_env = 256)
    "lucj52_chi64_env256": ("lucj52", 64, 256, 64),
    "lucj72_chi64_env256": ("lucj72", 64, 256, 64),
}
PHASES = ["gemm_tc_incl_prep", "gemm_simt", "permute", "orth", "tail", "misc", "tc_kernel"]
DEFAULT_WORKLOAD = "willow105_chi32_env128"
STATE_SEED = 2507
UNIFORM_SEED = 1005
E2E_SEED = 77
# SURVEY 8(d) "Algorithmic work per unit": per-sample complex MACs of the method's own
# contractions (bonds at their R6 values, nh = 2) for the configurations it tabulates
ALG_CMACS_PER_SAMPLE = {
    "willow105_chi32_env128": 4.9e13,  # cfg 4b
    "eagle127_chi16_env64": 6.5e10,    # cfg 3
    "square6x6_chi8_env32": 2.9e9,     # cfg 2
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[0]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": sorted(reasons),
                "samples": len(rows)}


STATE_KIND = "vidal"
QUENCH_LAYERS = 15


def make_state(lat, chi):
    """The benchmark state (--state): 'vidal' (default: Vidal-gauge-like, bond spectra
    ~exp(-k/8)), 'vidal_steep' (spectra ~exp(-k/2)), 'branch' (K = 11 branch superposition:
    exactly rank-deficient boundaries, the completion paths of the orthonormalisation) --
    the same tensor shapes with different value distributions, to show that the step time
    does not depend on the values."""
    from tninputs import synthetic as S
    if STATE_KIND == "quench":
        # the paper's workload itself: the domain-wall Heisenberg quench (config 4b: L = 15 Trotter
        # layers, dt = 0.1), built on the GPU by libtnsample's BP-gauged simple update (NEXT-4)
        from paper_2507_11424_b200 import construct
        from tninputs import lattices as L
        t0 = time.time()
        st = construct.heisenberg_quench(lat, L.domain_wall_bits(lat), chi, QUENCH_LAYERS)
        log(f"quench state built on the GPU in {time.time() - t0:.1f} s: fidelity {st['meta']['fidelity']:.4f}, "
            f"max bond {int(max(st['bond_dims']))}, BP residual max {st['meta']['bp_residual_max']:.2e}")
        return st
    if STATE_KIND == "vidal_steep":
        return S.vidal_like(lat, chi, seed=STATE_SEED, xi=2.0)
    if STATE_KIND == "branch":
        return S.branch_superposition(lat, chi, min(11, chi), seed=STATE_SEED)
    return S.vidal_like(lat, chi, seed=STATE_SEED)


class LazyRandomM:
    """Norm-environment sites with the shapes the method produces (R6), random values: the
    oracle's sampling time does not depend on the values, and its own precompute at the
    metric configuration would take days (SURVEY 0 finding 5)."""

    def __init__(self, P, R, rng):
        from oracle import bmps as B
        self.B = B
        self.P = P
        self.R = R
        self.rng = rng
        nb = len(P.rows)
        # shapes from the bottom row up, exactly as norm_envs() would produce them
        self.shapes = [None] * nb
        tops = None
        for b in range(nb - 1, 0, -1):
            row = P.rows[b]
            fake = None if tops is None else [np.zeros(s, dtype=np.complex64) for s in tops]
            tps = B._tops_for_row(P, row, fake, "down", "double")
            strip = B.Strip("double", tps, [P.A[v] for v in row], [P.has(v, "up") for v in row])
            D = B.bond_dims(strip, R)
            cols = [j for j in range(len(row)) if P.has(row[j], "up")]
            shp = [(D[k], P.A[row[c]].shape[1], P.A[row[c]].shape[1], D[k + 1]) for k, c in enumerate(cols)]
            self.shapes[b - 1] = shp
            tops = shp
        self.cache = {}

    def __getitem__(self, b):
        if self.shapes[b] is None:
            return None
        if b not in self.cache:
            self.cache = {}
            sites = []
            for s in self.shapes[b]:
                x = (self.rng.standard_normal(s) + 1j * self.rng.standard_normal(s)) / math.sqrt(np.prod(s[1:]))
                sites.append(x)
            self.cache[b] = sites
        return self.cache[b]


def oracle_dry_run(P, M, R):
    """Complex MACs per row of one oracle sample, counted on the oracle's own pairwise
    contractions (oracle.bmps.pair) in a shape-only dry run, and the shapes of the incoming
    boundary MPS of every row: every pair() returns zeros of the output shape and _merge's
    outputs are recorded, so the whole sample costs milliseconds. The oracle's arithmetic is
    untouched (the dry run replaces the two functions only for the duration of the count)."""
    from oracle import bmps as B
    counts = [0.0]
    real_pair, real_merge = B.pair, B._merge
    merged = []

    def dry_pair(a, sa, b, sb, out):
        dims = {}
        for lab, t in ((sa, a), (sb, b)):
            for ch, d in zip(lab, t.shape):
                dims[ch] = d
        cm = 1.0
        for d in dims.values():
            cm *= d
        counts[0] += cm
        return np.zeros([dims[ch] for ch in out], dtype=np.complex128)

    def rec_merge(P_, row, sites):
        m = real_merge(P_, row, sites)
        merged.append(None if m is None else [t.shape for t in m])
        return m

    real_nstrip = B._n_strip
    marks = []

    def mark_nstrip(P_, b, m_prev):  # called once at the start of every row
        marks.append(counts[0])
        return real_nstrip(P_, b, m_prev)

    B.pair, B._merge, B._n_strip = dry_pair, rec_merge, mark_nstrip
    try:
        with np.errstate(all="ignore"):
            B.sample(P, M, R, np.zeros(P.n), forced=np.zeros(P.n, dtype=np.uint8))
    finally:
        B.pair, B._merge, B._n_strip = real_pair, real_merge, real_nstrip
    marks.append(counts[0])
    per_row = [marks[i + 1] - marks[i] for i in range(len(P.rows))]
    m_shapes = [None] + list(merged[:-1])  # incoming MPS of row b = merge of row b-1
    return per_row, m_shapes


class OracleTimer:
    """Bounded timing of the CPU oracle (oracle/bmps.sample, as it stands) on the same
    workload: ONE row of one sample, run from a random incoming boundary MPS and random
    norm-environment sites of the method's shapes (the oracle's own precompute at the metric
    configuration takes days). Interior rows run every vertex at the same full-bond shapes
    (bonds R = chi_env, chi), so a row's time gives the oracle's rate at the sample's dominant
    contraction shapes; the row is the one with the largest share of the sample's complex
    MACs (counted on the oracle's own contractions, oracle_dry_run) whose predicted time fits
    the budget, and one row's time / its share of the sample's MACs = the oracle's time per
    sample. A 'step' of the reference arm is one such row."""

    def __init__(self, st, lat, R, budget_s, seed=7, workload=None):
        from oracle import bmps as B
        self.B = B
        try:
            from threadpoolctl import threadpool_info
            self.threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count()])
        except Exception:
            self.threads = os.cpu_count()
        t0 = time.time()
        self.P = B.Prepared(st, lat.rows)
        self.rng = np.random.default_rng(seed)
        self.M = LazyRandomM(self.P, R, self.rng)
        try:  # cached dry run (scripts/oracle_row_cmacs.py); minutes at the metric shapes
            ent = json.load(open(os.path.join(ROOT, "profiles", "oracle_row_cmacs.json")))[workload]
            rc = ent["row_cmacs"]
            self.m_shapes = [None if m is None else [tuple(t) for t in m] for m in ent["m_shapes"]]
        except Exception:
            rc, self.m_shapes = oracle_dry_run(self.P, self.M, R)
        self.rc = np.asarray(rc, dtype=np.float64)
        self.total = float(self.rc.sum())
        self.R = R
        self.nrows = len(lat.rows)
        self.u = np.random.default_rng(seed).random(lat.n)
        # host complex-GEMM rate (one 2048^3 zgemm) as the prior for choosing the row
        a = np.ones((2048, 2048), dtype=np.complex128)
        _ = a @ a
        t1 = time.time()
        _ = a @ a
        self.zrate = 2048.0 ** 3 / max(time.time() - t1, 1e-6)
        pred = self.rc / (0.5 * self.zrate)
        ok = [b for b in range(self.nrows) if pred[b] <= budget_s] or [int(np.argmin(self.rc + (self.rc == 0) * 1e30))]
        self.row = max(ok, key=lambda b: self.rc[b])
        shp = self.m_shapes[self.row]
        self.m_in = None if shp is None else [
            (self.rng.standard_normal(s) + 1j * self.rng.standard_normal(s)) / math.sqrt(np.prod(s)) for s in shp]
        self.setup = time.time() - t0

    def run(self):
        t0 = time.time()
        self.B.sample(self.P, self.M, self.R, self.u, first_row=self.row, max_rows=self.row + 1, m_in=self.m_in)
        return time.time() - t0

    def measure(self):
        t = self.run()
        frac = self.rc[self.row] / self.total
        rate = frac / t if t > 0 else float("nan")
        return {"value": rate, "unit": "samples/s", "cores": int(self.threads), "kind": "oracle",
                "seconds": t, "fraction_of_sample": frac,
                "sample": (f"row {self.row} of {self.nrows} of one sample ({100 * frac:.3g}% of the sample's complex MACs, "
                           f"counted on the oracle's own contractions by a shape-only dry run; every vertex at the "
                           f"full-bond shapes that dominate the sample), measured {t:.1f} s on the host from a random "
                           f"incoming boundary MPS and random norm-environment sites of the method's shapes (the "
                           f"oracle's precompute at this size takes days); samples/s = fraction / seconds; host "
                           f"zgemm rate {self.zrate / 1e9:.0f} G complex MAC/s; setup {self.setup:.0f} s not timed")}


def oracle_rate(st, lat, R, budget_s, seed=7, workload=None):
    return OracleTimer(st, lat, R, budget_s, seed, workload).measure()


def apply_partition(st, lat, partition):
    """--partition chip: the chip-row partition through the exact vertex split (NEXT-3); the
    returned lattice stand-in carries the split network's rows and vertex count."""
    if partition != "chip":
        return st, lat
    from types import SimpleNamespace

    from tninputs import lattices as L
    from tninputs import synthetic as S
    st2, rows2, _ = S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])
    return st2, SimpleNamespace(rows=rows2, n=st2["n"], name=lat.name + "_chiprows", edges=st2["edges"].tolist())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="samples per GPU per step (0 = workload default)")
    ap.add_argument("--order", type=int, default=0, choices=[0, 1],
                    help="0: compress-then-sample (R3, default); 1: the paper's literal order (NEXT-3, R <= chi)")
    ap.add_argument("--cpu-budget", type=float, default=40.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--state", default="vidal", choices=["vidal", "vidal_steep", "branch", "quench"])
    ap.add_argument("--layers", type=int, default=15, help="Trotter layers of --state quench")
    ap.add_argument("--partition", default="rows", choices=["rows", "chip"],
                    help="rows: lattice rows (the paper's column-wise partition, default); chip: the chip-row "
                         "('diagonal', P:256-260) partition of Willow through the vertex split (NEXT-3)")
    a = ap.parse_args()
    global STATE_KIND, QUENCH_LAYERS
    STATE_KIND = a.state
    QUENCH_LAYERS = a.layers
    if a.impl == "reference" and a.state == "quench":
        STATE_KIND = "vidal"  # the oracle's row timing depends on the shapes only (same shapes)
    assert a.warmup >= 1 and a.steps >= 1

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    lat_name, chi, R, batch = WORKLOADS[a.workload]
    if a.batch:
        batch = a.batch
    from tninputs import lattices as L
    lat = L.by_name(lat_name)
    config = {"precompute": "shared by the ranks (NEXT-2, NCCL)" if world > 1 else "one GPU",
              "workload": a.workload, "lattice": lat_name, "n_qubits": lat.n, "chi": chi, "chi_env": R,
              "samples_per_gpu_per_step": batch, "fit_half_sweeps": 2, "row_order": "lattice rows",
              "within_row_order": "paper-literal (NEXT-3)" if a.order else "compress-then-sample (R3)",
              "partition": "chip rows via vertex split (NEXT-3)" if a.partition == "chip" else "lattice rows",
              "state": {"vidal": "synthetic Vidal-gauge-like TNS (dense, singular-value-weighted bonds ~exp(-k/8), every "
                                 "bond at chi)",
                        "vidal_steep": "synthetic Vidal-gauge-like TNS, bond spectra ~exp(-k/2), every bond at chi",
                        "branch": "K = 11 branch superposition at bond chi (rank-deficient boundaries)",
                        "quench": f"domain-wall Heisenberg quench, {a.layers} Trotter layers, dt = 0.1, built on the "
                                  f"GPU by BP-gauged simple update (NEXT-4)"}[a.state],
              "l2": "L2 flushed between timed steps (256 MB write); per-step working set >> 126 MB"}

    if a.impl == "reference":
        if rank != 0:
            return
        st = make_state(lat, chi)
        st, lat = apply_partition(st, lat, a.partition)
        # rows' cost shares: complex MACs of the oracle's own contractions, counted by a
        # shape-only dry run of oracle.bmps.sample (oracle_row_cmacs)
        # each step a bounded sample; the whole run stays within ~4 minutes after setup
        timer = OracleTimer(st, lat, R, budget_s=min(a.cpu_budget, 240.0 / (a.warmup + a.steps)),
                            workload=a.workload + ("_chip" if a.partition == "chip" else ""))
        vals, secs = [], []
        for i in range(a.warmup + a.steps):
            cb = timer.measure()
            if i >= a.warmup:
                vals.append(cb["value"])
                secs.append(cb["seconds"])
        v = float(np.mean(vals))
        # a step = one row of one sample (cb["fraction_of_sample"] of a sample), measured seconds
        out = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": a.gpus, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": 1000.0 * float(np.mean(secs)), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
               "config": config, "impl": "reference",
               "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cb["cores"], "kind": "oracle",
                                "sample": cb["sample"]},
               "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2507_11424_b200 import TNState, _lib
    LIB = _lib.lib()
    LIB.tn_debug_counters.argtypes = [C.c_void_p, C.c_int]
    LIB.tn_debug_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    LIB.tn_debug_set_profile.argtypes = [C.c_int]
    LIB.tn_debug_row_cmacs.argtypes = [C.c_void_p, C.c_int]

    from paper_2507_11424_b200.dist import DistSampler, broadcast_state, gather_samples, shard_range, uniforms_rows
    t0 = time.time()
    st = make_state(lat, chi) if rank == 0 else None
    if world > 1:
        st = broadcast_state(st, dist, dev)  # NCCL broadcast of the TNS from rank 0
    st, lat = apply_partition(st, lat, a.partition)
    g = TNState(st)
    if a.order:
        g.set_option("order", a.order)
    if world > 1:
        # NEXT-2: the ranks share the norm-environment precompute (tn_set_comm: the double-layer
        # fits' chunks split over an NCCL communicator, bitwise the same environments everywhere)
        from paper_2507_11424_b200._lib import comm_unique_id
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        g.set_comm(uid.cpu().numpy().tobytes(), rank, world)
    t_load = time.time() - t0
    t0 = time.time()
    pre_prof = np.zeros(7)
    LIB.tn_debug_set_profile(1)
    LIB.tn_debug_profile(pre_prof.ctypes.data, None, 7, 1)
    g.prepare(lat.rows, R)
    torch.cuda.synchronize()
    t_pre = time.time() - t0
    LIB.tn_debug_profile(pre_prof.ctypes.data, None, 7, 1)
    LIB.tn_debug_set_profile(0)
    pre_phase = {k: round(float(v), 1) for k, v in zip(PHASES, pre_prof)}
    log(f"[rank {rank}] state {t_load:.1f}s, precompute {t_pre:.1f}s, phases (ms) {pre_phase}")

    N = lat.n
    nsteps = a.warmup + a.steps
    # contiguous shard of the global sample index: rank r owns samples
    # [floor(r n / G), floor((r+1) n / G)), n = G * batch * nsteps, uniforms of the global index
    n_total = world * batch * nsteps
    k0, k1 = shard_range(n_total, world, rank)
    u_mine = uniforms_rows(UNIFORM_SEED, N, k0, k1).reshape(nsteps, batch, N)
    u_dev = torch.from_numpy(u_mine).to(dev)
    bits_dev = torch.empty((nsteps, batch, N), dtype=torch.uint8, device=dev)
    logp_dev = torch.empty((nsteps, batch), dtype=torch.float64, device=dev)
    flags_dev = torch.zeros((nsteps, batch), dtype=torch.int32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(s):
        g.sample_dev(lat.rows, R, batch, u_dev[s].data_ptr(), bits_dev[s].data_ptr(), logp_dev[s].data_ptr(),
                     0, flags_dev[s].data_ptr(), stream.cuda_stream)

    for s in range(a.warmup):
        step(s)
        flush.zero_()
    torch.cuda.synchronize()
    cnt0 = np.zeros(4)
    LIB.tn_debug_counters(cnt0.ctypes.data, 1)
    prof = np.zeros(7)
    # inside the timed region only the tensor-core GEMM kernels are bracketed by CUDA events
    # (for the roofline); the per-phase breakdown comes from one extra, untimed step below
    LIB.tn_debug_set_profile(1 << 6)  # P_TC_KERNEL
    LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
    clocks = Clocks(local)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(a.warmup, nsteps):
        step(s)
        flush.zero_()
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
    LIB.tn_debug_set_profile(0)
    cnt = np.zeros(4)
    LIB.tn_debug_counters(cnt.ctypes.data, 0)
    rows = np.zeros(len(lat.rows))
    LIB.tn_debug_row_cmacs(rows.ctypes.data, len(rows))
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * batch * a.steps / (ms / 1000.0)

    # validation of the benchmarked samples (all ranks): per-sample flags (TN_FLAG_*, R9),
    # non-finite ln q, mean -ln q, bits in {0, 1}
    fl = flags_dev[a.warmup:].reshape(-1).to(torch.int64)
    lq = logp_dev[a.warmup:].reshape(-1)
    stats = torch.stack([(fl & 1 != 0).sum(), (fl & 2 != 0).sum(), (fl & 4 != 0).sum(),
                         (~torch.isfinite(lq)).sum(), (bits_dev[a.warmup:] > 1).sum()]).to(torch.float64)
    nlq = torch.where(torch.isfinite(lq), -lq, torch.zeros_like(lq)).sum().reshape(1)
    stats = torch.cat([stats, nlq])
    if dist:
        dist.all_reduce(stats)
    stats = stats.cpu().numpy()
    n_timed = world * batch * a.steps
    validation = {"samples": n_timed, "flag_clamped": int(stats[0]), "flag_zero_mass": int(stats[1]),
                  "flag_nonfinite": int(stats[2]), "logq_nonfinite": int(stats[3]), "bits_not_01": int(stats[4]),
                  "mean_minus_logq": float(stats[5]) / max(1, n_timed - int(stats[3])),
                  "valid": bool(stats[2] == 0 and stats[3] == 0 and stats[4] == 0)}
    # the product path's gather (dist.py, all_gather_into_tensor of bits and ln q), timed apart
    gather_ms = None
    if dist:
        torch.cuda.synchronize()
        tg = time.perf_counter()
        gb, gl = gather_samples(bits_dev[a.warmup:].reshape(-1, N), logp_dev[a.warmup:].reshape(-1),
                                world * batch * a.steps, dist, dev)
        torch.cuda.synchronize()
        gather_ms = 1e3 * (time.perf_counter() - tg)

    # e2e through the public API at N GPUs (DistSampler.sample: uniforms built on the host and
    # copied H2D from pinned memory, sampling, the gather, D2H of bits + ln q), wall clock
    e2e_steps = 1 if chi >= 32 else a.steps
    ds = DistSampler(st, lat.rows, R, dist, dev, tn=g) if dist else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(e2e_steps):
        if ds is not None:
            eb, el = ds.sample(world * batch, seed=E2E_SEED + s)
            eb, el = eb.cpu(), el.cpu()
        else:
            g.sample(lat.rows, R, uniforms_rows(E2E_SEED + s, N, 0, batch))
    torch.cuda.synchronize()
    te = time.perf_counter() - t0
    if dist:
        t = torch.tensor([te], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e = {"value": world * batch * e2e_steps / te, "unit": "samples/s",
           "h2d_bytes_per_step": int(world * batch * N * 8),
           "d2h_bytes_per_step": int(world * batch * (N + 8)), "steps": e2e_steps,
           "api": "paper_2507_11424_b200.dist.DistSampler.sample" if dist else "tn_sample (host buffers)"}

    # per-phase device time of one extra (untimed) step, every phase bracketed by CUDA events
    phase = np.zeros(7)
    LIB.tn_debug_set_profile(1)
    LIB.tn_debug_profile(phase.ctypes.data, None, 7, 1)
    step(0)
    torch.cuda.synchronize()
    LIB.tn_debug_profile(phase.ctypes.data, None, 7, 1)
    LIB.tn_debug_set_profile(0)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    pk, which = peaks()
    ratio = 1.1 / 2.25  # nominal dense TF32 / BF16
    tf32_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * ratio
    tc_ms = prof[6]
    tc_cmacs = cnt[1]
    executed_per_sample = float(cnt[0]) / (batch * a.steps)
    # algorithmic work: SURVEY 8(d)'s per-sample complex MACs for this configuration (the
    # method's own contractions), x the samples the timed kernels processed; where 8(d) has no
    # figure, the engine's executed count of the tensor-core GEMMs
    alg_ps = ALG_CMACS_PER_SAMPLE.get(a.workload)
    alg_cmacs = alg_ps * batch * a.steps if alg_ps else tc_cmacs
    achieved = (8.0 * alg_cmacs) / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else None
    achieved_exec = (8.0 * tc_cmacs) / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else None
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "tc_gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(a.workload)
            traffic, traffic_src = float(t["bytes_per_launch"]), t["source"]
        except Exception:
            traffic = None
    fp16_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    roofline = {"bound": "tensor",
                "kernel": "tc_gemm2_kernel / tc_gemm_kernel (tcgen05 kind::f16, CTA pair, FP16x3 split complex GEMM)",
                "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": (achieved / tf32_peak) if achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": f"{which}: FP32-class tensor peak = bf16_tflops_sustained x 1.1/2.25 (dense TF32/BF16 "
                               f"nominal ratio); the path computes complex64 products to FP32 accuracy",
                "algorithmic": (f"8 real flops per complex MAC; {alg_ps:.3g} complex MACs per sample = SURVEY 8(d) "
                                f"per-sample figure for this configuration, x {batch * a.steps} samples"
                                if alg_ps else "8 real flops per executed complex MAC of the tensor-core GEMMs "
                                               "(no SURVEY 8(d) figure for this configuration)"),
                "achieved_on_executed": achieved_exec,
                "fp16_issued": {"split_factor": 3, "peak_fp16_sustained": fp16_peak,
                                "issued_frac": (3.0 * achieved_exec / fp16_peak) if achieved_exec else None,
                                "note": "each executed complex MAC issues 3 FP16 MMAs (hi*hi + hi*lo + lo*hi) on the "
                                        "[Re -Im; Im Re] real embedding"},
                "tc_launches": int(cnt[2]), "tc_ms_total": tc_ms, "tc_share_of_step": tc_ms / ms if ms else None,
                "cmacs_per_sample_executed": executed_per_sample, "cmacs_per_sample_algorithmic": alg_ps,
                "row_cmacs_executed": [float(x) for x in rows]}
    out = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "c64", "data": "synthetic", "config": dict(config, precompute_s=t_pre),
           "roofline": roofline, "e2e": e2e, "gpu_launches": int(cnt[3] - cnt0[3]), "clocks": clk,
           "phase_ms_per_step": {k: round(float(v), 1) for k, v in zip(PHASES, phase)},
           "precompute_phase_ms": pre_phase, "validation": validation, "gather_ms": gather_ms,
           "samples_per_s_incl_precompute_1e5": 1e5 / (t_pre + 1e5 / value) if value > 0 else None}
    if world == 1 and not a.no_cpu_baseline:
        try:
            out["cpu_baseline"] = oracle_rate(st, lat, R, budget_s=a.cpu_budget, workload=a.workload + ("_chip" if a.partition == "chip" else ""))
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "oracle",
                                   "sample": f"failed: {e}"}
    print(json.dumps(out), flush=True)
    if os.environ.get("TN_GEMM_LOG"):
        LIB.tn_debug_gemm_log()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
