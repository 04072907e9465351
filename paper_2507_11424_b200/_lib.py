"""ctypes binding of libtnsample.so (argument marshalling only; see include/tnsample.h).

Every step of the sampling path runs in the library's CUDA kernels; there is no Python or
CPU fallback: if the shared library is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtnsample.so")

TN_OK = 0
ERRORS = {-1: "TN_E_ARG", -2: "TN_E_GRAPH", -3: "TN_E_ROWS", -4: "TN_E_NOMEM", -5: "TN_E_CUDA",
          -6: "TN_E_NCCL", -7: "TN_E_NUMERIC"}
EXPORTS = ["tn_load_state", "tn_prepare", "tn_sample", "tn_sample_ex", "tn_sample_dev", "tn_sample_path",
           "tn_amplitude", "tn_log_norm", "tn_certify", "tn_observables", "tn_set_option", "tn_get_stats",
           "tn_comm_unique_id", "tn_set_comm", "tn_free_state", "tn_last_error", "tn_su_create", "tn_su_bp",
           "tn_su_apply2", "tn_su_bond_dims", "tn_su_export", "tn_su_free", "tn_su_last_error"]


class TNError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class CertStats(C.Structure):
    """tn_cert_stats (include/tnsample.h)."""
    _fields_ = [("log_norm_estimate", C.c_double), ("norm_rel_stderr", C.c_double), ("kld", C.c_double),
                ("ess", C.c_double), ("n_used", C.c_int64), ("n_excluded", C.c_int64)]


class _Graph(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("n_edges", C.c_int32),
                ("edges", C.POINTER(C.c_int32)), ("bond_dims", C.POINTER(C.c_int32))]


def load_library(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libtnsample.so not built at {path}: run paper_2507_11424_b200.build")
    lib = C.CDLL(path)
    P = C.c_void_p
    i32p = C.POINTER(C.c_int32)
    lib.tn_load_state.argtypes = [C.POINTER(_Graph), C.POINTER(P), C.c_int32, C.POINTER(P)]
    lib.tn_prepare.argtypes = [P, i32p, i32p, C.c_int32, C.c_int32]
    lib.tn_sample.argtypes = [P, i32p, i32p, C.c_int32, C.c_int32, C.c_int64, P, P, P]
    lib.tn_sample_ex.argtypes = [P, i32p, i32p, C.c_int32, C.c_int32, C.c_int64, C.c_int64, P, P, P, P, P]
    lib.tn_sample_dev.argtypes = [P, i32p, i32p, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P]
    lib.tn_sample_path.argtypes = [P, i32p, i32p, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P]
    lib.tn_observables.argtypes = [P, P, P, C.c_int64, C.c_int32, P, C.c_int32, P, P, P, P, P]
    lib.tn_amplitude.argtypes = [P, P, C.c_int64, C.c_int32, P, P]
    lib.tn_comm_unique_id.argtypes = [P]
    lib.tn_set_comm.argtypes = [P, P, C.c_int32, C.c_int32]
    lib.tn_log_norm.argtypes = [P, C.c_int32, C.POINTER(C.c_double)]
    lib.tn_certify.argtypes = [P, P, P, C.c_int64, C.c_int32, C.c_double, P, C.POINTER(CertStats)]
    lib.tn_set_option.argtypes = [P, C.c_char_p, C.c_int64]
    lib.tn_get_stats.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
    lib.tn_free_state.argtypes = [P]
    lib.tn_last_error.restype = C.c_char_p
    lib.tn_su_create.argtypes = [C.c_int32, C.c_int32, P, P, C.POINTER(P)]
    lib.tn_su_bp.argtypes = [P, C.c_double, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    lib.tn_su_apply2.argtypes = [P, C.c_int32, P, C.c_int32, C.c_double, C.POINTER(C.c_double)]
    lib.tn_su_bond_dims.argtypes = [P, P]
    lib.tn_su_export.argtypes = [P, P]
    lib.tn_su_free.argtypes = [P]
    lib.tn_su_last_error.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("tn_last_error", "tn_su_last_error"):
            getattr(lib, name).restype = C.c_int
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load_library()
    return _LIB


def _check(rc):
    if rc != TN_OK:
        raise TNError(rc, lib().tn_last_error().decode())


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _rows_csr(rows):
    ptr = np.zeros(len(rows) + 1, dtype=np.int32)
    verts = []
    for i, r in enumerate(rows):
        verts += list(r)
        ptr[i + 1] = len(verts)
    return ptr, np.asarray(verts, dtype=np.int32)


class TNState:
    """A tensor-network state loaded on the current CUDA device (tn_load_state)."""

    def __init__(self, state: dict):
        edges = np.ascontiguousarray(np.asarray(state["edges"], dtype=np.int32).reshape(-1, 2))
        bd = np.ascontiguousarray(np.asarray(state["bond_dims"], dtype=np.int32))
        self.n = int(state["n"])
        self._tensors = [np.ascontiguousarray(t, dtype=np.complex128) for t in state["tensors"]]
        g = _Graph(self.n, len(bd), edges.ctypes.data_as(C.POINTER(C.c_int32)),
                   bd.ctypes.data_as(C.POINTER(C.c_int32)))
        arr = (C.c_void_p * self.n)(*[t.ctypes.data for t in self._tensors])
        h = C.c_void_p()
        _check(lib().tn_load_state(C.byref(g), arr, int(state["chi"]), C.byref(h)))
        self._h = h
        self._tensors = None  # copied by the library
        self._rows = None

    def close(self):
        if getattr(self, "_h", None):
            lib().tn_free_state(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _csr(self, rows):
        ptr, verts = _rows_csr(rows)
        self._rows = (ptr, verts)
        return (ptr.ctypes.data_as(C.POINTER(C.c_int32)), verts.ctypes.data_as(C.POINTER(C.c_int32)),
                len(rows), ptr, verts)

    def set_option(self, name: str, value: int):
        _check(lib().tn_set_option(self._h, name.encode(), int(value)))

    def prepare(self, rows, chi_env: int):
        p, v, nr, *_keep = self._csr(rows)
        _check(lib().tn_prepare(self._h, p, v, nr, int(chi_env)))

    def sample(self, rows, chi_env: int, uniforms, sample_offset: int = 0, want_cond: bool = False):
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        n = u.shape[0]
        assert u.shape[1] == self.n
        bits = np.zeros((n, self.n), dtype=np.uint8)
        logp = np.zeros(n, dtype=np.float64)
        cond = np.zeros((n, self.n), dtype=np.float64) if want_cond else None
        flags = np.zeros(n, dtype=np.uint32)
        p, v, nr, *_keep = self._csr(rows)
        _check(lib().tn_sample_ex(self._h, p, v, nr, int(chi_env), n, int(sample_offset), _ptr(u), _ptr(bits),
                                  _ptr(logp), _ptr(cond), _ptr(flags)))
        return bits, logp, cond, flags

    def sample_dev(self, rows, chi_env: int, n: int, u_ptr: int, bits_ptr: int, logp_ptr: int,
                   cond_ptr: int = 0, flags_ptr: int = 0, stream: int = 0):
        p, v, nr, *_keep = self._csr(rows)
        _check(lib().tn_sample_dev(self._h, p, v, nr, int(chi_env), int(n), C.c_void_p(u_ptr),
                                   C.c_void_p(bits_ptr), C.c_void_p(logp_ptr), C.c_void_p(cond_ptr or None),
                                   C.c_void_p(flags_ptr or None), C.c_void_p(stream or None)))

    def sample_path(self, rows, chi_env: int, uniforms):
        """tn_sample_path: bits, ln q and the amplitude carried along each sample's sampling path
        (ln|a|, arg a; p ~ |a|^2 when the fits are near exact)."""
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        n = u.shape[0]
        bits = np.zeros((n, self.n), dtype=np.uint8)
        logq = np.zeros(n)
        la = np.zeros(n)
        ph = np.zeros(n)
        p, v, nr, *_keep = self._csr(rows)
        _check(lib().tn_sample_path(self._h, p, v, nr, int(chi_env), n, _ptr(u), _ptr(bits), _ptr(logq), _ptr(la),
                                    _ptr(ph)))
        return bits, logq, la, ph

    def set_comm(self, uid: bytes, rank: int, world: int):
        """tn_set_comm: join the NCCL communicator that shares tn_prepare (NEXT-2)."""
        buf = np.frombuffer(bytes(uid), dtype=np.uint8).copy()
        _check(lib().tn_set_comm(self._h, _ptr(buf), int(rank), int(world)))

    def amplitude(self, bits, chi_env: int):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        n = b.shape[0]
        la = np.zeros(n)
        ph = np.zeros(n)
        _check(lib().tn_amplitude(self._h, _ptr(b), n, int(chi_env), _ptr(la), _ptr(ph)))
        return la, ph

    def log_norm(self, chi_env: int) -> float:
        out = C.c_double()
        _check(lib().tn_log_norm(self._h, int(chi_env), C.byref(out)))
        return out.value

    def certify(self, bits, logq, chi_env_verify: int, log_z: float = float("nan")):
        """ln p(x) of every sample and the weight statistics of tn_certify (NEXT-1)."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        q = np.ascontiguousarray(logq, dtype=np.float64)
        n = b.shape[0]
        lp = np.zeros(n)
        st = CertStats()
        _check(lib().tn_certify(self._h, _ptr(b), _ptr(q), n, int(chi_env_verify), float(log_z), _ptr(lp),
                                C.byref(st)))
        return lp, {k: getattr(st, k) for k, _ in CertStats._fields_}

    def stats(self):
        n = C.c_int64()
        t = C.c_double()
        _check(lib().tn_get_stats(self._h, C.byref(n), C.byref(t)))
        return {"launches": n.value, "precompute_s": t.value}


def observables(bits, logq, logp, groups=None, targets=None):
    """tn_observables (NEXT-1): importance-sampled <Z_v>, the plain
    sample mean of Z_v, and the sector pass rate (plain and weighted). groups: [N] group id per
    vertex (-1 = none) with targets[g] = required number of ones in group g."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    n, N = b.shape
    q = np.ascontiguousarray(logq, dtype=np.float64)
    lp = np.ascontiguousarray(logp, dtype=np.float64)
    zw = np.zeros(N)
    zp = np.zeros(N)
    pr = C.c_double()
    prw = C.c_double()
    if groups is None:
        g = t = None
        ng = 0
    else:
        g = np.ascontiguousarray(groups, dtype=np.int32)
        t = np.ascontiguousarray(targets, dtype=np.int32)
        ng = len(t)
    _check(lib().tn_observables(_ptr(b), _ptr(q), _ptr(lp), n, N, _ptr(g), ng, _ptr(t), _ptr(zw), _ptr(zp),
                                C.byref(pr), C.byref(prw)))
    return {"z_weighted": zw, "z_plain": zp, "pass_rate": pr.value, "pass_rate_weighted": prw.value}


def comm_unique_id() -> bytes:
    """tn_comm_unique_id: a new NCCL unique id (rank 0), to be sent to the other ranks."""
    buf = np.zeros(128, dtype=np.uint8)
    _check(lib().tn_comm_unique_id(_ptr(buf)))
    return buf.tobytes()
