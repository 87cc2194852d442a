"""TEST INFRASTRUCTURE ONLY.  ctypes wrapper around fs_oracle.c (plain single-threaded C).

Every function cites the passage it follows; see fs_oracle.c's header for the readings.
Parity status: all functions pinned by tests/test_oracle_pins.py.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile fs_oracle.c (gcc, -O2, no fast-math, no FP contraction, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u32, u64, i64, dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        L.or_splitmix64_fill.argtypes = [u64, u64, P]
        L.or_splitmix64_fill.restype = None
        L.or_build_cdf.argtypes = [ctypes.c_int, u32, dbl, dbl, P, P, u32, P, P]
        L.or_build_cdf.restype = ctypes.c_int
        L.or_generate_graph.argtypes = [u32, u32, u32, u32, u64, ctypes.c_int, dbl, dbl, P, P, u32,
                                        P, P, P, P]
        L.or_generate_graph.restype = i64
        L.or_generate_graph_ex.argtypes = [u32, u32, u32, u32, u64, ctypes.c_int, dbl, dbl, P, P, u32,
                                           ctypes.c_int, u32, P, P, P, P]
        L.or_generate_graph_ex.restype = i64
        L.or_array_precode.argtypes = [u32, u32, P, P]
        L.or_array_precode.restype = ctypes.c_int32
        L.or_encode_stripe.argtypes = [u32, u32, u32, u64, P, P, P, P, P, P, P]
        L.or_encode_stripe.restype = None
        L.or_encode_stripes.argtypes = [u32, u32, u32, u32, u64, P, P, P, P, P, u64, P, u64, P, u64]
        L.or_encode_stripes.restype = None
        L.or_decode.argtypes = [u32, u32, u32, u64, P, P, P, P, P, P, ctypes.c_int, P, P]
        L.or_decode.restype = i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def splitmix64(seed, count):
    """splitmix64 stream (reading R2): outputs 1..count for the given seed."""
    out = np.zeros(count, dtype=np.uint64)
    lib().or_splitmix64_fill(seed, count, _p(out))
    return out


def build_cdf(dist, K, rsd_c=0.0, rsd_delta=0.0, fin_deg=(), fin_prob=()):
    """Degree support and CDF (readings R7-R10)."""
    fd = np.ascontiguousarray(fin_deg, dtype=np.uint32)
    fp = np.ascontiguousarray(fin_prob, dtype=np.float64)
    cap = max(K, len(fd)) + 1
    deg = np.zeros(cap, dtype=np.uint32)
    cdf = np.zeros(cap, dtype=np.float64)
    n = lib().or_build_cdf(dist, K, rsd_c, rsd_delta, _p(fd), _p(fp), len(fd), _p(deg), _p(cdf))
    if n < 0:
        raise ValueError("invalid degree distribution")
    return deg[:n].copy(), cdf[:n].copy()


class Graph:
    """Precode CSR (p rows over [0,k)) and LT CSR (n rows over [0,K)), rows sorted."""

    def __init__(self, cfg, pre_row_ptr, pre_col, lt_row_ptr, lt_col):
        self.k, self.p, self.n, self.t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
        self.K = self.k + self.p
        self.pre_row_ptr, self.pre_col = pre_row_ptr, pre_col
        self.lt_row_ptr, self.lt_col = lt_row_ptr, lt_col

    @property
    def nnz(self):
        return int(self.lt_row_ptr[-1])

    def lt_row(self, j):
        return self.lt_col[self.lt_row_ptr[j]:self.lt_row_ptr[j + 1]]

    def pre_row(self, i):
        return self.pre_col[self.pre_row_ptr[i]:self.pre_row_ptr[i + 1]]


def array_precode(k, K):
    """Alg 2 check sets for k data of K symbols: (pre_row_ptr, pre_col)."""
    pre_row_ptr = np.zeros(K - k + 1, dtype=np.int32)
    pre_col = np.zeros(max(1, (K - k) * K), dtype=np.int32)
    d = lib().or_array_precode(k, K, _p(pre_row_ptr), _p(pre_col))
    if d < 0:
        raise ValueError("array precode not realizable for (k=%d, K=%d)" % (k, K))
    return pre_row_ptr, pre_col[:(K - k) * d].copy()


def generate_graph(cfg):
    """Graph generation a1 (readings R2-R15; NEXT-2: Alg 2 precode;
    NEXT-4: cfg["files"] = s per-file streams seed + i, reading R17)."""
    k, p, n = cfg["k"], cfg["p"], cfg["n"]
    array = cfg.get("precode", "random") == "array"
    d_p = cfg["d_p"]
    if array:
        d_p = int(np.diff(array_precode(k, k + p)[0])[0])
    K = k + p
    fd = np.ascontiguousarray(cfg.get("fin_deg", ()), dtype=np.uint32)
    fp = np.ascontiguousarray(cfg.get("fin_prob", ()), dtype=np.float64)
    deg, _ = build_cdf(cfg["dist"], K, cfg.get("rsd_c", 0.0), cfg.get("rsd_delta", 0.0), fd, fp)
    cap = n * int(deg.max())
    pre_row_ptr = np.zeros(p + 1, dtype=np.int32)
    pre_col = np.zeros(max(p * d_p, 1), dtype=np.int32)
    lt_row_ptr = np.zeros(n + 1, dtype=np.int32)
    lt_col = np.zeros(cap, dtype=np.int32)
    nnz = lib().or_generate_graph_ex(k, p, d_p, n, cfg["seed"], cfg["dist"], cfg.get("rsd_c", 0.0),
                                     cfg.get("rsd_delta", 0.0), _p(fd), _p(fp), len(fd), 1 if array else 0,
                                     int(cfg.get("files", 1)), _p(pre_row_ptr), _p(pre_col), _p(lt_row_ptr), _p(lt_col))
    if nnz < 0:
        raise ValueError("invalid graph parameters")
    return Graph(cfg, pre_row_ptr, pre_col[:p * d_p].copy(), lt_row_ptr, lt_col[:nnz].copy())


def encode(g, data):
    """Encode a3+a4: data [S,k,t] or [k,t] uint8 -> (checks, coded)."""
    d = np.ascontiguousarray(data, dtype=np.uint8)
    single = d.ndim == 2
    if single:
        d = d[None]
    S = d.shape[0]
    assert d.shape[1:] == (g.k, g.t)
    checks = np.zeros((S, g.p, g.t), dtype=np.uint8)
    coded = np.zeros((S, g.n, g.t), dtype=np.uint8)
    lib().or_encode_stripes(S, g.k, g.p, g.n, g.t, _p(g.pre_row_ptr), _p(g.pre_col),
                            _p(g.lt_row_ptr), _p(g.lt_col), _p(d), g.k * g.t,
                            _p(checks), g.p * g.t, _p(coded), g.n * g.t)
    if single:
        return checks[0], coded[0]
    return checks, coded


def decode(g, recv_mask, coded, use_elim=True):
    """Decoder (Algorithm 1 + precode pass; then GF(2) elimination).
    recv_mask: bool[n]; coded: [n,t] (rows where mask is False are ignored).
    Returns (I [K,t], state [K]: 0 unrecovered, 1 by BP, 2 by elimination)."""
    recv = np.ascontiguousarray(recv_mask, dtype=np.uint8)
    y = np.ascontiguousarray(coded, dtype=np.uint8)
    out = np.zeros((g.K, g.t), dtype=np.uint8)
    state = np.zeros(g.K, dtype=np.uint8)
    r = lib().or_decode(g.k, g.p, g.n, g.t, _p(g.pre_row_ptr), _p(g.pre_col), _p(g.lt_row_ptr),
                        _p(g.lt_col), _p(recv), _p(y), 1 if use_elim else 0, _p(out), _p(state))
    if r < 0:
        raise MemoryError("oracle decode failed")
    return out, state
