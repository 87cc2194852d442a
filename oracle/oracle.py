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
        L.or_cga.argtypes = [u32, u32, P, P, P, P]
        L.or_cga.restype = ctypes.c_int32
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


# ------------------------------------------------------------------ NEXT-3: repair and update
def cga(g):
    """Algorithm 4 (CGA) on B = the LT generator (K x n).  Returns the final
    B (K x n, 0/1), L^{(2,3)} (n x n: column j = the coded symbols of local set j) and the number
    of sweeps.  Dense and slow: small graphs only."""
    K, n = g.K, g.n
    Bt = np.zeros((n, K), dtype=np.uint8)          # column-major: row j of Bt = column j of B
    Lt = np.zeros((n, n), dtype=np.uint8)
    sweeps = lib().or_cga(K, n, _p(g.lt_row_ptr), _p(g.lt_col), _p(Bt), _p(Lt))
    return Bt.T.copy(), Lt.T.copy(), int(sweeps)


CHECKS_M1 = 1      # PAPER.md:247, first method: degree-one coded nodes
CHECKS_M2 = 2      # PAPER.md:248-260, second method: check #1 groups via setXOR (Eq 4)


def local_groups(g, B, L):
    """The local recovery sets of PAPER.md:266-268 from CGA's output: column j of B with weight 0
    -> Group #3 {C_s : l_{s,j} = 1}; weight 1 (symbol x) -> Group #2 (x, {C_s : l_{s,j} = 1});
    weight >= 2 -> no group.  Returns [(kind, x or -1, sorted members, order key j)]."""
    out = []
    for j in range(g.n):
        w = int(B[:, j].sum())
        members = [int(s) for s in np.nonzero(L[:, j])[0]]
        if w == 0:
            out.append((3, -1, members, j))
        elif w == 1:
            out.append((2, int(np.nonzero(B[:, j])[0][0]), members, j))
    return out


def set_xor(*sets):
    """setXOR: symmetric difference of index sets."""
    acc = set()
    for s in sets:
        acc ^= set(s)
    return acc


def derived_groups(g, groups, flags):
    """Extra Group #3 sets.  G_x = the first Group #2 set of symbol x in
    (cardinality, j) order (reading R20).  Method 1: coded node j of degree one
    with neighbour x gives G_x XOR {j}.  Method 2: a check #1 group (members
    of precode check i and the check symbol k+i) whose symbols all have a G_x gives
    setXOR of those G_x (Eq 4).  Empty results are dropped.  Order keys n, n+1, ..."""
    g2 = {}
    for kind, x, mem, j in sorted(groups, key=lambda t: (len(t[2]), t[3])):
        if kind == 2 and x not in g2:
            g2[x] = mem
    out = []
    if flags & CHECKS_M1:
        for j in range(g.n):
            row = list(g.lt_row(j))
            if len(row) == 1 and row[0] in g2:
                d = set_xor(g2[row[0]], [j])
                if d:
                    out.append(d)
    if flags & CHECKS_M2:
        for i in range(g.p):
            grp = [int(m) for m in g.pre_row(i)] + [g.k + i]
            if all(x in g2 for x in grp):
                d = set_xor(*[g2[x] for x in grp])
                if d:
                    out.append(d)
    return [(3, -1, sorted(d), g.n + m) for m, d in enumerate(out)]


def check_data(g, flags=0):
    """The <filename>_check.data integer array: per local set, Group #3 as
    [0, deg, members...], Group #2 as [1, x, deg, members...]; sets ordered by cardinality
    (smallest first), ties by order key (reading R20).  Returns (int32 array,
    number of CGA sweeps)."""
    B, L, sweeps = cga(g)
    groups = local_groups(g, B, L)
    groups = groups + derived_groups(g, groups, flags)
    arr = []
    for kind, x, mem, _ in sorted(groups, key=lambda t: (len(t[2]), t[3])):
        arr += ([0, len(mem)] if kind == 3 else [1, x, len(mem)]) + mem
    return np.array(arr, dtype=np.int32), sweeps


def parse_check_data(arr):
    """Inverse of the format: [(kind, x or -1, members)]."""
    out, i, a = [], 0, [int(v) for v in arr]
    while i < len(a):
        if a[i] == 0:
            d = a[i + 1]
            out.append((3, -1, a[i + 2:i + 2 + d]))
            i += 2 + d
        elif a[i] == 1:
            x, d = a[i + 1], a[i + 2]
            out.append((2, x, a[i + 3:i + 3 + d]))
            i += 3 + d
        else:
            raise ValueError("bad check data flag %d at %d" % (a[i], i))
    return out


def repair_plan(g, arr, erased, want=()):
    """Repair / update / degraded read (reading R21).
    Unknowns: the erased coded symbols (and, for a degraded read, the wanted intermediate
    symbols; the data is not stored).  Local sets from the check data, in array order:
      A  Group #3 set with exactly one unknown member x: x = XOR of the other members
         ("sequentially searches only one unknown over the available local sets").
      B  unknown coded symbol j, ascending: if every neighbour x of j (the base graph) has an
         available Group #2 set G_x (first in array order whose members are all known):
         C_j = XOR over x of XOR(G_x) = XOR of setXOR(G_x ...)   (the Eq 4 construction)
    Rounds of [one A sweep, one B sweep] repeat while either resolves something.  Then
      C  each wanted intermediate x, in the given order: XOR of its first available G_x.
    A source-free recipe stands for the all-zero symbol.  level(x) = 1 + max level of its
    sources (known coded symbols: level 0).
    Returns ([(target kind 'c'|'i', index, sources)], unknown coded set, unresolved wanted)."""
    sets = parse_check_data(arr)
    g3 = [m for kind, _, m in sets if kind == 3]
    g2 = [(x, m) for kind, x, m in sets if kind == 2]
    unknown = set(int(e) for e in erased)
    level, steps = {}, []

    def lv(srcs):
        return 1 + max([level.get(c, 0) for c in srcs] + [0])

    def avail_g2(x):
        for xx, m in g2:
            if xx == x and not any(c in unknown for c in m):
                return m
        return None

    progress = True
    while progress and unknown:
        progress = False
        for mem in g3:                                                       # A
            miss = [c for c in mem if c in unknown]
            if len(miss) == 1:
                x = miss[0]
                srcs = [c for c in mem if c != x]
                level[x] = lv(srcs)
                steps.append(("c", x, srcs))
                unknown.discard(x)
                progress = True
        for j in sorted(unknown):                                            # B
            parts = [avail_g2(int(x)) for x in g.lt_row(j)]
            if all(m is not None for m in parts):
                srcs = sorted(set_xor(*parts))
                level[j] = lv(srcs)
                steps.append(("c", j, srcs))
                unknown.discard(j)
                progress = True
    missing = []
    for x in want:                                                           # C
        m = avail_g2(int(x))
        if m is None:
            missing.append(int(x))
        else:
            steps.append(("i", int(x), list(m)))
    return steps, unknown, missing


def repair(g, arr, erased, coded, want=()):
    """Execute repair_plan on coded [n, t] (erased rows are ignored): returns (coded copy with
    the repaired rows, wanted intermediate symbols [len(want), t], unknown coded set)."""
    steps, unknown, missing = repair_plan(g, arr, erased, want)
    y = np.array(coded, dtype=np.uint8, copy=True)
    inter = {}
    for kind, x, srcs in steps:
        acc = np.zeros(y.shape[1], dtype=np.uint8)
        for c in srcs:
            acc ^= y[c]
        if kind == "c":
            y[x] = acc
        else:
            inter[x] = acc
    I = np.zeros((len(want), y.shape[1]), dtype=np.uint8)
    for r, x in enumerate(want):
        if int(x) in inter:
            I[r] = inter[int(x)]
    return y, I, unknown
