"""Thin Python binding of libfsb200.so (include/fsb.h) -- argument marshalling only.

Every step of the encode runs in the library's CUDA kernels; PyTorch supplies device
memory (uint8 CUDA tensors) and streams.  There is no CPU fallback: if the extension is
missing or a call fails, this module raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSB_LIB selects another build of the same sources (same-box A/B runs, tools/gpu/ab/run_ab.sh);
# the default is the in-tree libfsb200.so that build() writes
LIB_PATH = os.environ.get("FSB_LIB") or os.path.join(_HERE, "libfsb200.so")

FS_OK, FS_EINVAL, FS_EDIST, FS_ENOMEM, FS_ECUDA, FS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
FS_DIST_RSD, FS_DIST_FINITE = 1, 2
FS_PRECODE_RANDOM, FS_PRECODE_ARRAY = 0, 1
FS_GRAPH_HOST_ONLY = 1
FS_DECODE_ELIMINATE = 2
VARIANT_AUTO, VARIANT_SMEM, VARIANT_GLOBAL = 0, 1, 2

# Every symbol include/fsb.h declares (checked by tests/test_capi.py).
EXPORTS = ("fs_graph_create", "fs_graph_from_csr", "fs_graph_csr", "fs_graph_get_info",
           "fs_graph_set_variant", "fs_encode", "fs_encode_stripes", "fs_last_launch_count",
           "fs_free", "fs_last_error", "fs_version", "fs_graph_schedule", "fs_graph_windows", "fs_debug_counters",
           "fs_decode_plan_create", "fs_decode_plan_info", "fs_decode_plan_state", "fs_decode",
           "fs_decode_plan_free", "fs_encode_range", "fs_checks_create", "fs_checks_from_data",
           "fs_checks_data", "fs_checks_info_get", "fs_checks_free", "fs_repair_plan_create",
           "fs_repair_plan_info", "fs_repair_plan_rows", "fs_repair", "fs_repair_plan_free",
           "fs_graph_extend", "fs_encode_host")


class FsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("fsb error %d: %s" % (status, msg))
        self.status = status


class fs_params(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("p", ctypes.c_uint32), ("d_p", ctypes.c_uint32),
                ("n", ctypes.c_uint32), ("t", ctypes.c_uint64), ("dist", ctypes.c_int32),
                ("rsd_c", ctypes.c_double), ("rsd_delta", ctypes.c_double),
                ("fin_deg", ctypes.POINTER(ctypes.c_uint32)),
                ("fin_prob", ctypes.POINTER(ctypes.c_double)), ("fin_len", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("precode", ctypes.c_int32), ("files", ctypes.c_uint32)]


class fs_graph_info(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("p", ctypes.c_uint32), ("d_p", ctypes.c_uint32),
                ("n", ctypes.c_uint32), ("t", ctypes.c_uint64), ("lt_nnz", ctypes.c_uint64),
                ("pre_nnz", ctypes.c_uint64), ("max_degree", ctypes.c_uint32),
                ("variant", ctypes.c_int32), ("smem_eligible", ctypes.c_int32),
                ("smem_bytes", ctypes.c_uint32), ("sched_bytes", ctypes.c_uint32),
                ("sched_steps_max", ctypes.c_uint32), ("sched_steps_avg", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("lt_windows", ctypes.c_uint32)]


class fs_checks_info(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_uint32), ("zero_columns", ctypes.c_uint32),
                ("weight1_columns", ctypes.c_uint32), ("group2", ctypes.c_uint32),
                ("group3", ctypes.c_uint32), ("derived", ctypes.c_uint32), ("len", ctypes.c_uint64)]


class fs_repair_info(ctypes.Structure):
    _fields_ = [("erased", ctypes.c_uint32), ("repaired", ctypes.c_uint32), ("unrepaired", ctypes.c_uint32),
                ("want_missing", ctypes.c_uint32), ("levels", ctypes.c_uint32), ("rows", ctypes.c_uint32),
                ("xor_sources", ctypes.c_uint64)]


class fs_decode_info(ctypes.Structure):
    _fields_ = [("K", ctypes.c_uint32), ("n", ctypes.c_uint32), ("received", ctypes.c_uint32),
                ("recovered", ctypes.c_uint32), ("recovered_data", ctypes.c_uint32),
                ("levels", ctypes.c_uint32), ("rows", ctypes.c_uint32),
                ("max_level_rows", ctypes.c_uint32), ("xor_sources", ctypes.c_uint64),
                ("eliminated", ctypes.c_uint32), ("elim_skipped", ctypes.c_uint32),
                ("inactivated", ctypes.c_uint32), ("work_rows", ctypes.c_uint32)]


_lib = None


def lib():
    """Load libfsb200.so (fails loudly if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libfsb200.so not built at %s (run __graft_entry__.build())" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        P, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
        PP = ctypes.POINTER(ctypes.c_void_p)
        L.fs_graph_create.argtypes = [ctypes.POINTER(fs_params), u32, PP]
        L.fs_graph_from_csr.argtypes = [ctypes.POINTER(fs_params), P, P, P, P, u32, PP]
        L.fs_graph_csr.argtypes = [P, PP, PP, PP, PP, ctypes.POINTER(u64)]
        L.fs_graph_get_info.argtypes = [P, ctypes.POINTER(fs_graph_info)]
        L.fs_graph_set_variant.argtypes = [P, i32]
        L.fs_encode.argtypes = [P, P, P, P, u32, u32, P]
        L.fs_encode_range.argtypes = [P, P, P, P, u32, u32, u64, u64, P]
        L.fs_encode_range.restype = ctypes.c_int
        L.fs_encode_stripes.argtypes = [P, u32, P, u64, P, u64, P, u64, P]
        L.fs_encode_host.argtypes = [P, u32, P, u64, P, u64, P, u64, u32, P]
        L.fs_encode_host.restype = ctypes.c_int
        L.fs_graph_schedule.argtypes = [P, PP, ctypes.POINTER(u64), ctypes.POINTER(u32), PP,
                                        ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(u32)]
        L.fs_graph_windows.argtypes = [P, PP, PP, ctypes.POINTER(u32), ctypes.POINTER(u32)]
        for f in ("fs_graph_create", "fs_graph_from_csr", "fs_graph_csr", "fs_graph_get_info",
                  "fs_graph_set_variant", "fs_encode", "fs_encode_stripes", "fs_graph_schedule",
                  "fs_graph_windows"):
            getattr(L, f).restype = ctypes.c_int
        L.fs_decode_plan_create.argtypes = [P, P, u32, PP]
        L.fs_decode_plan_info.argtypes = [P, ctypes.POINTER(fs_decode_info)]
        L.fs_decode_plan_state.argtypes = [P, PP, PP]
        L.fs_decode.argtypes = [P, u32, P, u64, P, u64, P]
        for f in ("fs_decode_plan_create", "fs_decode_plan_info", "fs_decode_plan_state", "fs_decode"):
            getattr(L, f).restype = ctypes.c_int
        L.fs_decode_plan_free.argtypes = [P]
        L.fs_decode_plan_free.restype = None
        L.fs_checks_create.argtypes = [P, u32, PP]
        L.fs_checks_from_data.argtypes = [P, P, u64, PP]
        L.fs_checks_data.argtypes = [P, PP, ctypes.POINTER(u64)]
        L.fs_checks_info_get.argtypes = [P, ctypes.POINTER(fs_checks_info)]
        L.fs_repair_plan_create.argtypes = [P, P, P, P, u32, u32, PP]
        L.fs_repair_plan_info.argtypes = [P, ctypes.POINTER(fs_repair_info)]
        L.fs_repair_plan_rows.argtypes = [P, PP, ctypes.POINTER(u32), PP, PP, PP]
        L.fs_repair.argtypes = [P, u32, P, u64, P, u64, P]
        L.fs_graph_extend.argtypes = [P, u32, u32, PP]
        for f in ("fs_checks_create", "fs_checks_from_data", "fs_checks_data", "fs_checks_info_get",
                  "fs_repair_plan_create", "fs_repair_plan_info", "fs_repair_plan_rows", "fs_repair",
                  "fs_graph_extend"):
            getattr(L, f).restype = ctypes.c_int
        for f in ("fs_checks_free", "fs_repair_plan_free"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = None
        L.fs_debug_counters.argtypes = [P, u32]
        L.fs_debug_counters.restype = ctypes.c_int
        L.fs_last_launch_count.restype = u32
        L.fs_last_launch_count.argtypes = []
        L.fs_free.argtypes = [P]
        L.fs_free.restype = None
        L.fs_last_error.restype = ctypes.c_char_p
        L.fs_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(st):
    if st != FS_OK:
        raise FsError(st, lib().fs_last_error().decode())


def last_launch_count():
    return int(lib().fs_last_launch_count())


def _ptr(x):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if x is None:
        return None
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not x.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(x.data_ptr())


def _buf(x, name, nbytes, cuda=True, optional=False):
    """Pointer of a caller buffer after checking what the C ABI cannot (it only sees a raw
    pointer): uint8 dtype, placement (CUDA tensor on the current device, or a host tensor),
    contiguity and at least `nbytes` bytes -- an undersized tensor would otherwise be read or
    written past its end by the kernels (or by the D2H copies of fs_encode_host)."""
    import torch
    if x is None:
        if optional:
            return None
        raise ValueError("%s: a tensor is required" % name)
    if x.dtype != torch.uint8:
        raise ValueError("%s: expected dtype uint8, got %s" % (name, x.dtype))
    if cuda:
        if not x.is_cuda:
            raise ValueError("%s: expected a CUDA tensor" % name)
        if x.device.index != torch.cuda.current_device():
            raise ValueError("%s: tensor on cuda:%d, current device is cuda:%d"
                             % (name, x.device.index, torch.cuda.current_device()))
    elif x.is_cuda:
        raise ValueError("%s: expected a host tensor" % name)
    if not x.is_contiguous():
        raise ValueError("%s: expected a contiguous tensor" % name)
    if x.numel() < nbytes:
        raise ValueError("%s: expected %d bytes, got %d" % (name, nbytes, x.numel()))
    return ctypes.c_void_p(x.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_params(cfg):
    """fs_params from a config dict (keys of configs.get())."""
    prm = fs_params()
    prm.k, prm.p, prm.d_p, prm.n, prm.t = cfg["k"], cfg["p"], cfg.get("d_p", 0), cfg["n"], cfg["t"]
    prm.dist = cfg["dist"]
    prm.rsd_c = cfg.get("rsd_c", 0.0)
    prm.rsd_delta = cfg.get("rsd_delta", 0.0)
    fd = np.ascontiguousarray(cfg.get("fin_deg", ()), dtype=np.uint32)
    fp = np.ascontiguousarray(cfg.get("fin_prob", ()), dtype=np.float64)
    prm._keep = (fd, fp)
    if len(fd):
        prm.fin_deg = fd.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        prm.fin_prob = fp.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    prm.fin_len = len(fd)
    prm.seed = cfg["seed"]
    prm.precode = {"random": FS_PRECODE_RANDOM, "array": FS_PRECODE_ARRAY}[cfg.get("precode", "random")]
    prm.files = int(cfg.get("files", 1))
    return prm


class Graph:
    """Owner of an fs_graph handle."""

    def __init__(self, handle, cfg):
        self._h = handle
        self.cfg = dict(cfg)
        self.k, self.p, self.n, self.t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
        self.d_p = cfg.get("d_p", 0)
        self.precode = cfg.get("precode", "random")
        self.K = self.k + self.p

    @classmethod
    def create(cls, cfg, host_only=False):
        """fs_graph_create: seeded generation (+ upload to the current CUDA device)."""
        prm = make_params(cfg)
        h = ctypes.c_void_p()
        _check(lib().fs_graph_create(ctypes.byref(prm), FS_GRAPH_HOST_ONLY if host_only else 0,
                                     ctypes.byref(h)))
        return cls(h, cfg)

    @classmethod
    def from_csr(cls, cfg, pre_row_ptr, pre_col, lt_row_ptr, lt_col, host_only=False):
        """fs_graph_from_csr (e.g. after an NCCL broadcast of the CSR)."""
        prm = make_params(cfg)
        arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in (pre_row_ptr, pre_col, lt_row_ptr, lt_col)]
        ptrs = [a.ctypes.data_as(ctypes.c_void_p) if a.size else None for a in arrs]
        h = ctypes.c_void_p()
        _check(lib().fs_graph_from_csr(ctypes.byref(prm), *ptrs, FS_GRAPH_HOST_ONLY if host_only else 0,
                                       ctypes.byref(h)))
        return cls(h, cfg)

    def csr(self):
        """(pre_row_ptr, pre_col, lt_row_ptr, lt_col) as numpy int32 copies."""
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        nnz = ctypes.c_uint64()
        _check(lib().fs_graph_csr(self._h, *[ctypes.byref(x) for x in ptrs], ctypes.byref(nnz)))

        def arr(p, n):
            if n == 0 or not p.value:
                return np.zeros(0, np.int32)
            return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), (n,)).copy()

        pre_rp = arr(ptrs[0], self.p + 1)
        pre_c = arr(ptrs[1], int(pre_rp[-1]) if self.p else 0)
        lt_rp = arr(ptrs[2], self.n + 1)
        lt_c = arr(ptrs[3], int(nnz.value))
        return pre_rp, pre_c, lt_rp, lt_c

    def info(self):
        inf = fs_graph_info()
        _check(lib().fs_graph_get_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in fs_graph_info._fields_}

    def schedule(self):
        """(words uint32[nwords], cont_base, warp_info uint32[nwarps,3], kpad, zero_even) of the
        SMEM schedule (copies; format in include/fsb.h)."""
        w, wi = ctypes.c_void_p(), ctypes.c_void_p()
        nw = ctypes.c_uint64()
        cb, nwarps, kpad, z0 = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib().fs_graph_schedule(self._h, ctypes.byref(w), ctypes.byref(nw), ctypes.byref(cb),
                                       ctypes.byref(wi), ctypes.byref(nwarps), ctypes.byref(kpad),
                                       ctypes.byref(z0)))
        words = np.ctypeslib.as_array(ctypes.cast(w, ctypes.POINTER(ctypes.c_uint32)), (nw.value,)).copy()
        info = np.ctypeslib.as_array(ctypes.cast(wi, ctypes.POINTER(ctypes.c_uint32)),
                                     (3 * nwarps.value,)).copy()
        return words, cb.value, info.reshape(-1, 3), kpad.value, z0.value

    def windows(self):
        """(hdr uint32[count, 2], ent uint32[count, entries]) of the GLOBAL kernel's LT edge
        windows (copies; format in include/fsb.h)."""
        hp, ep = ctypes.c_void_p(), ctypes.c_void_p()
        cnt, ne = ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib().fs_graph_windows(self._h, ctypes.byref(hp), ctypes.byref(ep), ctypes.byref(cnt),
                                      ctypes.byref(ne)))
        hdr = np.ctypeslib.as_array(ctypes.cast(hp, ctypes.POINTER(ctypes.c_uint32)), (2 * cnt.value,)).copy()
        ent = np.ctypeslib.as_array(ctypes.cast(ep, ctypes.POINTER(ctypes.c_uint32)),
                                    (cnt.value * ne.value,)).copy()
        return hdr.reshape(-1, 2), ent.reshape(cnt.value, ne.value)

    def extend(self, extra_files, host_only=False):
        """fs_graph_extend (update): the graph with extra_files more output files."""
        s = max(int(self.cfg.get("files", 1)), 1)
        cfg = dict(self.cfg, n=self.n + extra_files * (self.n // s), files=s + extra_files)
        h = ctypes.c_void_p()
        _check(lib().fs_graph_extend(self._h, extra_files, FS_GRAPH_HOST_ONLY if host_only else 0,
                                     ctypes.byref(h)))
        return Graph(h, cfg)

    def set_variant(self, variant):
        _check(lib().fs_graph_set_variant(self._h, variant))

    def encode(self, data, checks, coded, row_begin=0, row_end=None, stream=None):
        """fs_encode: one stripe, coded rows [row_begin, row_end) into `coded`."""
        row_end = self.n if row_end is None else row_end
        t = self.t
        rows = max(int(row_end) - int(row_begin), 0)
        _check(lib().fs_encode(self._h, _buf(data, "data", self.k * t), self._checks_ptr(checks, 1, True),
                               _buf(coded, "coded", rows * t), row_begin, row_end, _stream(stream)))

    def _checks_ptr(self, checks, S, cuda):
        # None goes through: the library rejects a missing checks buffer when p > 0 (FS_EINVAL)
        return _buf(checks, "checks", S * self.p * self.t, cuda=cuda, optional=True)

    def encode_range(self, data, checks, coded, row_begin, row_end, col_begin, col_end, stream=None):
        """fs_encode_range: rows [row_begin, row_end) and bytes [col_begin, col_end) of one stripe."""
        t = self.t
        rows = max(int(row_end) - int(row_begin), 0)
        _check(lib().fs_encode_range(self._h, _buf(data, "data", self.k * t), self._checks_ptr(checks, 1, True),
                                     _buf(coded, "coded", rows * t), row_begin, row_end, col_begin, col_end,
                                     _stream(stream)))

    def encode_stripes(self, data, checks, coded, stream=None):
        """fs_encode_stripes over contiguous [S,k,t] / [S,p,t] / [S,n,t] uint8 CUDA tensors."""
        S = data.shape[0]
        t = self.t
        _check(lib().fs_encode_stripes(self._h, S, _buf(data, "data", S * self.k * t), self.k * t,
                                       self._checks_ptr(checks, S, True), self.p * t,
                                       _buf(coded, "coded", S * self.n * t), self.n * t, _stream(stream)))

    def encode_host(self, data, checks, coded, chunks=0, stream=None):
        """fs_encode_host over contiguous [S,k,t] / [S,p,t] / [S,n,t] uint8 CPU tensors (pinned for
        overlap): the library stages them through its own device buffers.  Asynchronous on
        `stream` (the current stream by default): synchronise it before using the outputs."""
        S = data.shape[0]
        t = self.t
        _check(lib().fs_encode_host(self._h, S, _buf(data, "data", S * self.k * t, cuda=False), self.k * t,
                                    self._checks_ptr(checks, S, False), self.p * t,
                                    _buf(coded, "coded", S * self.n * t, cuda=False), self.n * t, chunks,
                                    _stream(stream)))

    def encode_stripes_raw(self, S, data_ptr, data_stride, checks_ptr, checks_stride, coded_ptr,
                           coded_stride, stream=None):
        """fs_encode_stripes with explicit device pointers and byte strides."""
        _check(lib().fs_encode_stripes(self._h, S, ctypes.c_void_p(data_ptr), data_stride,
                                       ctypes.c_void_p(checks_ptr) if checks_ptr else None,
                                       checks_stride, ctypes.c_void_p(coded_ptr), coded_stride,
                                       _stream(stream)))

    def free(self):
        if self._h:
            lib().fs_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DecodePlan:
    """Owner of an fs_decode_plan: Alg 5 (DPG) levels for a graph and a received set."""

    def __init__(self, graph, received, host_only=False, eliminate=False):
        rv = np.ascontiguousarray(np.asarray(received, dtype=bool).astype(np.uint8))
        if rv.shape != (graph.n,):
            raise ValueError("received must have n entries")
        self.graph = graph
        self._h = None
        h = ctypes.c_void_p()
        flags = (FS_GRAPH_HOST_ONLY if host_only else 0) | (FS_DECODE_ELIMINATE if eliminate else 0)
        _check(lib().fs_decode_plan_create(graph._h, rv.ctypes.data_as(ctypes.c_void_p), flags, ctypes.byref(h)))
        self._h = h

    def info(self):
        inf = fs_decode_info()
        _check(lib().fs_decode_plan_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in fs_decode_info._fields_}

    def state(self):
        """(state uint8[K], level_of int32[K]) copies."""
        s, lv = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().fs_decode_plan_state(self._h, ctypes.byref(s), ctypes.byref(lv)))
        K = self.graph.K
        st = np.ctypeslib.as_array(ctypes.cast(s, ctypes.POINTER(ctypes.c_uint8)), (K,)).copy()
        lev = np.ctypeslib.as_array(ctypes.cast(lv, ctypes.POINTER(ctypes.c_int32)), (K,)).copy()
        return st, lev

    def decode(self, coded, inter, stream=None):
        """fs_decode over contiguous [S,n,t] coded and [S,K,t] intermediate uint8 CUDA tensors."""
        S = coded.shape[0]
        t = self.graph.t
        _check(lib().fs_decode(self._h, S, _buf(coded, "coded", S * self.graph.n * t), self.graph.n * t,
                               _buf(inter, "inter", S * self.graph.K * t), self.graph.K * t, _stream(stream)))

    def free(self):
        if self._h:
            lib().fs_decode_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


CHECKS_M1, CHECKS_M2 = 1, 2


class Checks:
    """Owner of an fs_checks: CGA (Alg 4) local sets in the <filename>_check.data format."""

    def __init__(self, handle, graph):
        self._h = handle
        self.graph = graph

    @classmethod
    def create(cls, graph, flags=0):
        h = ctypes.c_void_p()
        _check(lib().fs_checks_create(graph._h, flags, ctypes.byref(h)))
        return cls(h, graph)

    @classmethod
    def from_data(cls, graph, data):
        a = np.ascontiguousarray(data, dtype=np.int32)
        h = ctypes.c_void_p()
        _check(lib().fs_checks_from_data(graph._h, a.ctypes.data_as(ctypes.c_void_p) if a.size else None,
                                         a.size, ctypes.byref(h)))
        return cls(h, graph)

    def data(self):
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        _check(lib().fs_checks_data(self._h, ctypes.byref(p), ctypes.byref(n)))
        if not n.value:
            return np.zeros(0, np.int32)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), (n.value,)).copy()

    def info(self):
        inf = fs_checks_info()
        _check(lib().fs_checks_info_get(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in fs_checks_info._fields_}

    def free(self):
        if self._h:
            lib().fs_checks_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class RepairPlan:
    """Owner of an fs_repair_plan (repair / update / degraded read, NEXT-3)."""

    def __init__(self, graph, checks, erased, want=(), host_only=False):
        er = np.ascontiguousarray(np.asarray(erased, dtype=bool).astype(np.uint8))
        if er.shape != (graph.n,):
            raise ValueError("erased must have n entries")
        w = np.ascontiguousarray(want, dtype=np.uint32)
        self.graph = graph
        self._h = None
        h = ctypes.c_void_p()
        _check(lib().fs_repair_plan_create(graph._h, checks._h, er.ctypes.data_as(ctypes.c_void_p),
                                           w.ctypes.data_as(ctypes.c_void_p) if w.size else None, w.size,
                                           FS_GRAPH_HOST_ONLY if host_only else 0, ctypes.byref(h)))
        self._h = h

    def info(self):
        inf = fs_repair_info()
        _check(lib().fs_repair_plan_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in fs_repair_info._fields_}

    def rows(self):
        """(level_ptr, target, src_ptr, src) copies; see include/fsb.h for the flags."""
        lp, tg, sp, sr = (ctypes.c_void_p() for _ in range(4))
        nl = ctypes.c_uint32()
        _check(lib().fs_repair_plan_rows(self._h, ctypes.byref(lp), ctypes.byref(nl), ctypes.byref(tg),
                                         ctypes.byref(sp), ctypes.byref(sr)))

        def arr(p, n, ct):
            if n == 0 or not p.value:
                return np.zeros(0, dtype=np.dtype(ct))
            return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ct)), (n,)).copy()

        level_ptr = arr(lp, nl.value + 1, ctypes.c_uint32)
        rows = int(level_ptr[-1]) if len(level_ptr) else 0
        target = arr(tg, rows, ctypes.c_int32)
        src_ptr = arr(sp, rows + 1, ctypes.c_int32)
        src = arr(sr, int(src_ptr[-1]) if rows else 0, ctypes.c_uint32)
        return level_ptr, target, src_ptr, src

    def repair(self, coded, inter=None, stream=None):
        """fs_repair in place over contiguous [S,n,t] coded (and [S,K,t] inter) CUDA tensors."""
        S = coded.shape[0]
        t = self.graph.t
        _check(lib().fs_repair(self._h, S, _buf(coded, "coded", S * self.graph.n * t), self.graph.n * t,
                               _buf(inter, "inter", S * self.graph.K * t, optional=True), self.graph.K * t,
                               _stream(stream)))

    def free(self):
        if self._h:
            lib().fs_repair_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def debug_counters(n=64):
    """fs_debug_counters (profiling aid, FSB_DEBUG=2): uint64 counters, cleared on read."""
    out = (ctypes.c_uint64 * n)()
    _check(lib().fs_debug_counters(ctypes.cast(out, ctypes.c_void_p), n))
    return [int(x) for x in out]


def version():
    return lib().fs_version().decode()
