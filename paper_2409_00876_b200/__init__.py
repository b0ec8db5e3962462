"""paper_2409_00876_b200 — B200-native PG-SGD pangenome layout (the hot path
of /root/reference/proj, pglayout) behind the reference's own layout API.

Everything computes in libpgl_b200.so (sm_100a CUDA + C++ host driver),
reached through the C-ABI declared in include/pgl_b200.h. This module is a
thin ctypes mirror of the reference's C++ interface for Python callers
(tests, bench): same names, same argument meaning, same exception classes
(include/pglayout/errors.hpp:31-44). There is no CPU fallback: if the
native library is missing the import fails.

Reference interfaces mirrored (file:line under /root/reference/proj):
    LayoutConfig            include/pglayout/engine.hpp:13-23
    RunStats                include/pglayout/engine.hpp:61-70
    run_layout              include/pglayout/engine.hpp:80-82
    run_layout_reuse        include/pglayout/engine.hpp:86-88
    make_schedule           include/pglayout/engine.hpp:44
    init_layout             include/pglayout/layout.hpp:91
    StressReport            include/pglayout/metrics.hpp:13-20
    sampled_path_stress     include/pglayout/metrics.hpp:49-51
    build_graph             include/pglayout/graph.hpp:91-93
    generate_synthetic_pangenome  include/pglayout/synthetic.hpp:15-18
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, fields
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "LayoutConfig", "LayoutExt", "LayoutDiag", "RunStats", "StressReport", "PangenomeGraph", "DeviceGraph",
    "Timing", "run_layout", "run_layout_reuse", "sampled_path_stress", "make_schedule",
    "init_layout", "build_graph", "generate_synthetic_pangenome", "layout_shards", "shard_plan",
    "device_count", "Error", "MODE_HOGWILD", "MODE_REPLAY", "COORD_F32", "COORD_F64",
    "SPS_COUNTER", "SPS_STREAM", "SAMPLING_TILES", "SAMPLING_IID", "LIB_PATH",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGL_B200_LIB", os.path.join(_HERE, "libpgl_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libpgl_b200.so not found at {LIB_PATH}: build it with "
        f"`python -c 'import __graft_entry__ as g; g.build()'` (make -C {_HERE}/csrc). "
        "There is no CPU fallback for the layout path.")

_lib = C.CDLL(LIB_PATH)

MODE_HOGWILD, MODE_REPLAY = 0, 1
COORD_F32, COORD_F64, COORD_F32_ANCHORED, COORD_AUTO = 0, 1, 2, 3
SPS_COUNTER, SPS_STREAM = 0, 1
SAMPLING_TILES, SAMPLING_IID, SAMPLING_AUTO = 0, 1, 2
ORDER_AUTO, ORDER_SPREAD, ORDER_FRONTS, ORDER_RANDOM = 0, 1, 2, 3

_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


# ---- C structs (include/pgl_b200.h) -----------------------------------------

class _Cfg(C.Structure):
    _fields_ = [("global_seed", C.c_uint64), ("n_iters", C.c_uint32), ("threads", C.c_uint32),
                ("batch_size", C.c_uint32), ("_pad0", C.c_uint32), ("zipf_theta", C.c_double),
                ("zipf_space_max", C.c_uint64), ("eta_min_eps", C.c_double),
                ("drf", C.c_uint32), ("srf", C.c_uint32)]


class _Ext(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("mode", C.c_uint32), ("coord_precision", C.c_uint32),
                ("max_warps", C.c_uint32), ("block_threads", C.c_uint32), ("l2_persist", C.c_uint32),
                ("kernel_variant", C.c_uint32), ("l2_fetch_bytes", C.c_uint32),
                ("sampling", C.c_uint32), ("unit_order", C.c_uint32), ("front_warps", C.c_uint32),
                ("pair_window", C.c_uint32), ("record_hint", C.c_uint32), ("hop_lanes", C.c_uint32),
                ("reuse_shuffle", C.c_uint32), ("unit_len", C.c_uint32),
                ("diag", C.c_void_p)]


class _Diag(C.Structure):
    _fields_ = [("primary_visits", C.POINTER(C.c_uint32)), ("zipf_draws", C.POINTER(C.c_uint64)),
                ("zipf_draws_len", C.c_uint32), ("_pad", C.c_uint32), ("outcomes", C.c_uint64 * 4)]


class _PathStep(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("node_id", C.c_uint32), ("seq_len", C.c_uint32),
                ("orient", C.c_uint8), ("_pad", C.c_uint8 * 7)]


class _View(C.Structure):
    _fields_ = [("n_nodes", C.c_uint64), ("node_len", _u64p), ("n_paths", C.c_uint32),
                ("_pad0", C.c_uint32), ("path_steps", C.POINTER(C.c_void_p)),
                ("path_n_steps", _u64p), ("path_total_len", _u64p)]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "primary_steps", "updates_attempted", "updates_applied", "updates_skipped",
        "batches_first_half", "batches_first_half_cooling", "batches_second_half",
        "batches_second_half_cooling")]


class _Report(C.Structure):
    _fields_ = [("mean", C.c_double), ("n", C.c_uint64), ("std_dev", C.c_double),
                ("ci_low", C.c_double), ("ci_high", C.c_double), ("skipped", C.c_uint64)]


class _Info(C.Structure):
    _fields_ = [("n_nodes", C.c_uint64), ("n_paths", C.c_uint32), ("device", C.c_uint32),
                ("total_steps", C.c_uint64), ("total_nucleotides", C.c_uint64),
                ("max_path_len", C.c_uint64), ("device_bytes", C.c_uint64),
                ("usable", C.c_uint32), ("_pad0", C.c_uint32)]


class _Timing(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("init_ms", C.c_double), ("total_ms", C.c_double),
                ("device_ms", C.c_double), ("launches", C.c_uint32), ("grid_blocks", C.c_uint32), ("block_threads", C.c_uint32),
                ("nonfinite_nodes", C.c_uint32), ("device_threads", C.c_uint64),
                ("coord_kind", C.c_uint32), ("variant", C.c_uint32)]


class _GfaInfo(C.Structure):
    _fields_ = [("n_nodes", C.c_uint64), ("n_edges", C.c_uint64), ("total_steps", C.c_uint64),
                ("skipped_records", C.c_uint64), ("n_paths", C.c_uint32), ("_pad0", C.c_uint32)]


EDGE_DTYPE = np.dtype({"names": ["from", "to", "from_end", "to_end"],
                       "formats": [np.uint32, np.uint32, np.uint8, np.uint8],
                       "offsets": [0, 4, 8, 9], "itemsize": 16})

_CB = C.CFUNCTYPE(C.c_int, C.c_uint32, _f64p, C.c_double, C.c_double, C.c_void_p)

assert C.sizeof(_Cfg) == 56 and C.sizeof(_PathStep) == 24 and C.sizeof(_Ext) == 72 and C.sizeof(_Diag) == 56

_vp = C.c_void_p
_sig = {
    "pgl_last_error": ([], C.c_char_p), "pgl_last_error_type": ([], C.c_int),
    "pgl_abi_version": ([], C.c_int), "pgl_device_count": ([], C.c_int),
    "pgl_transfer_bytes": ([_u64p, _u64p], C.c_int),
    "pgl_graph_all_finite": ([_vp, _f64p, _u64p, _u64p], C.c_int),
    "pgl_layout_run": ([C.c_int, C.POINTER(_View), C.POINTER(_Cfg), C.POINTER(_Ext), C.c_int, _CB,
                        C.c_int, _vp, _f64p, C.POINTER(_Stats)], C.c_int),
    "pgl_graph_create": ([C.c_int, C.POINTER(_View), C.POINTER(_vp)], C.c_int),
    "pgl_graph_destroy": ([_vp], C.c_int),
    "pgl_graph_info_get": ([_vp, C.POINTER(_Info)], C.c_int),
    "pgl_graph_layout": ([_vp, C.POINTER(_Cfg), C.POINTER(_Ext), C.c_int, _CB, C.c_int, _vp, _f64p,
                          C.POINTER(_Stats)], C.c_int),
    "pgl_graph_export_index": ([_vp, _u64p, C.POINTER(C.c_uint32), _u64p], C.c_int),
    "pgl_graph_last_timing": ([_vp, C.POINTER(_Timing)], C.c_int),
    "pgl_sampled_path_stress": ([C.c_int, C.POINTER(_View), _f64p, C.c_uint64, C.c_uint32, C.c_uint32,
                                 C.POINTER(_Report)], C.c_int),
    "pgl_graph_stress": ([_vp, _f64p, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(_Report), _f64p],
                         C.c_int),
    "pgl_exact_path_stress": ([C.c_int, C.POINTER(_View), _f64p, C.POINTER(_Report)], C.c_int),
    "pgl_graph_exact_stress": ([_vp, _f64p, C.POINTER(_Report), _f64p], C.c_int),
    "pgl_make_schedule": ([C.POINTER(_View), C.POINTER(_Cfg), _f64p], C.c_int),
    "pgl_gfa_parse_file": ([C.c_char_p, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "pgl_graph_create_gfa": ([C.c_int, C.c_char_p, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "pgl_gfa_parse_buffer": ([C.c_char_p, C.c_uint64, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "pgl_gfa_info_get": ([_vp, C.POINTER(_GfaInfo)], C.c_int),
    "pgl_gfa_view": ([_vp, C.POINTER(_View)], C.c_int),
    "pgl_gfa_edges": ([_vp, _vp], C.c_int),
    "pgl_gfa_path_name": ([_vp, C.c_uint32], C.c_char_p),
    "pgl_gfa_free": ([_vp], C.c_int),
    "pgl_layout_write_tsv": ([C.c_char_p, _f64p, C.c_uint64, C.c_uint32], C.c_int),
    "pgl_layout_read_tsv": ([C.c_char_p, C.c_uint32, _u64p, C.POINTER(_f64p)], C.c_int),
    "pgl_free": ([_vp], None),
    "pgl_init_layout": ([C.POINTER(_View), C.c_uint64, _f64p], C.c_int),
    "pgl_layout_shards": ([C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.POINTER(_View)),
                           C.POINTER(_Cfg), C.POINTER(_Ext), C.POINTER(_f64p), C.POINTER(_Stats),
                           _f64p, C.POINTER(C.c_int)], C.c_int),
    "pgl_shard_plan": ([C.c_int, C.c_int, C.POINTER(C.POINTER(_View)), C.POINTER(_Cfg),
                        C.POINTER(C.c_int), _f64p, _f64p], C.c_int),
    "pgl_synthetic_generate": ([C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.POINTER(_vp)],
                               C.c_int),
    "pgl_synthetic_view": ([_vp, C.POINTER(_View)], C.c_int),
    "pgl_synthetic_generate_nested": ([C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                       C.POINTER(_vp)], C.c_int),
    "pgl_synthetic_free": ([_vp], C.c_int),
    "pgl_layout_config_default": ([C.POINTER(_Cfg)], None),
    "pgl_layout_ext_default": ([C.POINTER(_Ext)], None),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

if _lib.pgl_abi_version() != 1:
    raise ImportError("libpgl_b200.so ABI version mismatch")


# ---- errors: errors.hpp:10-42 -------------------------------------------------

class Error(RuntimeError):
    """Base of the typed failures; `kind` is the reference ErrorKind
    ("usage" -> exit 1, "input" -> 2, "internal" -> 3)."""
    kind = "internal"


def _mk(name, kind):
    return type(name, (Error,), {"kind": kind})


InvalidParameter = _mk("InvalidParameter", "usage")
UnknownNode = _mk("UnknownNode", "input")
EmptyPath = _mk("EmptyPath", "input")
IndexOutOfRange = _mk("IndexOutOfRange", "internal")
EmptyGraph = _mk("EmptyGraph", "input")
DegenerateGraph = _mk("DegenerateGraph", "input")
MalformedLine = _mk("MalformedLine", "input")
UnknownSegment = _mk("UnknownSegment", "input")
NoPaths = _mk("NoPaths", "input")
NonFiniteCoordinate = _mk("NonFiniteCoordinate", "input")
MalformedRow = _mk("MalformedRow", "input")
CountMismatch = _mk("CountMismatch", "input")
ZeroReference = _mk("ZeroReference", "input")
CorpusTooLarge = _mk("CorpusTooLarge", "input")
CudaError = _mk("CudaError", "internal")
CallbackAbort = _mk("CallbackAbort", "internal")
_BY_TYPE = {1: InvalidParameter, 2: UnknownNode, 3: EmptyPath, 4: IndexOutOfRange, 5: EmptyGraph,
            6: DegenerateGraph, 7: MalformedLine, 8: UnknownSegment, 9: NoPaths,
            10: NonFiniteCoordinate, 11: MalformedRow, 12: CountMismatch, 13: ZeroReference,
            14: CorpusTooLarge, 100: CudaError, 101: CallbackAbort}
__all__ += [c.__name__ for c in _BY_TYPE.values()]


def _check(rc: int):
    if rc != 0:
        t = _lib.pgl_last_error_type()
        raise _BY_TYPE.get(t, Error)(_lib.pgl_last_error().decode())


# ---- value types ----------------------------------------------------------------

@dataclass
class LayoutConfig:
    """engine.hpp:13-23, same fields and defaults."""
    global_seed: int = 42
    n_iters: int = 30
    threads: int = 1
    batch_size: int = 32
    zipf_theta: float = 0.99
    zipf_space_max: int = 1000
    eta_min_eps: float = 0.01
    drf: int = 1
    srf: int = 1

    def _c(self) -> _Cfg:
        c = _Cfg()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name in ("zipf_theta", "eta_min_eps"):
                setattr(c, f.name, float(v))
            else:
                if int(v) < 0:
                    raise InvalidParameter(f"InvalidParameter: {f.name} must be non-negative")
                setattr(c, f.name, int(v))
        return c


@dataclass
class LayoutExt:
    """B200 knobs outside LayoutConfig (pgl_layout_ext)."""
    mode: int = MODE_HOGWILD
    coord_precision: int = COORD_AUTO
    max_warps: int = 0
    block_threads: int = 0
    l2_persist: int = 0
    l2_fetch_bytes: int = 0
    kernel_variant: int = 0
    sampling: int = 2  # SAMPLING_AUTO: tiles where the graph fills the GPU, i.i.d. where the cap binds
    unit_order: int = 0  # ORDER_AUTO
    front_warps: int = 0
    pair_window: int = 0  # 0 auto (= 3), 1 independent draws, 2 shared uniform window, 3 window + shared Zipf hop
    record_hint: int = 0  # 0 evict_first, 1 evict_normal
    hop_lanes: int = 0  # lanes per shared Zipf hop (pair_window 3), 0 = auto
    reuse_shuffle: int = 0  # drf > 1 extras by warp-shuffle reuse (paper §7.4)
    unit_len: int = 0  # lean kernel: picks per unit (0 = 32; below 32 needs unit_order=ORDER_RANDOM)
    # sampler diagnostics (pgl_layout_diag), counted by the Hogwild kernels
    diag: Optional["LayoutDiag"] = None

    def _c(self) -> _Ext:
        e = _Ext()
        _lib.pgl_layout_ext_default(C.byref(e))
        e.mode, e.coord_precision = self.mode, self.coord_precision
        e.max_warps, e.block_threads, e.l2_persist = self.max_warps, self.block_threads, self.l2_persist
        e.l2_fetch_bytes = self.l2_fetch_bytes
        e.kernel_variant = self.kernel_variant
        e.sampling = self.sampling
        e.unit_order, e.front_warps = self.unit_order, self.front_warps
        e.pair_window, e.record_hint, e.hop_lanes = self.pair_window, self.record_hint, self.hop_lanes
        e.reuse_shuffle = self.reuse_shuffle
        e.unit_len = self.unit_len
        if self.diag is not None:
            e.diag = C.addressof(self.diag._c())
        return e


class LayoutDiag:
    """Sampler diagnostics (pgl_layout_diag): per-step primary visit counts,
    the histogram of Zipf hops drawn, and the primary updates' outcome counts
    {uniform attempted, uniform applied, cooling attempted, cooling applied},
    counted inside the Hogwild kernels. Pass as LayoutExt(diag=...); the
    arrays are filled when the layout returns."""

    def __init__(self, total_steps: int = 0, zipf_len: int = 0):
        self.primary_visits = np.zeros(total_steps, np.uint32) if total_steps else None
        self.zipf_draws = np.zeros(zipf_len, np.uint64) if zipf_len else None
        self._s = _Diag()

    def _c(self) -> "_Diag":
        s = self._s
        if self.primary_visits is not None:
            s.primary_visits = self.primary_visits.ctypes.data_as(C.POINTER(C.c_uint32))
        if self.zipf_draws is not None:
            s.zipf_draws = self.zipf_draws.ctypes.data_as(C.POINTER(C.c_uint64))
            s.zipf_draws_len = self.zipf_draws.size
        return s

    @property
    def outcomes(self):
        return [int(x) for x in self._s.outcomes]


@dataclass
class RunStats:
    """engine.hpp:61-70."""
    primary_steps: int = 0
    updates_attempted: int = 0
    updates_applied: int = 0
    updates_skipped: int = 0
    batches_first_half: int = 0
    batches_first_half_cooling: int = 0
    batches_second_half: int = 0
    batches_second_half_cooling: int = 0

    def _load(self, s: _Stats):
        for f in fields(self):
            setattr(self, f.name, int(getattr(s, f.name)))


@dataclass
class StressReport:
    """metrics.hpp:13-20."""
    mean: float = 0.0
    n: int = 0
    std_dev: float = 0.0
    ci_low: float = 0.0
    ci_high: float = 0.0
    skipped: int = 0

    @classmethod
    def _of(cls, r: _Report):
        return cls(r.mean, int(r.n), r.std_dev, r.ci_low, r.ci_high, int(r.skipped))

    def tsv(self) -> str:
        """report_tsv (metrics.cpp:44-50)."""
        return "%.9g\t%d\t%.9g\t%.9g\t%.9g\t%d" % (self.mean, self.n, self.std_dev, self.ci_low,
                                                   self.ci_high, self.skipped)


@dataclass
class Timing:
    kernel_ms: float
    init_ms: float
    total_ms: float
    device_ms: float
    launches: int
    grid_blocks: int
    block_threads: int
    device_threads: int
    nonfinite_nodes: int = 0
    coord_kind: int = 0
    variant: int = 0  # tile kernel variant that ran (0: i.i.d. kernel or replay)


# ---- graphs -----------------------------------------------------------------------

PATH_STEP_DTYPE = np.dtype({"names": ["offset", "node_id", "seq_len", "orient"],
                            "formats": [np.uint64, np.uint32, np.uint32, np.uint8],
                            "offsets": [0, 8, 12, 16], "itemsize": 24})


class PangenomeGraph:
    """A built graph in the reference's host format (graph.hpp:61-88): node
    lengths plus, per path, a PathStep array (24-byte records). Owns the
    memory; `view()` is the borrowed pgl_graph_view handed to the C-ABI."""

    def __init__(self, node_len, path_steps: Sequence[np.ndarray], path_names=None, _owner=None):
        self.node_len = np.ascontiguousarray(node_len, np.uint64)
        self.path_steps = [np.ascontiguousarray(p) for p in path_steps]
        for p in self.path_steps:
            assert p.dtype == PATH_STEP_DTYPE
        self.path_names = path_names or [f"p{k}" for k in range(len(self.path_steps))]
        self._owner = _owner
        self._build_view()

    def _build_view(self):
        P = len(self.path_steps)
        self._ptrs = (C.c_void_p * max(P, 1))(*[p.ctypes.data for p in self.path_steps])
        self.path_n_steps = np.array([len(p) for p in self.path_steps], np.uint64)
        self.path_total_len = np.array(
            [int(p["offset"][-1]) + int(p["seq_len"][-1]) if len(p) else 0 for p in self.path_steps],
            np.uint64)
        self._view = _View(len(self.node_len), self.node_len.ctypes.data_as(_u64p), P, 0,
                           C.cast(self._ptrs, C.POINTER(C.c_void_p)),
                           self.path_n_steps.ctypes.data_as(_u64p),
                           self.path_total_len.ctypes.data_as(_u64p))

    @classmethod
    def _from_view(cls, v: _View, owner):
        P = v.n_paths
        node_len = np.ctypeslib.as_array(v.node_len, (v.n_nodes,)) if v.n_nodes else np.zeros(0, np.uint64)
        steps = []
        for p in range(P):
            n = v.path_n_steps[p]
            buf = (C.c_char * (24 * n)).from_address(v.path_steps[p])
            steps.append(np.frombuffer(buf, PATH_STEP_DTYPE, n))
        g = cls.__new__(cls)
        g.node_len, g.path_steps, g._owner = node_len, steps, owner
        g.path_names = [f"hap{k}" for k in range(P)]
        g._build_view()
        return g

    def view(self) -> _View:
        return self._view

    @property
    def n_nodes(self) -> int:
        return len(self.node_len)

    def node_count(self) -> int:
        return self.n_nodes

    @property
    def n_paths(self) -> int:
        return len(self.path_steps)

    def total_steps(self) -> int:
        return int(self.path_n_steps.sum())

    def total_nucleotides(self) -> int:
        return int(self.node_len.sum())

    def cum_steps(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.path_n_steps)]).astype(np.uint64)

    def host_bytes(self) -> int:
        return 24 * self.total_steps() + 8 * self.n_nodes


class _SynthOwner:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            _lib.pgl_synthetic_free(self.h)
            self.h = None


def generate_synthetic_pangenome(seed: int, backbone_nodes: int, n_paths: int,
                                 variant_rate: float) -> PangenomeGraph:
    """synthetic.cpp:24-120 (native generator; same nodes, walks, offsets)."""
    h = C.c_void_p()
    _check(_lib.pgl_synthetic_generate(seed, backbone_nodes, n_paths, variant_rate, C.byref(h)))
    owner = _SynthOwner(h)
    v = _View()
    _check(_lib.pgl_synthetic_view(h, C.byref(v)))
    return PangenomeGraph._from_view(v, owner)


class _GfaOwner:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            _lib.pgl_gfa_free(self.h)
            self.h = None


def _gfa_graph(h) -> PangenomeGraph:
    owner = _GfaOwner(h)
    info = _GfaInfo()
    _check(_lib.pgl_gfa_info_get(h, C.byref(info)))
    v = _View()
    _check(_lib.pgl_gfa_view(h, C.byref(v)))
    g = PangenomeGraph._from_view(v, owner)
    g.path_names = [_lib.pgl_gfa_path_name(h, p).decode() for p in range(info.n_paths)]
    g.edges = np.zeros(info.n_edges, EDGE_DTYPE)
    if info.n_edges:
        _check(_lib.pgl_gfa_edges(h, g.edges.ctypes.data))
    g.skipped_records = int(info.skipped_records)
    return g


def parse_gfa_file(path: str, threads: int = 0) -> PangenomeGraph:
    """parse_gfa + build_graph (gfa.cpp:57-153, graph.cpp:7-59), mmap'd and
    multithreaded: same node ids, edges, paths, offsets and exceptions.
    The graph carries .edges (EDGE_DTYPE), .path_names, .skipped_records."""
    h = C.c_void_p()
    _check(_lib.pgl_gfa_parse_file(os.fsencode(path), threads, C.byref(h)))
    return _gfa_graph(h)


def parse_gfa(text, threads: int = 0) -> PangenomeGraph:
    """parse_gfa of an in-memory GFA text (str or bytes)."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    _check(_lib.pgl_gfa_parse_buffer(b, len(b), threads, C.byref(h)))
    return _gfa_graph(h)


def write_layout_tsv(path: str, layout: np.ndarray, threads: int = 0) -> None:
    """write_layout_tsv (layout_io.cpp:31-46), byte-identical, multithreaded."""
    c = np.ascontiguousarray(layout, np.float64).reshape(-1)
    if c.size % 4:
        raise CountMismatch("CountMismatch: layout size is not a multiple of 4")
    _check(_lib.pgl_layout_write_tsv(os.fsencode(path), c.ctypes.data_as(_f64p), c.size // 4, threads))


def read_layout_tsv(path: str, threads: int = 0) -> np.ndarray:
    """read_layout_tsv (layout_io.cpp:48-110) -> flat [4*n] snapshot-order array."""
    n = C.c_uint64()
    p = _f64p()
    _check(_lib.pgl_layout_read_tsv(os.fsencode(path), threads, C.byref(n), C.byref(p)))
    try:
        return np.ctypeslib.as_array(p, (4 * n.value,)).copy() if n.value else np.zeros(0)
    finally:
        _lib.pgl_free(p)


def generate_nested_pangenome(seed: int, backbone_nodes: int, n_paths: int, depth: int = 3,
                              site_rate: float = 0.05) -> PangenomeGraph:
    """Config 5 fixture: nested bubbles, inversions, deletions, duplications
    (pgl_synthetic_generate_nested)."""
    h = C.c_void_p()
    _check(_lib.pgl_synthetic_generate_nested(seed, backbone_nodes, n_paths, depth, site_rate, C.byref(h)))
    owner = _SynthOwner(h)
    v = _View()
    _check(_lib.pgl_synthetic_view(h, C.byref(v)))
    return PangenomeGraph._from_view(v, owner)


def build_graph(node_lengths, walks, names=None) -> PangenomeGraph:
    """build_graph (graph.cpp:7-59): walks = [[(node, reverse), ...], ...]."""
    nl = np.asarray(node_lengths, np.uint64)
    if np.any(nl == 0):
        raise InvalidParameter("InvalidParameter: node has zero sequence length")
    steps = []
    for k, w in enumerate(walks):
        if len(w) == 0:
            raise EmptyPath(f"EmptyPath: path '{names[k] if names else k}' has no steps")
        ids = np.array([s[0] for s in w], np.int64)
        if np.any(ids < 0) or np.any(ids >= len(nl)):
            raise UnknownNode("UnknownNode: path references a node outside the graph")
        lens = nl[ids]
        if np.any(lens > 0xFFFFFFFF):
            raise InvalidParameter("InvalidParameter: node is longer than a step record can hold")
        a = np.zeros(len(w), PATH_STEP_DTYPE)
        a["node_id"] = ids
        a["seq_len"] = lens
        a["orient"] = [1 if s[1] else 0 for s in w]
        a["offset"] = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        steps.append(a)
    return PangenomeGraph(nl, steps, names)


# ---- layout -----------------------------------------------------------------------

def _callback(on_iteration, n_nodes):
    if on_iteration is None:
        return _CB(), 0
    err = []

    def cb(it, coords, eta, secs, user):
        try:
            arr = np.ctypeslib.as_array(coords, (4 * n_nodes,)).copy() if coords else None
            on_iteration(int(it), arr, float(eta), float(secs))
            return 0
        except BaseException as e:  # propagate like the reference: abort the run
            err.append(e)
            return 1

    fn = _CB(cb)
    fn._err = err
    return fn, 1


def _check_diag(ext, total_steps):
    d = ext.diag if ext is not None else None
    if d is not None and d.primary_visits is not None and d.primary_visits.size != total_steps:
        raise InvalidParameter("InvalidParameter: LayoutDiag.primary_visits needs total_steps entries")


def _run(device, g, cfg, ext, reuse, on_iteration, stats, want_coords=True):
    cfg = cfg or LayoutConfig()
    out = np.zeros(4 * g.n_nodes)
    st = _Stats()
    cb, wants = _callback(on_iteration, g.n_nodes)
    _check_diag(ext, g.total_steps())
    e = ext._c() if ext else None
    rc = _lib.pgl_layout_run(device, C.byref(g.view()), C.byref(cfg._c()),
                             C.byref(e) if e else None, int(reuse), cb, wants, None,
                             out.ctypes.data_as(_f64p), C.byref(st))
    if rc and getattr(cb, "_err", None):
        raise cb._err[0]
    _check(rc)
    if stats is not None:
        stats._load(st)
    return out


def run_layout(g: PangenomeGraph, cfg: Optional[LayoutConfig] = None,
               on_iteration: Optional[Callable] = None, stats: Optional[RunStats] = None,
               device: int = 0, ext: Optional[LayoutExt] = None) -> np.ndarray:
    """run_layout (engine.hpp:80-82). Returns the layout as a flat float64
    array in Layout::snapshot order (sx, sy, ex, ey per node). The callback
    receives (iter, coords_snapshot, eta, seconds) at every boundary."""
    return _run(device, g, cfg, ext, 0, on_iteration, stats)


def run_layout_reuse(g: PangenomeGraph, cfg: LayoutConfig, on_iteration=None, stats=None,
                     device: int = 0, ext: Optional[LayoutExt] = None) -> np.ndarray:
    """run_layout_reuse (engine.hpp:86-88): drf in {2, 4}."""
    return _run(device, g, cfg, ext, 1, on_iteration, stats)


def sampled_path_stress(g: PangenomeGraph, layout: np.ndarray, seed: int,
                        samples_per_node: int = 100, method: int = SPS_COUNTER,
                        device: int = 0) -> StressReport:
    """sampled_path_stress (metrics.hpp:49-51) as a GPU reduction."""
    c = np.ascontiguousarray(layout, np.float64).reshape(-1)
    if c.size != 4 * g.n_nodes:
        raise CountMismatch("CountMismatch: layout size does not match the graph")
    r = _Report()
    _check(_lib.pgl_sampled_path_stress(device, C.byref(g.view()), c.ctypes.data_as(_f64p), seed,
                                        samples_per_node, method, C.byref(r)))
    return StressReport._of(r)


def exact_path_stress(g: PangenomeGraph, layout: np.ndarray, device: int = 0) -> StressReport:
    """exact_path_stress (metrics.hpp:39, metrics.cpp:75-106) on the GPU:
    every step pair of every path, deterministic double-double reduction."""
    c = np.ascontiguousarray(layout, np.float64).reshape(-1)
    if c.size != 4 * g.n_nodes:
        raise CountMismatch("CountMismatch: layout size does not match the graph")
    r = _Report()
    _check(_lib.pgl_exact_path_stress(device, C.byref(g.view()), c.ctypes.data_as(_f64p), C.byref(r)))
    return StressReport._of(r)


def make_schedule(g: PangenomeGraph, cfg: LayoutConfig) -> np.ndarray:
    etas = np.zeros(max(cfg.n_iters, 1))
    _check(_lib.pgl_make_schedule(C.byref(g.view()), C.byref(cfg._c()), etas.ctypes.data_as(_f64p)))
    return etas


def init_layout(g: PangenomeGraph, seed: int) -> np.ndarray:
    out = np.zeros(4 * g.n_nodes)
    _check(_lib.pgl_init_layout(C.byref(g.view()), seed, out.ctypes.data_as(_f64p)))
    return out


def device_count() -> int:
    return int(_lib.pgl_device_count())


def transfer_bytes():
    """(host->device, device->host) bytes the library has copied so far."""
    h, d = C.c_uint64(0), C.c_uint64(0)
    _check(_lib.pgl_transfer_bytes(C.byref(h), C.byref(d)))
    return int(h.value), int(d.value)


class DeviceGraph:
    """A graph packed and resident in HBM (pgl_graph_create): repeated layouts
    and stress evaluations without re-uploading the index."""

    def __init__(self, g: Optional[PangenomeGraph], device: int = 0, _handle=None):
        self.g, self.device = g, device
        if _handle is None:
            h = C.c_void_p()
            _check(_lib.pgl_graph_create(device, C.byref(g.view()), C.byref(h)))
        else:
            h = _handle
        self.h = h
        i = self.info()
        self.n_nodes, self.n_paths, self.total_steps = int(i["n_nodes"]), int(i["n_paths"]), int(i["total_steps"])

    @classmethod
    def from_gfa(cls, path: str, device: int = 0, threads: int = 0) -> "DeviceGraph":
        """pgl_graph_create_gfa: parse a GFA on the host into 4-byte step words
        and build the step records on the device (no PathStep arrays)."""
        h = C.c_void_p()
        _check(_lib.pgl_graph_create_gfa(device, os.fsencode(path), threads, C.byref(h)))
        return cls(None, device, _handle=h)

    def close(self):
        if getattr(self, "h", None):
            _lib.pgl_graph_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        i = _Info()
        _check(_lib.pgl_graph_info_get(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_ if not f.startswith("_")}

    def layout(self, cfg: Optional[LayoutConfig] = None, ext: Optional[LayoutExt] = None,
               reuse: bool = False, on_iteration=None, stats: Optional[RunStats] = None,
               copy_out: bool = True) -> Optional[np.ndarray]:
        cfg = cfg or LayoutConfig()
        out = np.zeros(4 * self.n_nodes) if copy_out else None
        st = _Stats()
        cb, wants = _callback(on_iteration, self.n_nodes)
        if ext is not None and ext.diag is not None:
            _check_diag(ext, self.info()["total_steps"])
        e = ext._c() if ext else None
        rc = _lib.pgl_graph_layout(self.h, C.byref(cfg._c()), C.byref(e) if e else None, int(reuse), cb,
                                   wants, None, out.ctypes.data_as(_f64p) if copy_out else None,
                                   C.byref(st))
        if rc and getattr(cb, "_err", None):
            raise cb._err[0]
        _check(rc)
        if stats is not None:
            stats._load(st)
        return out

    def export_index(self):
        """(positions [S,2], nodes [S], cum [P+1]) decoded from the device records."""
        S, P = self.total_steps, self.n_paths
        pos = np.zeros(2 * S, np.uint64)
        nodes = np.zeros(S, np.uint32)
        cum = np.zeros(P + 1, np.uint64)
        _check(_lib.pgl_graph_export_index(self.h, pos.ctypes.data_as(_u64p),
                                           nodes.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           cum.ctypes.data_as(_u64p)))
        return pos.reshape(-1, 2), nodes, cum

    def timing(self) -> Timing:
        t = _Timing()
        _check(_lib.pgl_graph_last_timing(self.h, C.byref(t)))
        return Timing(t.kernel_ms, t.init_ms, t.total_ms, t.device_ms, t.launches, t.grid_blocks, t.block_threads,
                      t.device_threads, t.nonfinite_nodes, t.coord_kind, t.variant)

    def all_finite(self, layout: Optional[np.ndarray] = None):
        """Layout::all_finite on the device: (bad node count, first bad node)
        of the resident layout or of `layout`."""
        c = None if layout is None else np.ascontiguousarray(layout, np.float64).reshape(-1)
        if c is not None and c.size != 4 * self.n_nodes:
            raise CountMismatch("CountMismatch: layout size does not match the graph")
        bad, first = C.c_uint64(0), C.c_uint64(0)
        _check(_lib.pgl_graph_all_finite(self.h, c.ctypes.data_as(_f64p) if c is not None else None,
                                         C.byref(bad), C.byref(first)))
        return int(bad.value), int(first.value)

    def stress(self, seed: int, samples_per_node: int = 100, layout: Optional[np.ndarray] = None,
               method: int = SPS_COUNTER, return_ms: bool = False):
        r = _Report()
        ms = C.c_double()
        c = None if layout is None else np.ascontiguousarray(layout, np.float64).reshape(-1)
        _check(_lib.pgl_graph_stress(self.h, c.ctypes.data_as(_f64p) if c is not None else None, seed,
                                     samples_per_node, method, C.byref(r), C.byref(ms)))
        rep = StressReport._of(r)
        return (rep, ms.value) if return_ms else rep

    def exact_stress(self, layout: Optional[np.ndarray] = None, return_ms: bool = False):
        """exact_path_stress on the resident graph (layout None = resident layout)."""
        r = _Report()
        ms = C.c_double()
        c = None if layout is None else np.ascontiguousarray(layout, np.float64).reshape(-1)
        _check(_lib.pgl_graph_exact_stress(self.h, c.ctypes.data_as(_f64p) if c is not None else None,
                                           C.byref(r), C.byref(ms)))
        rep = StressReport._of(r)
        return (rep, ms.value) if return_ms else rep


def shard_plan(graphs: Sequence[PangenomeGraph], cfgs: Sequence[LayoutConfig], n_devices: int):
    """The plan layout_shards runs (pgl_shard_plan), computed on the host:
    returns (assignment, work, device_load) with work = updates per graph."""
    n = len(graphs)
    views = (C.POINTER(_View) * max(n, 1))(*[C.pointer(g.view()) for g in graphs])
    cs = (_Cfg * max(n, 1))(*[c._c() for c in cfgs])
    assign = (C.c_int * max(n, 1))()
    work = np.zeros(max(n, 1))
    load = np.zeros(max(n_devices, 1))
    _check(_lib.pgl_shard_plan(n_devices, n, views, cs, assign, work.ctypes.data_as(_f64p),
                               load.ctypes.data_as(_f64p)))
    return list(assign)[:n], work[:n], load[:n_devices]


def layout_shards(graphs: Sequence[PangenomeGraph], cfgs: Sequence[LayoutConfig], devices: Sequence[int],
                  ext: Optional[LayoutExt] = None, copy_out: bool = True):
    """Multi-GPU scheduler (pgl_layout_shards): LPT over independent graphs,
    one host thread + stream per device, no collective. Returns
    (layouts, seconds, assignment)."""
    n = len(graphs)
    views = (C.POINTER(_View) * max(n, 1))(*[C.pointer(g.view()) for g in graphs])
    cs = (_Cfg * max(n, 1))(*[c._c() for c in cfgs])
    devs = (C.c_int * len(devices))(*devices)
    outs = [np.zeros(4 * g.n_nodes) for g in graphs] if copy_out else []
    optr = (_f64p * max(n, 1))(*[o.ctypes.data_as(_f64p) for o in outs]) if copy_out else None
    secs = np.zeros(max(n, 1))
    assign = (C.c_int * max(n, 1))()
    st = (_Stats * max(n, 1))()
    if ext is not None and ext.diag is not None:
        raise InvalidParameter("InvalidParameter: LayoutDiag is per graph; not available for layout_shards")
    e = ext._c() if ext else None
    _check(_lib.pgl_layout_shards(len(devices), devs, n, views, cs, C.byref(e) if e else None,
                                  optr, st, secs.ctypes.data_as(_f64p), assign))
    return outs, secs[:n].tolist(), list(assign)[:n]
