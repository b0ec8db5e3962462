"""ctypes bindings for the CHECKERS: oracle/_build/liboracle.so (the plain-C
restatement) and oracle/_ref/libpglref.so (the reference library built from
its own sources). Test infrastructure only — the product never imports this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpglref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)


class LayoutConfigC(C.Structure):
    """pgl_layout_config == LayoutConfig (engine.hpp:13-23)."""
    _fields_ = [("global_seed", C.c_uint64), ("n_iters", C.c_uint32),
                ("threads", C.c_uint32), ("batch_size", C.c_uint32),
                ("_pad0", C.c_uint32), ("zipf_theta", C.c_double),
                ("zipf_space_max", C.c_uint64), ("eta_min_eps", C.c_double),
                ("drf", C.c_uint32), ("srf", C.c_uint32)]


class StressReportC(C.Structure):
    _fields_ = [("mean", C.c_double), ("n", C.c_uint64), ("std_dev", C.c_double),
                ("ci_low", C.c_double), ("ci_high", C.c_double), ("skipped", C.c_uint64)]


class RunStatsC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "primary_steps", "updates_attempted", "updates_applied", "updates_skipped",
        "batches_first_half", "batches_first_half_cooling", "batches_second_half",
        "batches_second_half_cooling")]


def make_cfg(**kw) -> LayoutConfigC:
    c = LayoutConfigC(global_seed=42, n_iters=30, threads=1, batch_size=32,
                      zipf_theta=0.99, zipf_space_max=1000, eta_min_eps=0.01, drf=1, srf=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class FlatGraph:
    """The graph index flattened: what both checkers export."""
    node_len: np.ndarray      # u64 [V]
    cum: np.ndarray           # u64 [P+1]
    path_total: np.ndarray    # u64 [P]
    step_node: np.ndarray     # u32 [S]
    step_rev: np.ndarray      # u8  [S]
    step_off: np.ndarray      # u64 [S]
    step_len: np.ndarray      # u32 [S]

    @property
    def n_nodes(self):
        return len(self.node_len)

    @property
    def n_paths(self):
        return len(self.cum) - 1

    @property
    def total_steps(self):
        return int(self.cum[-1])

    def path_n_steps(self):
        return np.diff(self.cum).astype(np.uint64)

    def positions(self) -> np.ndarray:
        """path_position (graph.hpp:98-109) for (start, end) of every step."""
        far_end = np.where(self.step_rev == 0, 1, 0)
        off = self.step_off
        ln = self.step_len.astype(np.uint64)
        start = off + np.where(far_end == 0, ln, 0).astype(np.uint64)
        end = off + np.where(far_end == 1, ln, 0).astype(np.uint64)
        return np.stack([start, end], axis=1)


def _export(lib, prefix, h, counts) -> FlatGraph:
    V, P, S = int(counts[0]), int(counts[1]), int(counts[2])
    fg = FlatGraph(np.zeros(V, np.uint64), np.zeros(P + 1, np.uint64), np.zeros(P, np.uint64),
                   np.zeros(S, np.uint32), np.zeros(S, np.uint8), np.zeros(S, np.uint64),
                   np.zeros(S, np.uint32))
    getattr(lib, prefix + "export")(h, ptr(fg.node_len, u64p), ptr(fg.cum, u64p),
                                    ptr(fg.path_total, u64p), ptr(fg.step_node, u32p),
                                    ptr(fg.step_rev, u8p), ptr(fg.step_off, u64p),
                                    ptr(fg.step_len, u32p))
    return fg


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _Graph:
    def __init__(self, lib, handle, free):
        self._lib, self.h, self._free = lib, handle, free

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None


class Oracle:
    """liboracle.so: the C restatement."""

    def __init__(self, path=ORACLE_SO):
        self.lib = L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_rng_next.restype = C.c_uint64
        for name, args in {
            "orc_generate": [C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.POINTER(C.c_void_p)],
            "orc_build": [C.c_uint64, u64p, C.c_uint32, u64p, u32p, u8p, C.POINTER(C.c_void_p)],
            "orc_run_layout": [C.c_void_p, C.POINTER(LayoutConfigC), C.c_int, f64p,
                               C.POINTER(RunStatsC), C.c_void_p, C.c_void_p],
            "orc_sampled_path_stress": [C.c_void_p, f64p, C.c_uint64, C.c_uint32, C.POINTER(StressReportC)],
            "orc_sps_counter": [C.c_void_p, f64p, C.c_uint64, C.c_uint32, C.POINTER(StressReportC)],
            "orc_exact_path_stress": [C.c_void_p, f64p, C.POINTER(StressReportC)],
            "orc_init_layout": [C.c_void_p, C.c_uint64, f64p],
            "orc_make_schedule": [C.c_void_p, C.POINTER(LayoutConfigC), f64p],
            "orc_zipf_samples": [C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, u64p],
            "orc_zipf_constants": [C.c_uint64, C.c_double, f64p],
            "orc_weighted_select": [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p],
            "orc_rng_draws": [C.c_uint64, C.c_uint64, C.c_uint64, u64p],
            "orc_rng_seed": [C.c_uint64, C.c_uint64, u64p],
            "orc_apply_update": [f64p, C.c_uint32, C.c_int, C.c_uint32, C.c_int, C.c_double,
                                 C.c_double, u64p],
            "orc_free": [C.c_void_p], "orc_counts": [C.c_void_p, u64p],
            "orc_export": [C.c_void_p, u64p, u64p, u64p, u32p, u8p, u64p, u32p],
            "orc_positions": [C.c_void_p, u64p],
        }.items():
            getattr(L, name).argtypes = args

    def _check(self, rc):
        if rc:
            raise CheckerError(rc, self.lib.orc_last_error().decode())

    def _wrap(self, h):
        g = _Graph(self.lib, h, self.lib.orc_free)
        c = np.zeros(4, np.uint64)
        self.lib.orc_counts(h, ptr(c, u64p))
        g.n_nodes, g.n_paths, g.total_steps, g.total_nt = (int(x) for x in c)
        return g

    def generate(self, seed, backbone, paths, rate):
        h = C.c_void_p()
        self._check(self.lib.orc_generate(seed, backbone, paths, rate, C.byref(h)))
        return self._wrap(h)

    def build(self, node_len, walks):
        """walks: list of [(node, rev)]"""
        nl = np.asarray(node_len, np.uint64)
        pn = np.asarray([len(w) for w in walks], np.uint64)
        sn = np.asarray([s[0] for w in walks for s in w] or [0], np.uint32)
        sr = np.asarray([s[1] for w in walks for s in w] or [0], np.uint8)
        h = C.c_void_p()
        self._check(self.lib.orc_build(len(nl), ptr(nl, u64p), len(walks), ptr(pn, u64p),
                                       ptr(sn, u32p), ptr(sr, u8p), C.byref(h)))
        return self._wrap(h)

    def export(self, g) -> FlatGraph:
        c = np.array([g.n_nodes, g.n_paths, g.total_steps], np.uint64)
        return _export(self.lib, "orc_", g.h, c)

    def init_layout(self, g, seed):
        out = np.zeros(4 * g.n_nodes)
        self.lib.orc_init_layout(g.h, seed, ptr(out, f64p))
        return out

    def schedule(self, g, cfg):
        etas = np.zeros(cfg.n_iters)
        self._check(self.lib.orc_make_schedule(g.h, C.byref(cfg), ptr(etas, f64p)))
        return etas

    def run_layout(self, g, cfg, reuse=False, callback=None):
        out = np.zeros(4 * g.n_nodes)
        st = RunStatsC()
        cb = None
        if callback is not None:
            CB = C.CFUNCTYPE(None, C.c_uint32, f64p, C.c_double, C.c_void_p)
            cb = CB(lambda it, co, eta, u: callback(
                it, np.ctypeslib.as_array(co, (4 * g.n_nodes,)).copy(), eta))
        self._check(self.lib.orc_run_layout(g.h, C.byref(cfg), int(reuse), ptr(out, f64p),
                                            C.byref(st), C.cast(cb, C.c_void_p) if cb else None,
                                            None))
        return out, st

    def sps(self, g, coords, seed, spn=100):
        r = StressReportC()
        c = np.ascontiguousarray(coords, np.float64)
        self._check(self.lib.orc_sampled_path_stress(g.h, ptr(c, f64p), seed, spn, C.byref(r)))
        return r

    def sps_counter(self, g, coords, seed, spn=100):
        r = StressReportC()
        c = np.ascontiguousarray(coords, np.float64)
        self._check(self.lib.orc_sps_counter(g.h, ptr(c, f64p), seed, spn, C.byref(r)))
        return r

    def exact(self, g, coords):
        r = StressReportC()
        c = np.ascontiguousarray(coords, np.float64)
        self.lib.orc_exact_path_stress(g.h, ptr(c, f64p), C.byref(r))
        return r

    def rng_draws(self, seed, worker, count):
        out = np.zeros(count, np.uint64)
        self.lib.orc_rng_draws(seed, worker, count, ptr(out, u64p))
        return out

    def zipf(self, n, theta, seed, worker, count):
        out = np.zeros(count, np.uint64)
        self._check(self.lib.orc_zipf_samples(n, theta, seed, worker, count, ptr(out, u64p)))
        return out

    def zipf_constants(self, n, theta):
        out = np.zeros(3)
        self.lib.orc_zipf_constants(n, theta, ptr(out, f64p))
        return out

    def weighted_select(self, g, seed, worker, count):
        p = np.zeros(count, np.uint32)
        s = np.zeros(count, np.uint64)
        self._check(self.lib.orc_weighted_select(g.h, seed, worker, count, ptr(p, u32p), ptr(s, u64p)))
        return p, s

    def apply_update(self, coords, ni, ei_end, nj, ej_end, d_ref, eta, s4):
        c = np.ascontiguousarray(coords, np.float64)
        st = np.ascontiguousarray(s4, np.uint64)
        applied = self.lib.orc_apply_update(ptr(c, f64p), ni, ei_end, nj, ej_end, d_ref, eta, ptr(st, u64p))
        return c, st, bool(applied)


class Reference:
    """oracle/_ref/libpglref.so: the reference library itself."""

    def __init__(self, path=REF_SO):
        self.lib = L = C.CDLL(path)
        L.pglref_last_error.restype = C.c_char_p
        for name, args in {
            "pglref_generate": [C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.c_int,
                                C.POINTER(C.c_void_p)],
            "pglref_parse_gfa": [C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p), u64p],
            "pglref_parse_gfa_file": [C.c_char_p, C.POINTER(C.c_void_p), u64p, f64p],
            "pglref_write_gfa": [C.c_void_p, C.c_char_p],
            "pglref_write_layout_tsv": [C.c_char_p, f64p, C.c_uint64],
            "pglref_read_layout_tsv": [C.c_char_p, u64p, f64p, C.c_uint64],
            "pglref_edges": [C.c_void_p, u32p, u8p, u32p, u8p],
            "pglref_path_name": [C.c_void_p, C.c_uint32],
            "pglref_build": [C.c_uint64, u64p, C.c_uint32, u64p, u32p, u8p, C.POINTER(C.c_void_p)],
            "pglref_free": [C.c_void_p], "pglref_counts": [C.c_void_p, u64p],
            "pglref_export": [C.c_void_p, u64p, u64p, u64p, u32p, u8p, u64p, u32p],
            "pglref_positions": [C.c_void_p, u64p],
            "pglref_run_layout": [C.c_void_p, C.POINTER(LayoutConfigC), C.c_int, f64p, u64p,
                                  C.c_void_p, C.c_void_p, f64p],
            "pglref_init_layout": [C.c_void_p, C.c_uint64, f64p],
            "pglref_make_schedule": [C.c_void_p, C.POINTER(LayoutConfigC), f64p, f64p],
            "pglref_make_eta_schedule": [C.c_double, C.c_double, C.c_uint32, f64p],
            "pglref_sampled_path_stress": [C.c_void_p, f64p, C.c_uint64, C.c_uint32,
                                           C.POINTER(StressReportC)],
            "pglref_exact_path_stress": [C.c_void_p, f64p, C.POINTER(StressReportC)],
            "pglref_rng_draws": [C.c_uint64, C.c_uint64, C.c_uint64, u64p],
            "pglref_rng_state": [C.c_uint64, C.c_uint64, u64p],
            "pglref_zipf_samples": [C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, u64p],
            "pglref_weighted_select": [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p],
            "pglref_apply_update": [f64p, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32, C.c_int,
                                    C.c_double, C.c_double, u64p, C.POINTER(C.c_int)],
            "pglref_layout_steps": [C.c_void_p, f64p, C.c_uint64, C.c_uint64, C.c_double, C.c_int,
                                    C.POINTER(LayoutConfigC), C.c_uint64, u8p],
        }.items():
            getattr(L, name).argtypes = args

    def _check(self, rc):
        if rc:
            raise CheckerError(rc, self.lib.pglref_last_error().decode())

    def _wrap(self, h):
        g = _Graph(self.lib, h, self.lib.pglref_free)
        c = np.zeros(5, np.uint64)
        self.lib.pglref_counts(h, ptr(c, u64p))
        g.n_nodes, g.n_paths, g.total_steps, g.total_nt, g.n_edges = (int(x) for x in c)
        return g

    def generate(self, seed, backbone, paths, rate, gfa_roundtrip=False):
        h = C.c_void_p()
        self._check(self.lib.pglref_generate(seed, backbone, paths, rate, int(gfa_roundtrip), C.byref(h)))
        return self._wrap(h)

    def parse_gfa(self, text):
        """parse_gfa of an in-memory text -> (graph, skipped_records)."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        sk = np.zeros(1, np.uint64)
        self._check(self.lib.pglref_parse_gfa(b, len(b), C.byref(h), ptr(sk, u64p)))
        return self._wrap(h), int(sk[0])

    def parse_gfa_file(self, path):
        """parse_gfa through std::ifstream -> (graph, skipped_records, seconds)."""
        h = C.c_void_p()
        sk = np.zeros(1, np.uint64)
        secs = np.zeros(1)
        self._check(self.lib.pglref_parse_gfa_file(os.fsencode(path), C.byref(h), ptr(sk, u64p), ptr(secs, f64p)))
        return self._wrap(h), int(sk[0]), float(secs[0])

    def write_layout_tsv(self, path, coords):
        c = np.ascontiguousarray(coords, np.float64)
        self._check(self.lib.pglref_write_layout_tsv(os.fsencode(path), ptr(c, f64p), c.size // 4))

    def read_layout_tsv(self, path, cap=1 << 24):
        n = np.zeros(1, np.uint64)
        out = np.zeros(cap)
        self._check(self.lib.pglref_read_layout_tsv(os.fsencode(path), ptr(n, u64p), ptr(out, f64p), cap))
        return out[:4 * int(n[0])].copy()

    def write_gfa(self, g, path):
        self._check(self.lib.pglref_write_gfa(g.h, os.fsencode(path)))

    def edges(self, g):
        n = g.n_edges
        f, t = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
        fe, te = np.zeros(max(n, 1), np.uint8), np.zeros(max(n, 1), np.uint8)
        self.lib.pglref_edges(g.h, ptr(f, u32p), ptr(fe, u8p), ptr(t, u32p), ptr(te, u8p))
        return f[:n], fe[:n], t[:n], te[:n]

    def path_names(self, g):
        self.lib.pglref_path_name.restype = C.c_char_p
        return [self.lib.pglref_path_name(g.h, p).decode() for p in range(g.n_paths)]

    def build(self, node_len, walks):
        nl = np.asarray(node_len, np.uint64)
        pn = np.asarray([len(w) for w in walks], np.uint64)
        sn = np.asarray([s[0] for w in walks for s in w] or [0], np.uint32)
        sr = np.asarray([s[1] for w in walks for s in w] or [0], np.uint8)
        h = C.c_void_p()
        self._check(self.lib.pglref_build(len(nl), ptr(nl, u64p), len(walks), ptr(pn, u64p),
                                          ptr(sn, u32p), ptr(sr, u8p), C.byref(h)))
        return self._wrap(h)

    def build_steps(self, node_len, path_steps):
        """build_graph from PathStep-dtype arrays (node_id, orient per path), numpy only."""
        nl = np.asarray(node_len, np.uint64)
        pn = np.asarray([len(p) for p in path_steps], np.uint64)
        sn = np.ascontiguousarray(np.concatenate([p["node_id"] for p in path_steps]), np.uint32)
        sr = np.ascontiguousarray(np.concatenate([p["orient"] for p in path_steps]), np.uint8)
        h = C.c_void_p()
        self._check(self.lib.pglref_build(len(nl), ptr(nl, u64p), len(path_steps), ptr(pn, u64p),
                                          ptr(sn, u32p), ptr(sr, u8p), C.byref(h)))
        return self._wrap(h)

    def export(self, g) -> FlatGraph:
        c = np.array([g.n_nodes, g.n_paths, g.total_steps], np.uint64)
        return _export(self.lib, "pglref_", g.h, c)

    def positions(self, g):
        out = np.zeros(2 * g.total_steps, np.uint64)
        self.lib.pglref_positions(g.h, ptr(out, u64p))
        return out.reshape(-1, 2)

    def init_layout(self, g, seed):
        out = np.zeros(4 * g.n_nodes)
        self._check(self.lib.pglref_init_layout(g.h, seed, ptr(out, f64p)))
        return out

    def schedule(self, g, cfg):
        etas = np.zeros(cfg.n_iters)
        extra = np.zeros(3)
        self._check(self.lib.pglref_make_schedule(g.h, C.byref(cfg), ptr(etas, f64p), ptr(extra, f64p)))
        return etas

    def run_layout(self, g, cfg, reuse=False, callback=None, iter_secs=False):
        out = np.zeros(4 * g.n_nodes)
        st = np.zeros(8, np.uint64)
        secs = np.zeros(cfg.n_iters) if iter_secs else None
        cb = None
        if callback is not None:
            CB = C.CFUNCTYPE(None, C.c_uint32, f64p, C.c_double, C.c_double, C.c_void_p)
            cb = CB(lambda it, co, eta, s, u: callback(
                it, np.ctypeslib.as_array(co, (4 * g.n_nodes,)).copy(), eta))
        self._check(self.lib.pglref_run_layout(
            g.h, C.byref(cfg), int(reuse), ptr(out, f64p), ptr(st, u64p),
            C.cast(cb, C.c_void_p) if cb else None, None,
            ptr(secs, f64p) if secs is not None else None))
        stats = RunStatsC(*[int(x) for x in st])
        return (out, stats, secs) if iter_secs else (out, stats)

    def sps(self, g, coords, seed, spn=100):
        r = StressReportC()
        c = np.ascontiguousarray(coords, np.float64)
        self._check(self.lib.pglref_sampled_path_stress(g.h, ptr(c, f64p), seed, spn, C.byref(r)))
        return r

    def exact(self, g, coords):
        r = StressReportC()
        c = np.ascontiguousarray(coords, np.float64)
        self._check(self.lib.pglref_exact_path_stress(g.h, ptr(c, f64p), C.byref(r)))
        return r

    def rng_draws(self, seed, worker, count):
        out = np.zeros(count, np.uint64)
        self.lib.pglref_rng_draws(seed, worker, count, ptr(out, u64p))
        return out

    def rng_state(self, seed, worker):
        out = np.zeros(4, np.uint64)
        self.lib.pglref_rng_state(seed, worker, ptr(out, u64p))
        return out

    def zipf(self, n, theta, seed, worker, count):
        out = np.zeros(count, np.uint64)
        self._check(self.lib.pglref_zipf_samples(n, theta, seed, worker, count, ptr(out, u64p)))
        return out

    def weighted_select(self, g, seed, worker, count):
        p = np.zeros(count, np.uint32)
        s = np.zeros(count, np.uint64)
        self._check(self.lib.pglref_weighted_select(g.h, seed, worker, count, ptr(p, u32p), ptr(s, u64p)))
        return p, s

    def apply_update(self, coords, ni, ei_end, nj, ej_end, d_ref, eta, s4):
        c = np.ascontiguousarray(coords, np.float64).copy()
        st = np.ascontiguousarray(s4, np.uint64).copy()
        applied = C.c_int()
        self._check(self.lib.pglref_apply_update(ptr(c, f64p), len(c) // 4, ni, ei_end, nj, ej_end,
                                                 d_ref, eta, ptr(st, u64p), C.byref(applied)))
        return c, st, bool(applied.value)


def stress_tuple(r) -> tuple:
    return (r.mean, r.n, r.std_dev, r.ci_low, r.ci_high, r.skipped)
