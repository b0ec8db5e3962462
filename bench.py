#!/usr/bin/env python
"""bench.py — PG-SGD layout throughput on B200 (BASELINE.json metric).

Workload (N=1): config 3 of BASELINE.json, the north star's chr1-scale
synthetic graph generate_synthetic_pangenome(1, 9680000, 90, 0.05)
(10,002,606 nodes, 871,194,136 path steps), LayoutConfig{} defaults (30
iterations, theta 0.99, Zipf window 1000, batch 32, drf = srf = 1). One bench
step = one full run_layout of that graph: 30 x 10 x sum|p| = 2.61e11
attempted updates. (--config c1|c2|c5 select the other single-GPU configs.)

  value  : updates/s with the packed graph resident in HBM; device time from
           CUDA events on the library's stream (init upload -> last SGD
           kernel), L2 flushed between steps.
  e2e    : updates/s through the C-ABI drop-in pgl_layout_run with HOST
           buffers: pack + H2D of the graph and initial layout, 30 kernels,
           D2H of the coordinates, every step (host wall, synchronised);
           h2d/d2h bytes are the library's own copy counters
           (pgl_transfer_bytes) around the timed calls.
  roofline: k_sgd_tiles, bound "hbm": achieved = the DRAM bytes one launch
           moves (dram__bytes_read.sum + dram__bytes_write.sum of the
           committed ncu --set full capture of this kernel on this config,
           profiles/ncu_traffic.json) / the live mean launch time, against
           MEASURED_PEAKS.json hbm_gbs. The payload model (two 16-byte step
           records + two endpoint reads + two write-backs = 96 B f64 / 64 B
           f32 per update) is reported beside it as "payload"; SURVEY.md
           §8d's 192 B = six random sectors prices the reference's i.i.d.
           access pattern and does not apply to the tile sampler.
  iid_sampler: one layout with the reference's i.i.d. selection
           (SAMPLING_IID, k_sgd_hogwild) on the same graph, so the share of
           the speed-up that comes from the tile sampler is explicit.
  cpu_baseline: the reference library itself (oracle/_ref, built from the
           reference sources), all host cores, on a bounded sample.

--gpus N (torchrun): every rank lays out its own chromosome-scale graph
(config 3's shape, generator seed 1 + rank; one chromosome per GPU, no
collective: SURVEY.md §8e) -> weak scaling; value = all ranks' updates /
max-over-ranks time. Then (--c4 auto: when N > 1) config 4: the 24
chromosome graphs split over the ranks by LPT, made resident, laid out back
to back; "c4" reports the max-over-ranks makespan.
--impl reference: times the reference CPU implementation (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PG-SGD updates/sec and layout wall-time per chromosome; sampled path stress"
UNIT = "updates/s"
# payload bytes per update: 2 x 16-byte step records + 4 endpoint accesses
BYTES_PER_UPDATE = {"f64": 2 * 16 + 4 * 16, "f32": 2 * 16 + 4 * 8, "anch": 2 * 16 + 4 * 8}
CONFIGS = {
    "c1": (1, 9680, 8, 0.05),
    "c2": (1, 968000, 90, 0.05),
    "c3": (1, 9680000, 90, 0.05),
    "c5": (5, 200000, 500, 3, 0.05),  # generate_nested_pangenome(seed, backbone, paths, depth, site rate)
}
WORKLOAD_NAME = {
    "c1": "config 1: synthetic ~10k-node 8-path graph (generate_synthetic_pangenome(1, 9680, 8, 0.05)), 30 iters",
    "c2": "config 2: synthetic 1M-node 90-path graph (generate_synthetic_pangenome(1, 968000, 90, 0.05)), 30 iters",
    "c3": "config 3: chr1-scale synthetic 10M-node 90-path graph (generate_synthetic_pangenome(1, 9680000, 90, 0.05)), 30 iters",
    "c5": ("config 5: high-complexity synthetic graph, nested bubbles (depth 3), inversions, duplications, "
           "500 paths, zipf_space_max 1e5 (generate_nested_pangenome(5, 200000, 500, 3, 0.05)), 30 iters"),
}
FALLBACK_HBM_GBS = 6650.0
CONFIG_LAYOUT = {"c5": {"zipf_space_max": 100000}}  # LayoutConfig overrides per config


def make_graph(P, config, rank=0):
    """The config's graph; rank r > 0 of a multi-GPU run gets its own
    chromosome of the same shape (generator seed + r)."""
    args = CONFIGS[config]
    args = (args[0] + rank,) + tuple(args[1:])
    if config == "c5":
        return P.generate_nested_pangenome(*args)
    return P.generate_synthetic_pangenome(*args)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--no-iid", action="store_true", help="skip the i.i.d.-sampler comparison layout")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--coord", choices=["auto", "f32", "f64", "anch"], default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--c4", choices=["auto", "on", "off"], default="auto",
                    help="config 4 makespan over this rank's LPT share (auto: on when N > 1)")
    return ap.parse_args()


# ---- distributed plumbing (torch.distributed is plumbing only) -------------------

class Dist:
    def __init__(self, n_gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch, self.backend = dist, torch, backend

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device=f"cuda:{self.local}" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device=f"cuda:{self.local}" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def aggregate(dist: Dist, per_rank_units: float, per_rank_seconds: float):
    """Whole-job throughput: all ranks' units over the slowest rank's time."""
    t = dist.max(per_rank_seconds)
    units = dist.sum(per_rank_units)
    return units / t if t > 0 else 0.0, t


# ---- clocks sampler -------------------------------------------------------------

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class Clocks:
    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        busy = [r for r in rows if not (r[2] & 0x1)] or rows
        reasons = set()
        for r in busy:
            for bit, name in REASON_BITS.items():
                if r[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in busy) if busy else None,
                "sm_max_mhz": max(r[1] for r in busy) if busy else None,
                "reasons": sorted(reasons), "samples": len(busy)}


# ---- peaks, profiles ------------------------------------------------------------

def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def kernel_name(variant: int) -> str:
    """The SGD kernel a layout ran (pgl_timing.kernel_variant: 0 = the
    i.i.d. kernel, 7-12 the lean tile kernel, else the general tile kernel)."""
    return "k_sgd_hogwild" if variant == 0 else ("k_sgd_lean" if 7 <= variant <= 14 else "k_sgd_tiles")


def ncu_key(config: str, coord: str, variant: int) -> str:
    """profiles/ncu_traffic.json key of a capture of this kernel on this config."""
    return f"{config}_{coord}" + ("_iid" if variant == 0 else "")


def ncu_traffic(config: str, coord: str, variant: int = 10):
    """(dram bytes per SGD launch, ncu ms of that launch, cache/sector
    summary) from the committed ncu --set full capture
    (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f)[ncu_key(config, coord, variant)]
    except (OSError, KeyError, ValueError):
        return None, None, None
    keys = ("l2_hit_pct", "l1_hit_pct", "ld_bytes_per_sector", "st_bytes_per_sector", "lsu_sectors_per_update",
            "dram_bytes_per_update", "source")
    return (e.get("dram_bytes_per_launch"), e.get("mixed_iteration", {}).get("ms"),
            {k: e[k] for k in keys if k in e})


def sps_roofline(args, samples: int, kernel_ms: float, peak: float):
    """Roofline entry of the sampled-path-stress kernel (k_sps_chunks, one
    launch per estimate): measured DRAM bytes per sample from the committed
    ncu --set full capture (profiles/ncu_traffic.json "<config>_<store>_sps",
    per sample so it scales to this run's spn) x samples / the live kernel
    time. Payload model beside it: two 16-byte step records + two endpoint
    reads (16 B FP64, 8 B + the 8-byte block anchor anchored) per sample."""
    payload = 32 + 2 * 16
    out = {"kernel": "k_sps_chunks", "bound": "hbm", "unit": "GB/s", "peak": peak, "samples": samples,
           "launch_ms": kernel_ms,
           "payload": {"bytes_per_sample": payload,
                       "achieved": samples * payload / (kernel_ms / 1e3) / 1e9 if kernel_ms else None}}
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f)[f"{args.config}_{args.coord}_sps"]
        bps = e["dram_bytes_per_sample"]
        out.update({"traffic_bytes_per_sample": bps, "achieved": samples * bps / (kernel_ms / 1e3) / 1e9,
                    "source": e.get("source")})
        out["frac"] = out["achieved"] / peak
    except (OSError, KeyError, ValueError, TypeError, ZeroDivisionError):
        out.update({"achieved": None, "frac": None, "traffic_bytes_per_sample": None})
    return out


# ---- CPU baseline: the reference itself --------------------------------------------

def cpu_reference_sample(args, n_steps_total=1, budget_s=20.0):
    """Times pglref::run_layout (oracle/_ref, the reference's own sources) with
    threads = all host cores on a bounded sample of the workload: 2 iterations
    (one mixed, one forced-cooling, as SURVEY.md §8d extrapolates) with srf
    chosen so each sample takes ~budget_s. Returns (updates/s, cores, sample)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ffi import REF_SO, Reference, make_cfg  # checker infrastructure
    kind = "reference"
    if not os.path.exists(REF_SO):
        return None
    R = Reference()
    if args.config == "c5":  # the fixture's walks, built by the reference's own build_graph
        import paper_2409_00876_b200 as P
        gp = make_graph(P, "c5")
        g = R.build_steps(gp.node_len, gp.path_steps)
        del gp
    else:
        g = R.generate(*CONFIGS[args.config], gfa_roundtrip=(args.config == "c1"))
    cores = os.cpu_count() or 1
    # ~1.5 M updates/s per core measured for the reference at this scale
    est_rate = 1.5e6 * cores
    per_iter_full = 10 * g.total_steps
    want = max(est_rate * budget_s / 2.0, 2e6)
    srf = max(1, int(math.ceil(per_iter_full / want)))
    cfg = make_cfg(n_iters=2, threads=cores, srf=srf, global_seed=101, **CONFIG_LAYOUT.get(args.config, {}))
    rates = []
    sample = None
    for _ in range(n_steps_total):
        t0 = time.perf_counter()
        _, st = R.run_layout(g, cfg)
        dt = time.perf_counter() - t0
        rates.append(st.updates_attempted / dt)
        sample = (f"{args.config} graph, run_layout with n_iters=2 (mixed + forced-cooling iteration), "
                  f"srf={srf} -> {st.updates_attempted} updates per sample, threads={cores}")
    return statistics.median(rates), cores, sample, kind, rates


def run_reference_arm(args, dist: Dist):
    if dist.rank != 0:
        return
    steps = args.steps + args.warmup
    budget = max(3.0, min(args.cpu_budget_s, 150.0 / max(steps, 1)))
    res = cpu_reference_sample(args, n_steps_total=steps, budget_s=budget)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpglref.so not built"}))
        return
    _, cores, sample, kind, rates = res
    timed = rates[args.warmup:] or rates
    v = statistics.median(timed)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD_NAME[args.config], "threads": cores},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---- our arm ----------------------------------------------------------------------

# ---- config 4: 24 chromosomes over the ranks -----------------------

# GRCh38 primary assembly lengths (bp), chr1..22, X, Y; config 4's backbone of
# chromosome c is round(9.68e6 * L_c / L_chr1) (tools/c4_chromosomes.py)
GRCH38 = [248956422, 242193529, 198295559, 190214555, 181538259, 170805979, 159345973, 145138636,
          138394717, 133797422, 135086622, 133275309, 114364328, 107043718, 101991189, 90338345,
          83257441, 80373285, 58617616, 64444167, 46709983, 50818468, 156040895, 57227415]


def c4_share(n_ranks: int, rank: int):
    """This rank's chromosomes under LPT (longest first onto the least-loaded
    rank, ties to the lowest rank -- pgl_shard_plan's rule) by backbone size,
    which is proportional to sum|p| and so to the updates of a layout."""
    sizes = [int(round(9_680_000 * L / GRCH38[0])) for L in GRCH38]
    load = [0] * n_ranks
    mine = []
    for c in sorted(range(len(sizes)), key=lambda k: (-sizes[k], k)):
        r = min(range(n_ranks), key=lambda k: (load[k], k))
        load[r] += sizes[c]
        if r == rank:
            mine.append(c)
    return mine, sizes


def run_c4(args, dist: Dist, P, ext):
    """Config 4 on N GPUs, one rank per GPU, no collective: every rank
    generates its LPT share of the 24 chromosome graphs and makes them resident
    in HBM before the timed region (generation runs on the host and is not the
    layout path), then lays them out back to back. Makespan = max over ranks of
    the synchronised wall time of the rank's layouts (and of their summed
    device time)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    mine, sizes = c4_share(dist.world, dist.rank)
    t0 = time.perf_counter()

    def gen(c):  # ctypes releases the GIL: graphs are generated in parallel
        return c, P.generate_synthetic_pangenome(c + 1, sizes[c], 90, 0.05)

    graphs = {}
    with ThreadPoolExecutor(max_workers=2) as ex:
        for c, g in ex.map(gen, mine):
            graphs[c] = (P.DeviceGraph(g, device=dist.local), g.total_steps())
            del g
    prep_s = time.perf_counter() - t0
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_s, upd = 0.0, 0
    for c in mine:
        dg, S = graphs[c]
        cfg = P.LayoutConfig(global_seed=42 + c)
        dg.layout(cfg, ext=ext, copy_out=False)
        dev_s += dg.timing().device_ms / 1e3
        upd += cfg.n_iters * 10 * S
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    for dg, _ in graphs.values():
        dg.close()
    makespan = dist.max(wall)
    dev_makespan = dist.max(dev_s)
    total_upd = dist.sum(float(upd))
    sum_dev = dist.sum(dev_s)
    return {"workload": "config 4: 24 synthetic chromosome graphs generate_synthetic_pangenome(c+1, "
                        "round(9.68e6*L_c/L_chr1), 90, 0.05), LPT by backbone over the ranks, graphs resident",
            "ranks": dist.world, "graphs_this_rank0": [f"chr{c + 1}" if c < 22 else ("chrX", "chrY")[c - 22]
                                                        for c in mine] if dist.rank == 0 else None,
            "updates": total_upd, "makespan_s": makespan, "device_makespan_s": dev_makespan,
            "value": total_upd / makespan if makespan > 0 else 0.0, "unit": UNIT,
            "lpt_ideal_s": sum_dev / dist.world, "prep_s_rank0": prep_s}


def run_ours(args, dist: Dist):
    import paper_2409_00876_b200 as P
    import torch

    dev = dist.local
    torch.cuda.set_device(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2

    t_gen = time.perf_counter()
    g = make_graph(P, args.config, dist.rank)
    gen_s = time.perf_counter() - t_gen
    S = g.total_steps()
    cfg = P.LayoutConfig(global_seed=42 + dist.rank, **CONFIG_LAYOUT.get(args.config, {}))
    # auto = the library default (PGL_COORD_AUTO): FP64 while it fits L2,
    # anchored FP32 beyond when node ids follow path order
    coord_kind = {"auto": P.COORD_AUTO, "f64": P.COORD_F64, "f32": P.COORD_F32,
                  "anch": P.COORD_F32_ANCHORED}[args.coord]
    ext = P.LayoutExt(coord_precision=coord_kind)
    updates = cfg.n_iters * (10 * S // cfg.srf) * cfg.drf

    dg = P.DeviceGraph(g, device=dev)
    for _ in range(args.warmup):
        dg.layout(cfg, ext=ext, copy_out=False)
    torch.cuda.synchronize()
    args.coord = {P.COORD_F64: "f64", P.COORD_F32: "f32", P.COORD_F32_ANCHORED: "anch"}[dg.timing().coord_kind]

    clocks = Clocks(dev)
    clocks.start()
    dev_ms, kern_ms, launches = [], [], 0
    st = P.RunStats()
    dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dg.layout(cfg, ext=ext, copy_out=False, stats=st)
        tm = dg.timing()
        dev_ms.append(tm.device_ms)
        kern_ms.append(tm.kernel_ms)
        # SGD + seed_rng (+ the f64 -> store conversion, + one re-anchor per iteration after the first)
        launches += tm.launches + 1 + (0 if args.coord == "f64" else 1) + (cfg.n_iters - 1 if args.coord == "anch" else 0)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    step_s = sum(dev_ms) / 1e3 / args.steps
    value, t_max = aggregate(dist, updates * args.steps, step_s * args.steps)
    sgd_launch_ms = sum(kern_ms) / (args.steps * cfg.n_iters)
    # the device's own counts for the last timed layout (DevStats)
    stats = {"primary_steps": st.primary_steps, "updates_attempted": st.updates_attempted,
             "updates_applied": st.updates_applied, "updates_skipped": st.updates_skipped,
             "applied_fraction": st.updates_applied / max(st.updates_attempted, 1),
             "device_counts_match": st.updates_attempted == updates
             and st.updates_applied + st.updates_skipped == st.updates_attempted}

    # quality of the bench's own layout (device SPS kernel, spn 100, seed 7)
    sps, sps_ms = dg.stress(7, 100, return_ms=True)
    timing = dg.timing()
    info = dg.info()

    # the reference's i.i.d. selection on the same graph (k_sgd_hogwild): the
    # tile sampler's share of the speed-up
    iid = None
    if not args.no_iid:
        dg.layout(cfg, ext=P.LayoutExt(coord_precision=coord_kind, sampling=P.SAMPLING_IID), copy_out=False)
        ti = dg.timing()
        iid_sps = dg.stress(7, 100)
        iid = {"value": updates / (ti.device_ms / 1e3), "unit": UNIT, "layout_s": ti.device_ms / 1e3,
               "launch_ms": ti.kernel_ms / cfg.n_iters, "kernel": "k_sgd_hogwild",
               "sps_mean": iid_sps.mean, "sampling": "SAMPLING_IID (weighted_step_select i.i.d., graph.hpp:123-138)"}
    dg.close()

    # e2e through the C-ABI drop-in with host buffers
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 3))
    P.run_layout(g, cfg, ext=ext, device=dev)  # warm
    dist.barrier()
    torch.cuda.synchronize()
    h0, d0 = P.transfer_bytes()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        P.run_layout(g, cfg, ext=ext, device=dev)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    h1, d1 = P.transfer_bytes()
    dist.barrier()
    e2e_val, _ = aggregate(dist, updates * e2e_steps, e2e_s * e2e_steps)
    h2d, d2h = (h1 - h0) // e2e_steps, (d1 - d0) // e2e_steps  # counted by the library's copy wrappers
    n_nodes, n_paths = g.n_nodes, g.n_paths
    del g  # the CPU sample builds the reference's own copy of the graph

    c4 = None
    if args.c4 == "on" or (args.c4 == "auto" and dist.world > 1):
        c4 = run_c4(args, dist, P, ext)

    cpu = None
    if dist.rank == 0 and not args.no_cpu_baseline and args.gpus == 1:
        res = cpu_reference_sample(args, 1, args.cpu_budget_s)
        if res:
            v, cores, sample, kind, _ = res
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}

    peak, peak_src = hbm_peak()
    payload = BYTES_PER_UPDATE[args.coord]
    rec8 = timing.variant in (13, 14)  # 8-byte records: the primary's 8 B + the partner's two (k, k+1)
    if rec8:
        payload -= 32 - 24
    per_launch = (10 * S // cfg.srf) * cfg.drf
    payload_gbs = per_launch * payload / (sgd_launch_ms / 1e3) / 1e9
    traffic, ncu_ms, ncu_cache = ncu_traffic(args.config, args.coord, timing.variant)
    if traffic:
        achieved, model = traffic / (sgd_launch_ms / 1e3) / 1e9, "ncu-measured DRAM bytes per launch / live launch time"
    else:
        achieved, model = payload_gbs, "payload bytes (no ncu capture committed for this config)"
    if dist.rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME[args.config], "nodes": n_nodes, "paths": n_paths,
                       "path_steps": S, "iters": cfg.n_iters, "updates_per_step": updates,
                       "coord_storage": args.coord, "parallelism": f"graph-per-GPU x{args.gpus} (no collective)",
                       "l2": "flushed between steps (256 MiB write); graph index 16 B/step > L2",
                       "lanes": timing.device_threads, "grid": [timing.grid_blocks, timing.block_threads],
                       "generate_s": gen_s},
            "layout_wall_s": t_max / args.steps,
            "run_stats": stats,
            "sps": {"mean": sps.mean, "ci": [sps.ci_low, sps.ci_high], "n": sps.n,
                    "method": "counter (GPU), seed 7, 100 samples/step", "kernel_ms": sps_ms,
                    "roofline": sps_roofline(args, sps.n, sps_ms, peak)},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_s, "api": "pgl_layout_run (C-ABI) from host PathStep arrays",
                    "bytes": "pgl_transfer_bytes deltas around the timed calls"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_name(timing.variant),
                         "kernel_variant": timing.variant,
                         "model": model, "launch_ms": sgd_launch_ms, "ncu_launch_ms": ncu_ms,
                         "payload": {"bytes_per_update": payload, "achieved": payload_gbs,
                                     "frac": payload_gbs / peak,
                                     "model": ("8-byte primary record + 2 partner records (k, k+1)" if rec8 else
                                               "2 step records") + " + 2 endpoint reads + 2 endpoint writes"},
                         "peak_source": peak_src, "ncu": ncu_cache},
            "iid_sampler": iid,
            "c4": c4,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk,
            "device_bytes": info["device_bytes"],
        }
        print(json.dumps(out))


def main():
    args = parse()
    dist = Dist(args.gpus)
    try:
        if args.impl == "reference":
            run_reference_arm(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
