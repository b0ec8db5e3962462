"""Config 4: 24 synthetic whole-chromosome graphs sharded over the visible
GPUs. Backbone sizes round(9.68e6 * L_c / L_chr1) from the
GRCh38 lengths; generate_synthetic_pangenome(c, backbone_c, 90, 0.05).

Graphs are independent, so there is no exchange: LPT (longest first onto the
least-loaded GPU) by sum|p|, one worker thread per GPU that generates its
next graph on the host while the current one is laid out on the device
(ctypes releases the GIL around the native calls). Prints one JSON line
with per-chromosome wall times, the makespan and the LPT projection for
1/2/4/8 GPUs from the measured per-chromosome device times.

usage: python tools/c4_chromosomes.py [--gpus N] [--limit K] [--coord auto|f64|f32|anch]
"""
import argparse
import json
import os
import queue
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P  # noqa: E402

# GRCh38 primary assembly lengths (bp), chr1..22, X, Y
GRCH38 = [248956422, 242193529, 198295559, 190214555, 181538259, 170805979, 159345973, 145138636,
          138394717, 133797422, 135086622, 133275309, 114364328, 107043718, 101991189, 90338345,
          83257441, 80373285, 58617616, 64444167, 46709983, 50818468, 156040895, 57227415]
NAMES = [f"chr{k}" for k in range(1, 23)] + ["chrX", "chrY"]


def backbone(c):
    return int(round(9_680_000 * GRCH38[c] / GRCH38[0]))


def lpt(sizes, n_dev):
    load = [0.0] * n_dev
    assign = {}
    for c in sorted(range(len(sizes)), key=lambda k: -sizes[k]):
        d = min(range(n_dev), key=lambda k: load[k])
        load[d] += sizes[c]
        assign[c] = d
    return assign, max(load)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=max(1, P.device_count()))
    ap.add_argument("--limit", type=int, default=24)
    ap.add_argument("--coord", choices=["auto", "f32", "f64", "anch"], default="auto")
    ap.add_argument("--sps", action="store_true", help="score every layout on device (spn 10)")
    args = ap.parse_args()
    chroms = list(range(args.limit))
    sizes = [backbone(c) for c in chroms]
    assign, _ = lpt(sizes, args.gpus)
    ext = P.LayoutExt(coord_precision={"auto": P.COORD_AUTO, "f64": P.COORD_F64, "f32": P.COORD_F32,
                                       "anch": P.COORD_F32_ANCHORED}[args.coord])
    results = {}
    lock = threading.Lock()

    def worker(dev):
        mine = [c for c in sorted(chroms, key=lambda k: -sizes[k]) if assign[c] == dev]
        q = queue.Queue(maxsize=1)

        def producer():
            for c in mine:
                t0 = time.time()
                g = P.generate_synthetic_pangenome(c + 1, sizes[c], 90, 0.05)
                q.put((c, g, time.time() - t0))
            q.put(None)

        threading.Thread(target=producer, daemon=True).start()
        while True:
            item = q.get()
            if item is None:
                break
            c, g, gen_s = item
            t0 = time.time()
            dg = P.DeviceGraph(g, device=dev)
            st = P.RunStats()
            dg.layout(P.LayoutConfig(global_seed=42), ext=ext, stats=st, copy_out=False)
            tm = dg.timing()
            rec = {"chrom": NAMES[c], "device": dev, "backbone": sizes[c], "nodes": g.n_nodes,
                   "steps": g.total_steps(), "updates": st.updates_attempted, "gen_s": round(gen_s, 2),
                   "wall_s": None, "device_ms": tm.device_ms, "kernel_ms": tm.kernel_ms,
                   "gupd": st.updates_attempted / tm.kernel_ms / 1e6}
            if args.sps:
                rep = dg.stress(7, 10)
                rec["sps_7_10"] = rep.mean
            dg.close()
            rec["wall_s"] = round(time.time() - t0, 3)
            with lock:
                results[c] = rec
                print(json.dumps(rec), flush=True)
            del g

    t0 = time.time()
    threads = [threading.Thread(target=worker, args=(d,)) for d in range(args.gpus)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    makespan = time.time() - t0
    dev_s = [results[c]["device_ms"] / 1e3 for c in chroms]
    proj = {n: lpt(dev_s, n)[1] for n in (1, 2, 4, 8)}
    total_upd = sum(results[c]["updates"] for c in chroms)
    print(json.dumps({
        "config": "C4: 24 synthetic chromosome graphs, generate_synthetic_pangenome(c, round(9.68e6*L_c/L_chr1), 90, 0.05)",
        "gpus": args.gpus, "coord": args.coord, "graphs": len(chroms), "total_updates": total_upd,
        "total_steps": sum(results[c]["steps"] for c in chroms),
        "makespan_s": round(makespan, 2), "sum_device_s": round(sum(dev_s), 2),
        "device_updates_per_s": total_upd / sum(dev_s),
        "lpt_projection_device_s": {str(k): round(v, 2) for k, v in proj.items()},
        "lpt_projection_efficiency": {str(k): round(proj[1] / (k * v), 4) for k, v in proj.items()},
    }), flush=True)


if __name__ == "__main__":
    main()
