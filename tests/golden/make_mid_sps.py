"""Regenerates tests/golden/mid_sps_reference.json: the REFERENCE's own
layouts (oracle/_ref/libpglref.so, compiled from the reference sources by
oracle/Makefile; threads = 16) of a mid-size synthetic graph, scored with the
reference's sampled_path_stress (seed 7, spn 10), for layout seeds 101-105.

The graph (generate_synthetic_pangenome(1, 387200, 20, 0.05), ~400k nodes)
is large enough that the device runs its production tile kernel there --
the concurrency cap (one warp per 80 nodes) allows the lean async tile
kernel's full residency, so PGL_SAMPLING_AUTO picks the tile sampler -- so tests/test_gpu_parity.py::test_production_kernel_sps_parity_mid
gates exactly the kernels configs 2-5 run (FP64 and anchored stores) against
these medians without re-running the reference (~1 min per layout).

usage: python tests/golden/make_mid_sps.py [THREADS]   (needs oracle/_ref; ran on the B200 box's host)"""
import json
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ffi import Reference, make_cfg  # noqa: E402

MID = (1, 387200, 20, 0.05)
SEEDS = (101, 102, 103, 104, 105)


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    R = Reference()
    g = R.generate(*MID)
    per = []
    for s in SEEDS:
        t = time.time()
        lay, st = R.run_layout(g, make_cfg(global_seed=s, threads=threads))
        secs = time.time() - t
        r = R.sps(g, lay, 7, 10)
        per.append({"seed": s, "sps_mean": r.mean, "n": int(r.n), "layout_s": round(secs, 2),
                    "applied": int(st.updates_applied), "attempted": int(st.updates_attempted)})
        print(json.dumps(per[-1]), flush=True)
    out = {"graph": {"generator": "generate_synthetic_pangenome", "args": list(MID), "n_nodes": g.n_nodes,
                     "total_steps": g.total_steps},
           "layout": {"config": "LayoutConfig{} defaults", "threads": threads, "seeds": list(SEEDS)},
           "metric": {"estimator": "reference sampled_path_stress", "seed": 7, "spn": 10},
           "per_seed": per, "median_sps": statistics.median(p["sps_mean"] for p in per)}
    path = os.environ.get("MID_SPS_OUT", os.path.join(HERE, "mid_sps_reference.json"))
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
