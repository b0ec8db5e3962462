"""Reference layouts for the SPS parity gate (checker side, never the product).

Runs pglref::run_layout (oracle/_ref = the reference's own sources, compiled
by oracle/Makefile) on a synthetic config graph for the given layout seeds
with threads=T, and stores each layout as .npy plus one JSON line per seed
with its wall time and RunStats. Scoring happens elsewhere (tools/parity.py on
the GPU box scores reference and device layouts with the same estimator).

usage: python tools/ref_layouts.py CONFIG OUTDIR THREADS SEED [SEED ...]
CONFIG is c1 | c2 | c3 (SURVEY.md §8(d) generator calls)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from oracle_ffi import Reference, make_cfg  # noqa: E402

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}


def main():
    cfg_name, out, threads = sys.argv[1], sys.argv[2], int(sys.argv[3])
    seeds = [int(s) for s in sys.argv[4:]]
    os.makedirs(out, exist_ok=True)
    R = Reference()
    t = time.time()
    g = R.generate(*GEN[cfg_name])
    print("gen", cfg_name, round(time.time() - t, 1), "s", flush=True)
    for seed in seeds:
        path = os.path.join(out, f"{cfg_name}_ref_{seed}.npy")
        if os.path.exists(path):
            continue
        t = time.time()
        lay, st = R.run_layout(g, make_cfg(global_seed=seed, threads=threads))
        secs = time.time() - t
        np.save(path + ".tmp.npy", lay)
        os.replace(path + ".tmp.npy", path)
        rec = {"config": cfg_name, "seed": seed, "threads": threads, "layout_s": round(secs, 2),
               "attempted": st.updates_attempted, "applied": st.updates_applied,
               "upd_per_s": st.updates_attempted / secs}
        with open(os.path.join(out, f"{cfg_name}_ref_layouts.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")
        print(rec, flush=True)


if __name__ == "__main__":
    main()
