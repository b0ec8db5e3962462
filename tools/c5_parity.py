"""Config-5 SPS parity study (checker side): device sampler variants against
the reference's own layouts of the identical graph, scored with the same
estimators and metric seed on both sides (SURVEY.md §8(d) parity procedure).

  --size small : generate_nested_pangenome(5, 3000, 50, 3, 0.05), reference
                 threads = 1 (the -m gpu test's shape), reference estimator
                 spn 20
  --size full  : generate_nested_pangenome(5, 200000, 500, 3, 0.05) (config 5),
                 reference threads = nproc, reference estimator spn 1 and the
                 device counter estimator spn 100 on every layout

Layout seeds 101..105, zipf_space_max 1e5, metric seed 7. Prints and appends
one JSON line per variant (per-seed values, medians, ratio to the reference
median) to --out.

usage: python tools/c5_parity.py --size small|full --out F.jsonl [--variants a,b] [--cache DIR]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2409_00876_b200 as P  # noqa: E402
from oracle_ffi import Reference, make_cfg  # noqa: E402

SIZES = {"small": (5, 3000, 50, 3, 0.05), "full": (5, 200000, 500, 3, 0.05)}
VARIANTS = {
    "default": dict(),
    "hop4": dict(hop_lanes=4),
    "hop2": dict(hop_lanes=2),
    "hop1": dict(hop_lanes=1),
    "window_only": dict(pair_window=2),
    "independent": dict(pair_window=1),
    "iid": dict(sampling=1),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", choices=sorted(SIZES), default="small")
    ap.add_argument("--out", required=True)
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--cache", default=None, help="directory for reference layouts (.npy)")
    ap.add_argument("--seeds", default="101,102,103,104,105")
    ap.add_argument("--ref-only", action="store_true")
    args = ap.parse_args()
    seeds = [int(s) for s in args.seeds.split(",")]
    full = args.size == "full"
    threads = os.cpu_count() if full else 1
    ref_spn = 1 if full else 20
    R = Reference()
    g = P.generate_nested_pangenome(*SIZES[args.size])
    gr = R.build_steps(g.node_len, g.path_steps)

    def score(lay):
        rec = {"ref_est": R.sps(gr, lay, 7, ref_spn).mean}
        if full:
            rec["gpu_est"] = P.sampled_path_stress(g, lay, 7, 100).mean
        return rec

    ref = []
    for s in seeds:
        path = os.path.join(args.cache, f"c5{args.size}_ref_{s}.npy") if args.cache else None
        if path and os.path.exists(path):
            lay = np.load(path)
            secs = None
        else:
            t = time.time()
            lay, _ = R.run_layout(gr, make_cfg(global_seed=s, zipf_space_max=100000, threads=threads))
            secs = time.time() - t
            if path:
                os.makedirs(args.cache, exist_ok=True)
                np.save(path, lay)
        r = score(lay)
        r.update(seed=s, layout_s=secs, threads=threads)
        ref.append(r)
        print(json.dumps({"ref_seed": r}), flush=True)
    line = {"size": args.size, "variant": "reference", "per_seed": ref,
            "median_ref_est": statistics.median(r["ref_est"] for r in ref)}
    if full:
        line["median_gpu_est"] = statistics.median(r["gpu_est"] for r in ref)
    with open(args.out, "a") as f:
        f.write(json.dumps(line) + "\n")
    if args.ref_only:
        return
    for name in args.variants.split(","):
        per = []
        for s in seeds:
            t = time.time()
            lay = P.run_layout(g, P.LayoutConfig(global_seed=s, zipf_space_max=100000),
                               ext=P.LayoutExt(**VARIANTS[name]))
            r = score(lay)
            r.update(seed=s, layout_s=time.time() - t)
            per.append(r)
        out = {"size": args.size, "variant": name, "ext": VARIANTS[name], "per_seed": per}
        for est in ("ref_est", "gpu_est"):
            if est in per[0]:
                m = statistics.median(r[est] for r in per)
                out[f"median_{est}"] = m
                out[f"ratio_{est}"] = m / line[f"median_{est}"]
        print(json.dumps(out), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
