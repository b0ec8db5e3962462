"""Sampler quality study (checker side, never the product): device layouts
under several LayoutExt settings against the reference's own layouts of the
identical graph, both scored with the same estimator and metric seed
(SURVEY.md §8(d) parity procedure; gate: median SPS ratio in [0.98, 1.02]).

Configs:
  c1      generate_synthetic_pangenome(1, 9680, 8, 0.05); reference threads=1
          (the -m gpu gate's shape); reference estimator spn 100
  c5small generate_nested_pangenome(5, 3000, 50, 3, 0.05), zipf_space_max
          1e5; reference threads=1; reference estimator spn 20
  c5full  generate_nested_pangenome(5, 200000, 500, 3, 0.05) (config 5),
          zipf_space_max 1e5; reference threads = nproc; reference estimator
          spn 1 and the device counter estimator spn 100
  c2      config 2; reference threads = nproc; as c5full

Variants are name=JSON pairs of LayoutExt fields, e.g.
  --variants 'default={};hop2={"hop_lanes":2};iid={"sampling":1}'
Each prints and appends one JSON line (per-seed values, medians, ratio to the
reference median) to --out; the reference line comes first.

usage: python tools/sampler_quality.py CONFIG --out F.jsonl [--variants ...]
       [--seeds 101,...] [--cache DIR] [--ref-only] [--ref-json F]
--ref-json: reference per-seed scores from a committed file (the "reference"
object of profiles/r02_parity_c5.json, or a reference line of this tool's
output) instead of laying the reference out again."""
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

CONFIGS = {
    # name: (generator, args, LayoutConfig overrides, reference threads (0 = nproc), ref spn, gpu spn)
    "c1": ("synthetic", (1, 9680, 8, 0.05), {}, 1, 100, 0),
    "c5small": ("nested", (5, 3000, 50, 3, 0.05), {"zipf_space_max": 100000}, 1, 20, 0),
    "c5full": ("nested", (5, 200000, 500, 3, 0.05), {"zipf_space_max": 100000}, 0, 1, 100),
    "c2": ("synthetic", (1, 968000, 90, 0.05), {}, 0, 1, 100),
}
DEFAULT_VARIANTS = ('default={};hop4={"hop_lanes":4};hop2={"hop_lanes":2};hop1={"hop_lanes":1};'
                    'window_only={"pair_window":2};independent={"pair_window":1};iid={"sampling":1}')


def parse_variants(s):
    out = {}
    for part in s.split(";"):
        if part.strip():
            name, js = part.split("=", 1)
            out[name.strip()] = json.loads(js)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", required=True)
    ap.add_argument("--variants", default=DEFAULT_VARIANTS)
    ap.add_argument("--seeds", default="101,102,103,104,105")
    ap.add_argument("--cache", default=None, help="directory for reference layouts (.npy)")
    ap.add_argument("--ref-only", action="store_true")
    ap.add_argument("--ref-json", default=None)
    args = ap.parse_args()
    gen, gargs, over, threads, ref_spn, gpu_spn = CONFIGS[args.config]
    threads = threads or os.cpu_count()
    seeds = [int(s) for s in args.seeds.split(",")]
    R = Reference()
    g = P.generate_nested_pangenome(*gargs) if gen == "nested" else P.generate_synthetic_pangenome(*gargs)
    gr = R.build_steps(g.node_len, g.path_steps)
    dg = P.DeviceGraph(g)

    def score(lay):
        rec = {"ref_est": R.sps(gr, lay, 7, ref_spn).mean}
        if gpu_spn:
            rec["gpu_est"] = dg.stress(7, gpu_spn, layout=lay).mean
        return rec

    def emit(line):
        print(json.dumps(line), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(line) + "\n")

    ref = []
    if args.ref_json:
        with open(args.ref_json) as f:
            txt = f.read().strip()
        try:
            doc = json.loads(txt)
            doc = doc.get("reference", doc)
        except ValueError:  # JSON lines: the first reference line
            doc = next(json.loads(x) for x in txt.splitlines() if '"reference"' in x)
        ref = [r for r in doc["per_seed"] if r["seed"] in seeds]
    for s in ([] if args.ref_json else seeds):
        path = os.path.join(args.cache, f"{args.config}_ref_{s}.npy") if args.cache else None
        secs = None
        if path and os.path.exists(path):
            lay = np.load(path)
        else:
            t = time.time()
            lay, _ = R.run_layout(gr, make_cfg(global_seed=s, threads=threads, **over))
            secs = time.time() - t
            if path:
                os.makedirs(args.cache, exist_ok=True)
                np.save(path, lay)
        r = score(lay)
        r.update(seed=s, layout_s=secs, threads=threads)
        ref.append(r)
    line = {"config": args.config, "variant": "reference", "per_seed": ref, "source": args.ref_json or "computed",
            "median_ref_est": statistics.median(r["ref_est"] for r in ref)}
    if gpu_spn:
        line["median_gpu_est"] = statistics.median(r["gpu_est"] for r in ref)
    emit(line)
    if args.ref_only:
        return
    for name, kw in parse_variants(args.variants).items():
        per = []
        for s in seeds:
            st = P.RunStats()
            t = time.time()
            lay = dg.layout(P.LayoutConfig(global_seed=s, **over), ext=P.LayoutExt(**kw), stats=st)
            r = score(lay)
            r.update(seed=s, layout_s=round(time.time() - t, 3), coord=dg.timing().coord_kind,
                     applied_frac=st.updates_applied / max(st.updates_attempted, 1))
            per.append(r)
        out = {"config": args.config, "variant": name, "ext": kw, "per_seed": per}
        for est in ("ref_est", "gpu_est"):
            if est in per[0]:
                m = statistics.median(r[est] for r in per)
                out[f"median_{est}"] = m
                out[f"ratio_{est}"] = m / line[f"median_{est}"]
        emit(out)
    dg.close()


if __name__ == "__main__":
    main()
