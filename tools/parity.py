"""Layout parity at scale (SURVEY.md §8(d) "Parity procedure"), run on the GPU box.

For layout seeds 101..105 on a config graph: the reference's own run_layout
(oracle/_ref, threads = all host cores) and the device layout
(pgl_layout_run, default Hogwild/tile mode) of the same graph; both scored
with the SAME estimators and the same metric seed (7):
  - the GPU counter estimator at spn 100 (pgl_sampled_path_stress), and
  - the reference's own sampled_path_stress at spn 1 (host; the reference
    stores every term, so spn 100 does not fit host RAM at config 2+).
Gate: median(SPS_gpu) / median(SPS_ref) in [0.98, 1.02] for each estimator.
Reference layouts can also be loaded from --ref-dir (tools/ref_layouts.py
output) instead of being recomputed.

usage: python tools/parity.py CONFIG OUT.json [--ref-dir DIR] [--seeds 101,...]
       [--gpu-only] [--mode tiles|iid]"""
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
from oracle_ffi import Reference, make_cfg, stress_tuple  # noqa: E402

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}


def rep(r):
    t = stress_tuple(r) if not isinstance(r, P.StressReport) else (
        r.mean, r.n, r.std_dev, r.ci_low, r.ci_high, r.skipped)
    return {"mean": t[0], "n": int(t[1]), "ci": [t[3], t[4]], "skipped": int(t[5])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("out")
    ap.add_argument("--ref-dir", default=None)
    ap.add_argument("--seeds", default="101,102,103,104,105")
    ap.add_argument("--ref-seeds", default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--ref-spn", type=int, default=1)
    ap.add_argument("--sampling", choices=["tiles", "iid"], default="tiles")
    ap.add_argument("--gpu-spn", type=int, default=100, help="spn of the device counter estimator")
    ap.add_argument("--ref-json", default=None,
                    help="reference scores computed elsewhere (tools/score_ref_layout.py lines or a previous "
                         "parity.py output): the reference layouts are not recomputed")
    args = ap.parse_args()
    seeds = [int(s) for s in args.seeds.split(",") if s]  # empty: score reference layouts only
    ref_seeds = [int(s) for s in (args.ref_seeds or args.seeds).split(",") if s]
    R = Reference()
    t = time.time()
    gr = R.generate(*GEN[args.config])
    g = P.generate_synthetic_pangenome(*GEN[args.config])
    assert (g.n_nodes, g.total_steps()) == (gr.n_nodes, gr.total_steps)
    res = {"config": args.config, "graph": {"nodes": g.n_nodes, "steps": g.total_steps()},
           "host_threads": args.threads, "metric_seed": 7, "gen_s": round(time.time() - t, 1),
           "gpu": [], "ref": []}
    samp = P.SAMPLING_TILES if args.sampling == "tiles" else P.SAMPLING_IID
    res["sampling"] = args.sampling

    def flush():
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)

    with P.DeviceGraph(g) as dg:
        init = P.init_layout(g, 101)
        gk = "sps_gpu_spn%d" % args.gpu_spn
        res["init_" + gk] = rep(dg.stress(7, args.gpu_spn, layout=init))
        for seed in seeds:
            t = time.time()
            lay = dg.layout(P.LayoutConfig(global_seed=seed), ext=P.LayoutExt(sampling=samp))
            secs = time.time() - t
            res["gpu"].append({"seed": seed, "layout_s": round(secs, 3),
                               gk: rep(dg.stress(7, args.gpu_spn, layout=lay)),
                               "sps_ref_spn%d" % args.ref_spn: rep(R.sps(gr, lay, 7, args.ref_spn))})
            print("gpu", res["gpu"][-1], flush=True)
            flush()
        if args.ref_json:  # reference scores computed elsewhere
            with open(args.ref_json) as f:
                txt = f.read().strip()
            try:  # a previous parity.py output
                recs = json.loads(txt)["ref"]
            except (ValueError, KeyError, TypeError):  # JSON lines of tools/score_ref_layout.py
                recs = [json.loads(line) for line in txt.splitlines() if line.strip()]
            res["ref"] = [r for r in recs if r["seed"] in ref_seeds]
            res["ref_source"] = args.ref_json
            ref_seeds = []
        for seed in ref_seeds:
            path = args.ref_dir and os.path.join(args.ref_dir, f"{args.config}_ref_{seed}.npy")
            t = time.time()
            if path and os.path.exists(path):
                lay, secs, src = np.load(path), None, path
            else:
                lay, _ = R.run_layout(gr, make_cfg(global_seed=seed, threads=args.threads))
                secs, src = round(time.time() - t, 1), "computed"
            res["ref"].append({"seed": seed, "layout_s": secs, "source": src,
                               gk: rep(dg.stress(7, args.gpu_spn, layout=lay)),
                               "sps_ref_spn%d" % args.ref_spn: rep(R.sps(gr, lay, 7, args.ref_spn))})
            print("ref", res["ref"][-1], flush=True)
            flush()
    for key in ("sps_gpu_spn%d" % args.gpu_spn, "sps_ref_spn%d" % args.ref_spn):
        if not res["gpu"] or not res["ref"]:
            continue
        mg = statistics.median(r[key]["mean"] for r in res["gpu"])
        mr = statistics.median(r[key]["mean"] for r in res["ref"])
        res["ratio_" + key] = mg / mr
        res["gate_" + key] = bool(0.98 <= mg / mr <= 1.02)
    flush()
    print(json.dumps({k: v for k, v in res.items() if k.startswith(("ratio", "gate"))}))


if __name__ == "__main__":
    main()
