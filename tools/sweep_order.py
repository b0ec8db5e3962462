"""Experiment (GPU box): unit visit order of the tile sampler vs layout quality
and speed. For each variant: device time per 30-iteration layout and the
median SPS over layout seeds 101..105 (metric seed 7), next to the
reference's own threads=1 layouts at config 1.

usage: python tools/sweep_order.py OUT.json [c1,c2,c3] [variants]
variant syntax: spread | fronts:G (G warps per front) | ...:w<max_warps>"""
import json
import statistics
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2409_00876_b200 as P  # noqa: E402
from oracle_ffi import Reference, make_cfg  # noqa: E402

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}


def ext_of(v):
    e = P.LayoutExt()
    for part in v.split(":"):
        if part == "spread":
            e.unit_order = P.ORDER_SPREAD
        elif part == "fronts":
            e.unit_order = P.ORDER_FRONTS
        elif part.startswith("w") and part[1:].isdigit():
            e.max_warps = int(part[1:])
        elif part == "nowin":
            e.pair_window = 1
        elif part == "win":
            e.pair_window = 2
        elif part.startswith("hop"):
            e.pair_window = 3
            e.hop_lanes = int(part[3:] or 0)
        elif part == "rn":
            e.record_hint = 1
        elif part.startswith("v") and part[1:].isdigit():
            e.kernel_variant = int(part[1:])
        elif part == "anch":
            e.coord_precision = P.COORD_F32_ANCHORED
        elif part.startswith("f32"):
            e.coord_precision = P.COORD_F32
        elif part.isdigit():
            e.front_warps = int(part)
    return e


def main():
    out = sys.argv[1]
    cfgs = (sys.argv[2] if len(sys.argv) > 2 else "c1,c2").split(",")
    variants = (sys.argv[3] if len(sys.argv) > 3 else "spread,fronts:4,fronts:8,fronts:16,fronts:32").split(",")
    R = Reference()
    res = []
    for c in cfgs:
        g = P.generate_synthetic_pangenome(*GEN[c])
        seeds = [101, 102, 103, 104, 105] if c != "c3" else [101, 102]
        spn = 100 if c == "c1" else 10
        row = {"config": c}
        if c == "c1":
            gr = R.generate(*GEN[c], gfa_roundtrip=True)
        with P.DeviceGraph(g) as dg:
            if c == "c1":  # same estimator (GPU counter, seed 7, spn 100) on the reference's threads=1 layouts
                row["ref_sps"] = [dg.stress(7, 100, layout=R.run_layout(gr, make_cfg(global_seed=s))[0]).mean
                                  for s in seeds]
                row["ref_median"] = statistics.median(row["ref_sps"])
            for v in variants:
                e = ext_of(v)
                sps, ms = [], []
                for s in seeds:
                    lay = dg.layout(P.LayoutConfig(global_seed=s), ext=e)
                    ms.append(dg.timing().kernel_ms)
                    sps.append(dg.stress(7, spn, layout=lay).mean)
                upd = 30 * 10 * g.total_steps()
                r = {"config": c, "variant": v, "kernel_ms": ms, "gupd_s": upd / (min(ms) * 1e6),
                     "sps": sps, "sps_median": statistics.median(sps), "spn": spn}
                if "ref_median" in row:
                    r["ratio_vs_ref"] = r["sps_median"] / row["ref_median"]
                res.append(r)
                print(json.dumps(r), flush=True)
        res.append(row)
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
