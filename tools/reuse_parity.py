"""Update-reuse quality against the reference (checker side): config 1,
layout seeds 101-105, the reference's estimator (seed 7, spn 100).
For each (drf, srf): medians of the reference's drf=1 run_layout (the
acceptance #7 base, acceptance.cpp:327-350), the reference's own
run_layout_reuse, the device's reference-semantics reuse and the device's
warp-shuffle reuse (pgl_layout_ext.reuse_shuffle), with device wall times.
usage: python tools/reuse_parity.py OUT.jsonl"""
import json, os, statistics, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2409_00876_b200 as P
from oracle_ffi import Reference, make_cfg

C1 = (1, 9680, 8, 0.05)
R = Reference()
g = P.generate_synthetic_pangenome(*C1)
gr = R.generate(*C1, gfa_roundtrip=True)
seeds = range(101, 106)
sps = lambda lay: R.sps(gr, lay, 7, 100).mean
base = [sps(R.run_layout(gr, make_cfg(global_seed=s))[0]) for s in seeds]
mb = statistics.median(base)
out = open(sys.argv[1], "a")
out.write(json.dumps({"ref_drf1": base, "median": mb}) + "\n")
for drf, srf in [(2, 2), (4, 4), (2, 1), (4, 2), (2, 4), (4, 8)]:
    rec = {"drf": drf, "srf": srf}
    ref = [sps(R.run_layout(gr, make_cfg(global_seed=s, drf=drf, srf=srf), reuse=True)[0]) for s in seeds]
    rec["ref_reuse_median"] = statistics.median(ref)
    for name, shuffle in (("gpu_refsem", 0), ("gpu_shuffle", 1)):
        v, secs = [], []
        for s in seeds:
            t = time.perf_counter()
            lay = P.run_layout_reuse(g, P.LayoutConfig(global_seed=s, drf=drf, srf=srf),
                                     ext=P.LayoutExt(reuse_shuffle=shuffle))
            secs.append(time.perf_counter() - t)
            v.append(sps(lay))
        rec[name + "_median"] = statistics.median(v)
        rec[name + "_vs_ref_drf1"] = statistics.median(v) / mb
        rec[name + "_vs_ref_reuse"] = statistics.median(v) / rec["ref_reuse_median"]
        rec[name + "_wall_s"] = statistics.median(secs)
    rec["ref_reuse_vs_ref_drf1"] = rec["ref_reuse_median"] / mb
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
