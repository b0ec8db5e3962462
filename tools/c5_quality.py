"""Config-5 (small) quality study: median SPS over seeds 101-105 of several
device sampling variants against the reference's threads=1 layouts (same
estimator: the reference's sampled_path_stress, seed 7, spn 20)."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2409_00876_b200 as P
from oracle_ffi import Reference, make_cfg
args = tuple(json.loads(sys.argv[1])) if len(sys.argv) > 1 else (5, 3000, 50, 3, 0.05)
R = Reference()
g = P.generate_nested_pangenome(*args)
gr = R.build_steps(g.node_len, g.path_steps)
seeds = range(101, 106)
cfgs = {s: dict(global_seed=s, zipf_space_max=100000) for s in seeds}
ref = [R.sps(gr, R.run_layout(gr, make_cfg(**cfgs[s]))[0], 7, 20).mean for s in seeds]
mr = statistics.median(ref)
print(json.dumps({"ref": ref, "median": mr}), flush=True)
variants = {"default": P.LayoutExt(), "window_only": P.LayoutExt(pair_window=2),
            "iid": P.LayoutExt(sampling=P.SAMPLING_IID), "hop4": P.LayoutExt(hop_lanes=4),
            "hop2": P.LayoutExt(hop_lanes=2), "hop8_ownsign": P.LayoutExt(pair_window=4),
            "hop4_ownsign": P.LayoutExt(pair_window=4, hop_lanes=4)}
for name, e in variants.items():
    v = [R.sps(gr, P.run_layout(g, P.LayoutConfig(**cfgs[s]), ext=e), 7, 20).mean for s in seeds]
    print(json.dumps({"variant": name, "median": statistics.median(v), "ratio": statistics.median(v) / mr}), flush=True)
