"""Exact path stress: the reference's exact_path_stress
(serial, oracle/_ref) against pgl_exact_path_stress on the same layout, with
the agreement of the two reports. usage: python tools/bench_exact.py [c1|small]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2409_00876_b200 as P
from oracle_ffi import Reference
GEN = {"c1": (1, 9680, 8, 0.05), "small": (4, 2000, 4, 0.05)}
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
g = P.generate_synthetic_pangenome(*GEN[name])
R = Reference()
gr = R.generate(*GEN[name])
lay = P.run_layout(g, P.LayoutConfig(global_seed=101))
pairs = sum(int(n) * (int(n) - 1) // 2 for n in g.path_n_steps)
with P.DeviceGraph(g) as dg:
    dg.exact_stress(lay)  # warm
    got, ms = dg.exact_stress(lay, return_ms=True)
t = time.perf_counter()
want = R.exact(gr, lay)
ref_s = time.perf_counter() - t
print(json.dumps({"what": "exact path stress", "config": name, "step_pairs": pairs, "gpu_ms": ms, "reference_s": ref_s,
                  "speedup": ref_s / (ms / 1e3), "gpu_mean": got.mean, "ref_mean": want.mean,
                  "mean_rel_diff": abs(got.mean / want.mean - 1), "n_equal": got.n == want.n,
                  "sd_rel_diff": abs(got.std_dev / want.std_dev - 1)}))
