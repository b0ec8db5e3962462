"""A/B probe of the counter SPS kernel with the library named by PGL_B200_LIB:
kernel ms at spn 100 on a laid-out config graph (and the estimate, which must
be bit-identical across builds: same terms, same fold order).
usage: python tools/sps_ab.py CONFIG [REPS]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = P.generate_synthetic_pangenome(*GEN[name])
with P.DeviceGraph(g) as dg:
    dg.layout(P.LayoutConfig(global_seed=101), copy_out=False)
    ms, means = [], set()
    for _ in range(reps):
        r, t = dg.stress(7, 100, return_ms=True)
        ms.append(t)
        means.add((r.mean, r.n, r.skipped))
    print(json.dumps({"lib": os.path.basename(os.environ.get("PGL_B200_LIB", "tree")), "config": name,
                      "coord": dg.timing().coord_kind, "sps_ms": ms, "samples": r.n,
                      "gsamples_s": r.n / min(ms) / 1e6, "mean": r.mean, "distinct": len(means)}), flush=True)
