"""A/B throughput probe: layout kernel time and SPS for one config with the
library named by PGL_B200_LIB (or the in-tree one).
usage: python tools/ab_speed.py CONFIG [REPS] [PREC] [VARIANT] [EXT_JSON]   (CONFIG c1 c2 c3 c5)
EXT_JSON: extra LayoutExt fields, e.g. '{"l2_persist": 1}'."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prec = int(sys.argv[3]) if len(sys.argv) > 3 else P.COORD_AUTO
variant = int(sys.argv[4]) if len(sys.argv) > 4 else 0
extra = json.loads(sys.argv[5]) if len(sys.argv) > 5 else {}
g = (P.generate_nested_pangenome(5, 200000, 500, 3, 0.05) if name == "c5"
     else P.generate_synthetic_pangenome(*GEN[name]))
dg = P.DeviceGraph(g)
upd = 30 * 10 * g.total_steps()
ext = P.LayoutExt(**{"coord_precision": prec, "kernel_variant": variant, **extra})
kw = {"zipf_space_max": 100000} if name == "c5" else {}
dg.layout(P.LayoutConfig(n_iters=3, **kw), ext=ext, copy_out=False)
out = []
for k in range(reps):
    dg.layout(P.LayoutConfig(global_seed=101 + k, **kw), ext=ext, copy_out=False)
    out.append(dg.timing().kernel_ms)
tm = dg.timing()
r = dg.stress(7, 20)
print(json.dumps({"lib": os.environ.get("PGL_B200_LIB", "tree"), "config": name, "variant": variant,
                  "ran_variant": tm.variant, "coord": tm.coord_kind, "ext": extra, "kernel_ms": out,
                  "gupd_best": upd / min(out) / 1e6, "sps20": r.mean}), flush=True)
