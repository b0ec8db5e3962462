"""Short target for ncu: one layout of a config with few iterations.
usage: python tools/prof_target.py CONFIG ITERS PREC [ORDER [FRONT_WARPS]]   (CONFIG c1 c2 c3 c5)
ORDER: pgl_unit_order (0 auto = 1 spread). --iid: the i.i.d. kernel; --kv=N: its kernel_variant."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P
cfgs = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 1
args = [a for a in sys.argv if not a.startswith("--")]
order = int(args[4]) if len(args) > 4 else 0
fw = int(args[5]) if len(args) > 5 else 0
g = (P.generate_nested_pangenome(5, 200000, 500, 3, 0.05) if name == "c5"
     else P.generate_synthetic_pangenome(*cfgs[name]))
kw = {"zipf_space_max": 100000} if name == "c5" else {}
dg = P.DeviceGraph(g)
samp = P.SAMPLING_IID if "--iid" in sys.argv else P.SAMPLING_AUTO
kv = [int(a[5:]) for a in sys.argv if a.startswith("--kv=")]
dg.layout(P.LayoutConfig(n_iters=iters, **kw),
          ext=P.LayoutExt(coord_precision=prec, unit_order=order, front_warps=fw, sampling=samp,
                          kernel_variant=kv[0] if kv else 0), copy_out=False)
r = dg.stress(7, 10)
print("done", dg.timing(), r.mean)
