"""ncu target: the bit-exact replay (threads = 1) on config 1, 2 iterations."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P
g = P.generate_synthetic_pangenome(1, 9680, 8, 0.05)
dg = P.DeviceGraph(g)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dg.layout(P.LayoutConfig(n_iters=n, global_seed=101), ext=P.LayoutExt(mode=P.MODE_REPLAY), copy_out=False)
t = dg.timing()
print("replay: %d iters, kernel %.1f ms, %.2f us/update" % (n, t.kernel_ms, t.kernel_ms * 1e3 / (n * 10 * g.total_steps())))
