"""Short target for compute-sanitizer (memcheck / initcheck / racecheck):
every device path once on config 1 and small shapes -- the auto tile kernel,
the lean kernel (both stores, forced), the i.i.d. kernel, replay, reuse with
warp shuffles, both SPS estimators, exact stress, the GFA-free device index.
usage: compute-sanitizer --tool memcheck python tools/sanitize_target.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2409_00876_b200 as P

g = P.generate_synthetic_pangenome(1, 9680, 8, 0.05)
cfg = P.LayoutConfig(n_iters=4, global_seed=5)
outs = []
with P.DeviceGraph(g) as dg:
    for ext in [P.LayoutExt(), P.LayoutExt(kernel_variant=7, coord_precision=P.COORD_F64),
                P.LayoutExt(kernel_variant=8, coord_precision=P.COORD_F32_ANCHORED),
                P.LayoutExt(kernel_variant=7, unit_order=P.ORDER_RANDOM),
                P.LayoutExt(kernel_variant=6, coord_precision=P.COORD_F32_ANCHORED),
                P.LayoutExt(kernel_variant=10, coord_precision=P.COORD_F32_ANCHORED),
                P.LayoutExt(sampling=P.SAMPLING_IID),
                P.LayoutExt(sampling=P.SAMPLING_IID, kernel_variant=4, coord_precision=P.COORD_F32_ANCHORED),
                P.LayoutExt(sampling=P.SAMPLING_IID, kernel_variant=7),
                P.LayoutExt(sampling=P.SAMPLING_IID, kernel_variant=5)]:
        outs.append(dg.layout(cfg, ext=ext))
    outs.append(dg.layout(P.LayoutConfig(n_iters=1, global_seed=5), ext=P.LayoutExt(mode=P.MODE_REPLAY)))
    dg.stress(7, 5)
    dg.stress(7, 2, method=P.SPS_STREAM)
small = P.generate_synthetic_pangenome(3, 300, 3, 0.05)
outs.append(P.run_layout(small, P.LayoutConfig(n_iters=3, batch_size=7, threads=4),
                         ext=P.LayoutExt(sampling=P.SAMPLING_IID, kernel_variant=4)))
outs.append(P.run_layout_reuse(small, P.LayoutConfig(n_iters=3, drf=2, srf=2), ext=P.LayoutExt(reuse_shuffle=1)))
P.exact_path_stress(small, outs[-1])
assert all(np.isfinite(o).all() for o in outs)
print("sanitize target done", len(outs))
