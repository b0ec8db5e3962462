"""End-to-end breakdown probe: where the host-side time of a layout through
the C-ABI goes (graph packing + upload, init_layout, kernels, copy-out).
usage: python tools/e2e_probe.py [CONFIG] [REPS]   (CONFIG c2 | c3; default c2)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00876_b200 as P  # noqa: E402

GEN = {"c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = P.generate_synthetic_pangenome(*GEN[name])
cfg = P.LayoutConfig(global_seed=42)
for rep in range(reps):
    t0 = time.perf_counter()
    dg = P.DeviceGraph(g)
    t1 = time.perf_counter()
    dg.layout(cfg)
    t2 = time.perf_counter()
    tm = dg.timing()
    dg.close()
    t3 = time.perf_counter()
    P.run_layout(g, cfg)
    t4 = time.perf_counter()
    print(json.dumps({"config": name, "create_s": t1 - t0, "layout_d2h_s": t2 - t1, "device_s": tm.device_ms / 1e3,
                      "init_s": tm.init_ms / 1e3, "total_s": tm.total_ms / 1e3, "close_s": t3 - t2,
                      "run_layout_s": t4 - t3, "host_threads": os.cpu_count()}), flush=True)
