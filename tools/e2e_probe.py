import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2409_00876_b200 as P
g = P.generate_synthetic_pangenome(1, 968000, 90, 0.05)
cfg = P.LayoutConfig(global_seed=42)
for rep in range(3):
    t0 = time.perf_counter(); dg = P.DeviceGraph(g); t1 = time.perf_counter()
    out = dg.layout(cfg); t2 = time.perf_counter(); tm = dg.timing(); dg.close(); t3 = time.perf_counter()
    t4 = time.perf_counter(); P.run_layout(g, cfg); t5 = time.perf_counter()
    print(f"create {t1-t0:.3f}  layout+d2h {t2-t1:.3f} (device {tm.device_ms/1e3:.3f} init {tm.init_ms/1e3:.3f} total {tm.total_ms/1e3:.3f})  close {t3-t2:.3f}  run_layout {t5-t4:.3f}", flush=True)
