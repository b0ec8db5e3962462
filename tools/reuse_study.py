"""Data-reuse study (paper §7.4): layout time and
quality of drf/srf schemes with the reference's endpoint-recombination reuse
(engine.cpp:147-170) and with warp-shuffle reuse, against drf = srf = 1, on
a config graph. Quality = SPS ratio to the drf=1 layout (GPU counter
estimator, seed 7, spn 10; acceptance #7 calls <= 2 "good")."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_00876_b200 as P
GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
g = P.generate_synthetic_pangenome(*GEN[name])
rows = []
with P.DeviceGraph(g) as dg:
    lay = dg.layout(P.LayoutConfig(global_seed=101))
    base_ms = dg.timing().kernel_ms
    base = dg.stress(7, 10, layout=lay).mean
    rows.append({"config": name, "scheme": "drf1 srf1", "kernel_ms": base_ms, "sps": base, "sps_ratio": 1.0, "speedup": 1.0})
    for drf, srf in [(2, 2), (2, 4), (4, 4), (4, 8)]:
        for shuffle in (0, 1):
            cfg = P.LayoutConfig(global_seed=101, drf=drf, srf=srf)
            if drf in (2, 4) or shuffle:
                lay = dg.layout(cfg, reuse=drf in (2, 4), ext=P.LayoutExt(reuse_shuffle=shuffle))
            else:
                continue
            ms = dg.timing().kernel_ms
            s = dg.stress(7, 10, layout=lay).mean
            rows.append({"config": name, "scheme": f"drf{drf} srf{srf}", "reuse": "warp-shuffle" if shuffle else "endpoint combos",
                         "kernel_ms": ms, "sps": s, "sps_ratio": s / base, "speedup": base_ms / ms})
            print(json.dumps(rows[-1]), flush=True)
