import sys, time, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2409_00876_b200 as P
from oracle_ffi import Reference
R = Reference()
g = P.generate_synthetic_pangenome(1, 968000, 90, 0.05)
gr = R.generate(1, 968000, 90, 0.05)
with P.DeviceGraph(g) as dg:
    lay = dg.layout(P.LayoutConfig(global_seed=101))
    out = {}
    for spn in (1, 10, 100):
        r, ms = dg.stress(7, spn, layout=lay, method=P.SPS_STREAM, return_ms=True)
        r2, ms2 = dg.stress(7, spn, layout=lay, method=P.SPS_COUNTER, return_ms=True)
        out[spn] = {"stream_ms": ms, "stream_mean": r.mean, "n": r.n, "counter_ms": ms2, "counter_mean": r2.mean}
    t = time.perf_counter(); w = R.sps(gr, lay, 7, 1); out["ref_spn1_s"] = time.perf_counter() - t
    out["ref_spn1"] = {"mean": w.mean, "n": w.n, "skipped": w.skipped}
    out["stream_spn1_matches"] = (out[1]["n"] == w.n) and abs(out[1]["stream_mean"] / w.mean - 1) < 1e-12
print(json.dumps(out))
