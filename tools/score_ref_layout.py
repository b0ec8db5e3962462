"""Score a stored reference layout (tools/ref_layouts.py output) with the two
estimators tools/parity.py uses, in the build container: the C restatement
of the device counter estimator (orc_sps_counter, bit-identical to
pgl_sampled_path_stress(PGL_SPS_COUNTER)) and the reference's own
sampled_path_stress. Appends one JSON line to OUT for tools/parity.py
--ref-json.

usage: python tools/score_ref_layout.py CONFIG LAYOUT.npy SEED OUT.jsonl [counter_spn] [ref_spn]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle_ffi import Oracle, Reference, stress_tuple

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}
cfg, path, seed, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
cspn = int(sys.argv[5]) if len(sys.argv) > 5 else 10
rspn = int(sys.argv[6]) if len(sys.argv) > 6 else 1
lay = np.load(path)
rec = {"config": cfg, "seed": seed, "source": path}
O = Oracle()
go = O.generate(*GEN[cfg])
t = time.time()
c = stress_tuple(O.sps_counter(go, lay, 7, cspn))
rec[f"sps_gpu_spn{cspn}"] = {"mean": c[0], "n": int(c[1]), "ci": [c[3], c[4]], "skipped": int(c[5])}
rec["counter_s"] = round(time.time() - t, 1)
del go
R = Reference()
gr = R.generate(*GEN[cfg])
t = time.time()
w = stress_tuple(R.sps(gr, lay, 7, rspn))
rec[f"sps_ref_spn{rspn}"] = {"mean": w[0], "n": int(w[1]), "ci": [w[3], w[4]], "skipped": int(w[5])}
rec["ref_s"] = round(time.time() - t, 1)
with open(out, "a") as f:
    f.write(json.dumps(rec) + "\n")
print(json.dumps(rec))
