"""Background job (build container): reference layouts of config 2 for the
SPS parity gate. Runs pglref::run_layout (oracle/_ref, the reference's own
sources) with threads=T for layout seeds 101..105, then scores each layout
with the C restatement of the GPU's counter estimator (seed 7, spn 10) and
the reference estimator's own stream at spn 1. Appends JSON lines to
.refcache/c2_ref_sps.jsonl and keeps the layouts as .npy."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle_ffi import Oracle, Reference, make_cfg, stress_tuple
T = int(sys.argv[1]) if len(sys.argv) > 1 else 6
R, O = Reference(), Oracle()
out = os.path.join(ROOT, ".refcache")
t = time.time()
gr = R.generate(1, 968000, 90, 0.05)
go = O.generate(1, 968000, 90, 0.05)
print("gen", time.time() - t, flush=True)
for seed in (101, 102, 103, 104, 105):
    path = os.path.join(out, f"c2_ref_{seed}.npy")
    t = time.time()
    lay, st = R.run_layout(gr, make_cfg(global_seed=seed, threads=T))
    secs = time.time() - t
    np.save(path, lay)
    t = time.time()
    ctr = O.sps_counter(go, lay, 7, 10)
    ref1 = O.sps(go, lay, 7, 1)
    rec = {"seed": seed, "threads": T, "layout_s": secs, "applied": st.updates_applied,
           "attempted": st.updates_attempted, "sps_counter_7_10": list(stress_tuple(ctr)),
           "sps_ref_7_1": list(stress_tuple(ref1)), "score_s": time.time() - t}
    with open(os.path.join(out, "c2_ref_sps.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
    print(rec, flush=True)
