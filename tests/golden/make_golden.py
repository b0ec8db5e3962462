"""Regenerates tests/golden/reference_vectors.json from the REFERENCE ITSELF
(oracle/_ref/libpglref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the build container: python tests/golden/make_golden.py

The fixtures pin the C oracle (and through it the CUDA path) on boxes where
/root/reference does not exist.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ffi import Reference, make_cfg, stress_tuple  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_digest(R, g):
    f = R.export(g)
    return {"n_nodes": g.n_nodes, "n_paths": g.n_paths, "total_steps": g.total_steps,
            "total_nt": g.total_nt, "n_edges": g.n_edges,
            "node_len": sha(f.node_len), "cum": f.cum.tolist() if len(f.cum) < 200 else sha(f.cum),
            "step_node": sha(f.step_node), "step_rev": sha(f.step_rev), "step_off": sha(f.step_off),
            "step_len": sha(f.step_len), "path_total": f.path_total.tolist(),
            "positions": sha(R.positions(g))}


def main():
    R = Reference()
    out = {"source": "oracle/_ref/libpglref.so built from /root/reference/proj/src (-O3 -DNDEBUG)"}
    out["rng"] = {f"{s}_{w}": [str(x) for x in R.rng_draws(s, w, 16)]
                  for s, w in [(42, 0), (7, 2**61 + 3), (0, 0), (2**64 - 1, 5)]}
    out["zipf"] = {f"{n}_{t}": R.zipf(n, t, 99, 0, 64).tolist()
                   for n, t in [(1, 0.5), (4, 1.0), (1000, 0.99), (1000, 2.0), (10**6, 0.99), (7, 0.3)]}
    graphs = {"c1": (1, 9680, 8, 0.05, True), "t31": (31, 120, 2, 0.1, False),
              "t3": (3, 50, 4, 0.3, False), "desk": (7, 5000, 12, 0.05, False),
              "lin": (1, 100, 3, 0.0, False)}
    out["graphs"] = {}
    for name, (s, b, p, r, rt) in graphs.items():
        g = R.generate(s, b, p, r, gfa_roundtrip=rt)
        d = graph_digest(R, g)
        d["args"] = [s, b, p, r]
        d["init_42"] = sha(R.init_layout(g, 42))
        d["etas_30"] = R.schedule(g, make_cfg()).tolist()
        cases = {"default_101": make_cfg(global_seed=101)} if name in ("c1", "t31") else {}
        if name == "t3":
            cases = {"default_42": make_cfg(), "reuse_2_2": make_cfg(n_iters=5, drf=2, srf=2),
                     "reuse_4_4_b7": make_cfg(n_iters=5, drf=4, srf=4, batch_size=7),
                     "b1": make_cfg(n_iters=4, batch_size=1, global_seed=9)}
        d["layouts"] = {}
        for cname, cfg in cases.items():
            lay, st = R.run_layout(g, cfg, reuse=cfg.drf > 1)
            d["layouts"][cname] = {
                "cfg": {k: getattr(cfg, k) for k, _ in cfg._fields_ if not k.startswith("_")},
                "sha256": sha(lay), "first8": lay[:8].tolist(),
                "stats": [int(getattr(st, k)) for k, _ in st._fields_],
                "sps_7_100": list(stress_tuple(R.sps(g, lay, 7, 100))),
            }
        d["sps_init_42_7_10"] = list(stress_tuple(R.sps(g, R.init_layout(g, 42), 7, 10)))
        if g.total_steps <= 2000:
            d["exact_init_42"] = list(stress_tuple(R.exact(g, R.init_layout(g, 42))))
        out["graphs"][name] = d
    path = os.path.join(HERE, "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
