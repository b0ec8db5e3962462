"""Host IO around the path, reference vs ours
on a config graph, with equality checks:
  * GFA ingest: the reference's parse_gfa (std::ifstream, serial; oracle/_ref)
    against pgl_gfa_parse_file (mmap, all host threads) on write_gfa output;
  * layout TSV: write_layout_tsv / read_layout_tsv against
    pgl_layout_write_tsv / pgl_layout_read_tsv (byte-identical files).
Run on the GPU box host (its core count is the one the other CPU baselines
use); prints (and appends to OUT) one JSON line per measurement.

usage: python tools/bench_io.py CONFIG [OUT.jsonl]   (CONFIG: c1 | c2 | c3)"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2409_00876_b200 as P  # noqa: E402
from oracle_ffi import Reference  # noqa: E402

GEN = {"c1": (1, 9680, 8, 0.05), "c2": (1, 968000, 90, 0.05), "c3": (1, 9680000, 90, 0.05)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    out = sys.argv[2] if len(sys.argv) > 2 else None
    R = Reference()
    g = R.generate(*GEN[name])
    d = tempfile.mkdtemp(prefix="pgl_gfa_")
    path = os.path.join(d, f"{name}.gfa")
    R.write_gfa(g, path)
    size = os.path.getsize(path)
    del g
    with open(path, "rb") as f:  # page cache warm for both parsers
        while f.read(1 << 26):
            pass
    theirs, skipped, ref_s = R.parse_gfa_file(path)
    ours_s = []
    for _ in range(3):
        t = time.perf_counter()
        ours = P.parse_gfa_file(path)
        ours_s.append(time.perf_counter() - t)
    fo = R.export(theirs)
    same = (np.array_equal(ours.node_len, fo.node_len)
            and np.array_equal(np.concatenate([s["offset"] for s in ours.path_steps]), fo.step_off)
            and np.array_equal(np.concatenate([s["node_id"] for s in ours.path_steps]), fo.step_node)
            and np.array_equal(np.concatenate([s["orient"] for s in ours.path_steps]), fo.step_rev)
            and len(ours.edges) == theirs.n_edges and ours.skipped_records == skipped)
    best = min(ours_s)
    dev_s = None
    try:  # GFA straight into a resident device graph (needs a GPU)
        if P.device_count() > 0:
            with P.DeviceGraph.from_gfa(path):  # warm: CUDA context, memory pool
                pass
            t = time.perf_counter()
            with P.DeviceGraph.from_gfa(path):
                dev_s = time.perf_counter() - t
    except P.Error:
        dev_s = None
    rec = {"what": "GFA ingest: parse_gfa + build_graph", "config": name, "gfa_bytes": size,
           "nodes": int(ours.n_nodes), "edges": int(len(ours.edges)), "paths": int(ours.n_paths),
           "steps": int(ours.total_steps()), "reference_s": ref_s, "reference_threads": 1,
           "ours_s": best, "ours_all_s": ours_s, "ours_threads": os.cpu_count(),
           "reference_MBps": size / ref_s / 1e6, "ours_MBps": size / best / 1e6,
           "speedup": ref_s / best, "identical": bool(same),
           "gfa_to_device_graph_s": dev_s}
    recs = [rec]
    os.remove(path)

    # layout TSV of an init layout of the same graph
    lay = P.init_layout(ours, 7)
    a, b = os.path.join(d, "ours.tsv"), os.path.join(d, "ref.tsv")
    t = time.perf_counter()
    R.write_layout_tsv(b, lay)
    ref_w = time.perf_counter() - t
    ours_w = []
    for _ in range(3):
        t = time.perf_counter()
        P.write_layout_tsv(a, lay)
        ours_w.append(time.perf_counter() - t)
    with open(a, "rb") as fa, open(b, "rb") as fb:
        same_w = fa.read() == fb.read()
    tsize = os.path.getsize(a)
    t = time.perf_counter()
    back_ref = R.read_layout_tsv(b, cap=lay.size)
    ref_r = time.perf_counter() - t
    ours_r = []
    for _ in range(3):
        t = time.perf_counter()
        back = P.read_layout_tsv(a)
        ours_r.append(time.perf_counter() - t)
    recs.append({"what": "layout TSV write + read", "config": name, "tsv_bytes": tsize, "nodes": int(ours.n_nodes),
                 "reference_write_s": ref_w, "ours_write_s": min(ours_w), "write_speedup": ref_w / min(ours_w),
                 "reference_read_s": ref_r, "ours_read_s": min(ours_r), "read_speedup": ref_r / min(ours_r),
                 "ours_threads": os.cpu_count(), "reference_threads": 1,
                 "identical": bool(same_w and back.tobytes() == lay.tobytes() == back_ref.tobytes())})
    os.remove(a)
    os.remove(b)
    os.rmdir(d)
    for r in recs:
        print(json.dumps(r))
        if out:
            with open(out, "a") as f:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
