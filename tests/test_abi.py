"""CPU-side checks of the product boundary: libpgl_b200.so loads and exports
every symbol include/pgl_b200.h declares; the host-side helpers of the path
(generator fixture, make_schedule, init_layout, validation, error typing)
agree bit-for-bit with the oracle; the bench's multi-rank aggregation works
over gloo with world_size 2. No compute call needs a GPU here."""
import ctypes
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle_ffi import make_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgl_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pgl_[a-z0-9_]+)\s*\(", text)) - {"pgl_iteration_cb"})


def test_library_exports_every_declared_symbol(pgl):
    lib = ctypes.CDLL(pgl.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_cubin(pgl):
    out = subprocess.run(["cuobjdump", "--list-elf", pgl.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_oracle_linkage(pgl):
    """The product must not link the checker."""
    out = subprocess.run(["ldd", pgl.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "pglref" not in out
    syms = subprocess.run(["nm", "-D", pgl.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in syms and "pglref" not in syms


@pytest.mark.parametrize("args", [(1, 9680, 8, 0.05), (3, 50, 4, 0.3), (7, 5000, 12, 0.05),
                                  (1, 100, 3, 0.0), (5, 30, 3, 1.0), (9, 2, 1, 0.5)])
def test_generator_fixture_bit_exact(pgl, oracle, args):
    g, go = pgl.generate_synthetic_pangenome(*args), oracle.generate(*args)
    f = oracle.export(go)
    steps = np.concatenate(g.path_steps)
    assert np.array_equal(g.node_len, f.node_len)
    assert np.array_equal(g.cum_steps(), f.cum)
    assert np.array_equal(steps["node_id"], f.step_node)
    assert np.array_equal(steps["offset"], f.step_off)
    assert np.array_equal(steps["seq_len"], f.step_len)
    assert np.array_equal(steps["orient"], f.step_rev)
    assert np.array_equal(g.path_total_len, f.path_total)


@pytest.mark.parametrize("args", [(1, 9680, 8, 0.05), (3, 50, 4, 0.3)])
def test_schedule_and_init_bit_exact(pgl, oracle, args):
    g, go = pgl.generate_synthetic_pangenome(*args), oracle.generate(*args)
    for n in (1, 2, 7, 30):
        assert np.array_equal(pgl.make_schedule(g, pgl.LayoutConfig(n_iters=n)),
                              oracle.schedule(go, make_cfg(n_iters=n)))
    for seed in (0, 42, 2**63 + 5):
        assert np.array_equal(pgl.init_layout(g, seed), oracle.init_layout(go, seed))


def test_build_graph_matches_oracle(pgl, oracle):
    lens = [5, 3, 7, 2, 9, 4]
    walks = [[(0, 0), (1, 1), (2, 0), (1, 0), (3, 1), (0, 0), (4, 0)], [(5, 1), (2, 1)], [(1, 0)]]
    g, go = pgl.build_graph(lens, walks), oracle.build(lens, walks)
    f = oracle.export(go)
    steps = np.concatenate(g.path_steps)
    assert np.array_equal(steps["offset"], f.step_off)
    assert np.array_equal(steps["orient"], f.step_rev)
    assert np.array_equal(pgl.init_layout(g, 3), oracle.init_layout(go, 3))


def test_build_graph_validation(pgl):  # test_graph.cpp:40-47
    with pytest.raises(pgl.InvalidParameter):
        pgl.build_graph([0], [])
    with pytest.raises(pgl.UnknownNode):
        pgl.build_graph([5], [[(3, 0)]])
    with pytest.raises(pgl.EmptyPath):
        pgl.build_graph([5], [[]])


def test_generator_validation(pgl):  # test_graph.cpp:125-133
    for bad in [(1, 1, 1, 0.0), (1, 10, 0, 0.0), (1, 10, 1, -0.1), (1, 10, 1, 1.01)]:
        with pytest.raises(pgl.InvalidParameter):
            pgl.generate_synthetic_pangenome(*bad)
    pgl.generate_synthetic_pangenome(1, 10, 1, 1.0)


def test_config_validated_before_device(pgl):
    """Usage errors surface with the reference type and message before any
    device work (engine.cpp:15-28), so they are testable without a GPU."""
    g = pgl.build_graph([5, 3], [[(0, 0), (1, 0)]])
    cases = {"drf": (3, "drf must be 1, 2 or 4"), "threads": (0, "threads must be >= 1"),
             "batch_size": (0, "batch_size must be >= 1"), "n_iters": (0, "n_iters must be >= 1"),
             "zipf_theta": (0.0, "zipf_theta must be positive"),
             "zipf_space_max": (0, "zipf_space_max must be >= 1"),
             "eta_min_eps": (0.0, "eta_min_eps must be positive"), "srf": (0, "srf must be >= 1")}
    for field, (val, msg) in cases.items():
        with pytest.raises(pgl.InvalidParameter) as e:
            pgl.run_layout(g, pgl.LayoutConfig(**{field: val}))
        assert str(e.value) == "InvalidParameter: " + msg and e.value.kind == "usage"
    with pytest.raises(pgl.InvalidParameter, match="update reuse needs drf of 2 or 4"):
        pgl.run_layout_reuse(g, pgl.LayoutConfig(drf=1))
    with pytest.raises(pgl.DegenerateGraph, match="layout needs at least one path with two or more steps"):
        pgl.run_layout(pgl.build_graph([5], [[(0, 0)]]))
    with pytest.raises(pgl.DegenerateGraph):
        pgl.make_schedule(pgl.build_graph([5], [[(0, 0)]]), pgl.LayoutConfig())
    with pytest.raises(pgl.InvalidParameter, match="0 < eta_min <= eta_max"):
        pgl.make_schedule(g, pgl.LayoutConfig(eta_min_eps=1e9))


def test_no_device_is_a_loud_internal_error(pgl):
    if pgl.device_count() > 0:
        pytest.skip("a GPU is visible")
    g = pgl.build_graph([5, 3], [[(0, 0), (1, 0)]])
    with pytest.raises(pgl.CudaError) as e:
        pgl.run_layout(g)
    assert e.value.kind == "internal"


def test_config_struct_is_layout_config_abi(pgl):
    """pgl_layout_config mirrors LayoutConfig (engine.hpp:13-23) offsets."""
    C = pgl._Cfg
    assert ctypes.sizeof(C) == 56
    assert [getattr(C, f).offset for f in ("global_seed", "n_iters", "threads", "batch_size",
                                            "zipf_theta", "zipf_space_max", "eta_min_eps", "drf", "srf")] == \
        [0, 8, 12, 16, 24, 32, 40, 48, 52]
    d = pgl._Cfg()
    pgl._lib.pgl_layout_config_default(ctypes.byref(d))
    assert (d.global_seed, d.n_iters, d.threads, d.batch_size, d.zipf_theta, d.zipf_space_max,
            d.eta_min_eps, d.drf, d.srf) == (42, 30, 1, 32, 0.99, 1000, 0.01, 1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_aggregation_two_ranks_gloo(tmp_path):
    """bench.py's N>1 plumbing: barrier, sum of units, max over ranks."""
    script = tmp_path / "agg.py"
    script.write_text(f"""
import os, sys, json
sys.path.insert(0, {ROOT!r})
import bench
d = bench.Dist(2)
rank = d.rank
value, t = bench.aggregate(d, units=100.0 * (rank + 1), per_rank_seconds=1.0 + rank)
d.barrier()
if rank == 0:
    print(json.dumps({{"value": value, "t": t, "world": d.world}}))
d.close()
""".replace("units=", "").replace("per_rank_seconds=", ""))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE="2",
               CUDA_VISIBLE_DEVICES="")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    import json
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    assert res == {"value": 300.0 / 2.0, "t": 2.0, "world": 2}


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_c4_share_is_an_lpt_partition(n):
    """bench.py's config-4 split: the ranks' shares partition the 24
    chromosomes, follow LPT (longest first onto the least-loaded rank) and
    stay within Graham's 4/3 bound of the ideal makespan."""
    import bench
    shares = [bench.c4_share(n, r)[0] for r in range(n)]
    sizes = bench.c4_share(n, 0)[1]
    allc = sorted(c for s in shares for c in s)
    assert allc == list(range(24))
    loads = [sum(sizes[c] for c in s) for s in shares]
    assert max(loads) <= 4 / 3 * sum(sizes) / n + max(sizes)
    # rank 0 of any split takes chr1, the largest
    assert shares[0][0] == 0


def test_c4_shares_two_ranks_gloo(tmp_path):
    """The config-4 phase's plumbing over two gloo ranks: disjoint shares
    whose union is the set, summed work and max-over-ranks makespan."""
    script = tmp_path / "c4.py"
    script.write_text(f"""
import os, sys, json
sys.path.insert(0, {ROOT!r})
import bench
d = bench.Dist(2)
mine, sizes = bench.c4_share(d.world, d.rank)
work = d.sum(float(sum(sizes[c] for c in mine)))
ms = d.max(float(len(mine)))
print(json.dumps({{"rank": d.rank, "mine": mine, "work": work, "max": ms}}))
d.close()
""")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE="2",
               CUDA_VISIBLE_DEVICES="")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    import json
    res = [json.loads(o[0].strip().splitlines()[-1]) for o in outs]
    assert sorted(res[0]["mine"] + res[1]["mine"]) == list(range(24))
    assert not set(res[0]["mine"]) & set(res[1]["mine"])
    import bench
    assert res[0]["work"] == res[1]["work"] == float(sum(bench.c4_share(1, 0)[1]))
    assert res[0]["max"] == max(len(r["mine"]) for r in res)
