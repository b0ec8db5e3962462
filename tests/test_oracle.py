"""Pins the C oracle (oracle/pgl_oracle.c) before it is trusted as the GPU
checker: against golden vectors produced by the reference itself
(tests/golden/reference_vectors.json, from tests/golden/make_golden.py), against
the live reference library when it is built (oracle/_ref), and against the
known answers of the reference's own tests (test_graph.cpp, test_rng.cpp,
test_engine.cpp, test_metrics.cpp)."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle_ffi import make_cfg, stress_tuple

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- golden vectors (the reference's own outputs) ------------------------------

def test_rng_streams_match_golden(oracle):
    for key, vals in GOLD["rng"].items():
        s, w = (int(x) for x in key.split("_"))
        assert [str(x) for x in oracle.rng_draws(s, w, 16)] == vals


def test_zipf_streams_match_golden(oracle):
    for key, vals in GOLD["zipf"].items():
        n, t = key.split("_")
        assert oracle.zipf(int(n), float(t), 99, 0, 64).tolist() == vals


@pytest.mark.parametrize("name", sorted(GOLD["graphs"]))
def test_graph_index_matches_golden(oracle, name):
    d = GOLD["graphs"][name]
    g = oracle.generate(*d["args"])
    f = oracle.export(g)
    assert (g.n_nodes, g.n_paths, g.total_steps, g.total_nt) == (
        d["n_nodes"], d["n_paths"], d["total_steps"], d["total_nt"])
    assert sha(f.node_len) == d["node_len"]
    assert sha(f.step_node) == d["step_node"] and sha(f.step_rev) == d["step_rev"]
    assert sha(f.step_off) == d["step_off"] and sha(f.step_len) == d["step_len"]
    assert f.path_total.tolist() == d["path_total"]
    assert (f.cum.tolist() if len(f.cum) < 200 else sha(f.cum)) == d["cum"]
    assert sha(f.positions().reshape(-1)) == d["positions"]


@pytest.mark.parametrize("name", sorted(GOLD["graphs"]))
def test_init_schedule_stress_match_golden(oracle, name):
    d = GOLD["graphs"][name]
    g = oracle.generate(*d["args"])
    init = oracle.init_layout(g, 42)
    assert sha(init) == d["init_42"]
    assert oracle.schedule(g, make_cfg()).tolist() == d["etas_30"]
    assert list(stress_tuple(oracle.sps(g, init, 7, 10))) == d["sps_init_42_7_10"]
    if "exact_init_42" in d:
        assert list(stress_tuple(oracle.exact(g, init))) == d["exact_init_42"]


@pytest.mark.parametrize("name,case", [(n, c) for n in sorted(GOLD["graphs"])
                                       for c in sorted(GOLD["graphs"][n]["layouts"])])
def test_layouts_match_golden(oracle, name, case):
    d = GOLD["graphs"][name]
    L = d["layouts"][case]
    g = oracle.generate(*d["args"])
    cfg = make_cfg(**L["cfg"])
    lay, st = oracle.run_layout(g, cfg, reuse=cfg.drf > 1)
    assert lay[:8].tolist() == L["first8"]
    assert sha(lay) == L["sha256"]
    assert [int(getattr(st, k)) for k, _ in st._fields_] == L["stats"]
    assert list(stress_tuple(oracle.sps(g, lay, 7, 100))) == L["sps_7_100"]


# ---- live reference (build container, or wherever oracle/_ref travelled) -----------

@pytest.mark.parametrize("args", [(4, 60, 2, 0.2), (9, 200, 4, 0.1), (2, 80, 2, 0.0), (21, 45, 3, 0.05)])
def test_oracle_equals_reference_library(oracle, ref, args):
    go, gr = oracle.generate(*args), ref.generate(*args)
    fo, fr = oracle.export(go), ref.export(gr)
    for k in fo.__dataclass_fields__:
        assert np.array_equal(getattr(fo, k), getattr(fr, k)), k
    for kw in [dict(n_iters=3, global_seed=5), dict(n_iters=4, batch_size=3, zipf_theta=1.5),
               dict(n_iters=3, drf=4, srf=2, zipf_space_max=5)]:
        cfg = make_cfg(**kw)
        a, sa = oracle.run_layout(go, cfg, reuse=cfg.drf > 1)
        b, sb = ref.run_layout(gr, cfg, reuse=cfg.drf > 1)
        assert np.array_equal(a, b)
        assert [getattr(sa, k) for k, _ in sa._fields_] == [getattr(sb, k) for k, _ in sb._fields_]
        assert stress_tuple(oracle.sps(go, a, 3, 7)) == stress_tuple(ref.sps(gr, b, 3, 7))


def test_oracle_revisits_and_reverse_match_reference(oracle, ref):
    lens = [5, 3, 7, 2, 9, 4]
    walks = [[(0, 0), (1, 1), (2, 0), (1, 0), (3, 1), (0, 0), (4, 0)],
             [(5, 1), (2, 1), (2, 1), (3, 0), (4, 1)], [(1, 0)]]
    go, gr = oracle.build(lens, walks), ref.build(lens, walks)
    assert np.array_equal(oracle.export(go).positions(), ref.positions(gr))
    cfg = make_cfg(n_iters=6, global_seed=9, batch_size=3)
    a, _ = oracle.run_layout(go, cfg)
    b, _ = ref.run_layout(gr, cfg)
    assert np.array_equal(a, b)
    assert stress_tuple(oracle.exact(go, a)) == stress_tuple(ref.exact(gr, b))


def test_oracle_errors_match_reference(oracle, ref):
    g = oracle.generate(2, 20, 1, 0.0)
    gr = ref.generate(2, 20, 1, 0.0)
    for bad in [dict(drf=3), dict(threads=0), dict(batch_size=0), dict(n_iters=0),
                dict(zipf_theta=0.0), dict(zipf_space_max=0), dict(eta_min_eps=0.0), dict(srf=0),
                dict(eta_min_eps=1e30)]:
        with pytest.raises(Exception) as eo:
            oracle.run_layout(g, make_cfg(**bad))
        with pytest.raises(Exception) as er:
            ref.run_layout(gr, make_cfg(**bad))
        assert str(eo.value) == str(er.value)


# ---- the reference tests' known answers ----------------------------------------------

def test_two_node_index(oracle):  # test_graph.cpp:24-38
    g = oracle.build([5, 3], [[(0, 0), (1, 0)]])
    f = oracle.export(g)
    assert f.step_off.tolist() == [0, 5] and f.step_len.tolist() == [5, 3]
    assert f.path_total.tolist() == [8] and f.cum.tolist() == [0, 2] and g.total_nt == 8


def test_reverse_positions(oracle):  # test_graph.cpp:49-62
    g = oracle.build([5, 3], [[(0, 0), (1, 1)]])
    assert oracle.export(g).positions().tolist() == [[0, 5], [8, 5]]


def test_linear_generator_shape(oracle):  # test_graph.cpp:93-108
    g = oracle.generate(1, 100, 3, 0.0)
    f = oracle.export(g)
    assert g.n_nodes == 100 and g.total_steps == 300
    assert f.step_node.tolist() == list(range(100)) * 3


def test_schedule_closed_forms(oracle):  # test_engine.cpp:36-77
    g = oracle.build([5, 3], [[(0, 0), (1, 0)]])
    etas = oracle.schedule(g, make_cfg(n_iters=10))
    assert abs(etas[0] - 64.0) <= 64 * 1e-9 and abs(etas[-1] - 0.01) <= 1e-11
    e30 = oracle.schedule(oracle.build([64], [[(0, 0), (0, 0)]]), make_cfg(n_iters=30))
    for t in range(30):
        closed = 16384.0 * (0.01 / 16384.0) ** (t / 29.0)
        assert abs(e30[t] - closed) <= 1e-12 * closed


def test_init_layout_known_answers(oracle):  # test_engine.cpp:79-96
    g = oracle.build([5, 3], [[(0, 0), (1, 0)]])
    a = oracle.init_layout(g, 42).reshape(2, 4)
    assert a[:, [0, 2]].tolist() == [[0.0, 5.0], [5.0, 8.0]]
    assert np.all(np.abs(a[:, [1, 3]]) <= math.sqrt(8.0))
    assert np.array_equal(oracle.init_layout(g, 42), oracle.init_layout(g, 42))
    assert not np.array_equal(oracle.init_layout(g, 42), oracle.init_layout(g, 43))


def test_update_math(oracle):  # test_engine.cpp:98-208
    s4 = np.zeros(4, np.uint64)
    c = np.zeros(8)
    c[1], c[5] = 0.0, 10.0  # (0,0) and (0,10), start endpoints
    out, _, applied = oracle.apply_update(c, 0, 0, 1, 0, 5.0, 1e6, s4)
    assert applied and abs(out[1] - 2.5) <= 1e-12 and abs(out[5] - 7.5) <= 1e-12
    rng = np.random.default_rng(0)
    for _ in range(100):  # saturated contraction, symmetry
        vi, vj = rng.uniform(-100, 100, 2), rng.uniform(-100, 100, 2)
        d = rng.uniform(0.5, 50)
        c = np.array([0, 0, *vi, 0, 0, *vj])
        out, _, _ = oracle.apply_update(c, 0, 1, 1, 1, d, 2 * d * d, s4)
        assert abs(np.hypot(*(out[2:4] - out[6:8])) - d) <= 1e-9 * d
        assert np.all(np.abs((out[2:4] - vi) + (out[6:8] - vj)) <= 1e-12 * max(np.abs([*vi, *vj]).max(), 1))
    c = np.array([3.0, 7.0, 0, 0, 3.0, 7.0, 0, 0])  # coincident: jitter, midpoint kept
    s4 = np.array([1, 2, 3, 4], np.uint64)
    out, _, _ = oracle.apply_update(c, 0, 0, 1, 0, 4.0, 1e9, s4)
    assert abs(np.hypot(*(out[0:2] - out[4:6])) - 4.0) <= 4e-9
    assert abs(0.5 * (out[0] + out[4]) - 3.0) <= 1e-12 and abs(0.5 * (out[1] + out[5]) - 7.0) <= 1e-12
    before = np.array([1.0, 2.0, 0, 0, 3.0, 4.0, 0, 0])
    out, _, applied = oracle.apply_update(before, 0, 0, 1, 0, 0.0, 10.0, s4)
    assert not applied and np.array_equal(out, before)


def test_update_follows_gradient(oracle):  # test_engine.cpp:151-180
    rng = np.random.default_rng(4)
    s4 = np.zeros(4, np.uint64)

    def ps(vi, vj, d):
        return ((np.hypot(*(vi - vj)) - d) / d) ** 2

    checked = 0
    while checked < 100:
        vi, vj = rng.uniform(-100, 100, 2), rng.uniform(-100, 100, 2)
        mag = np.hypot(*(vi - vj))
        d = rng.uniform(0.5, 50)
        if mag < 1 or abs(mag - d) < 0.1 * d:
            continue
        eta = rng.uniform(0.05, 0.9) * d * d
        c = np.array([0, 0, *vi, 0, 0, *vj])
        out, _, _ = oracle.apply_update(c, 0, 1, 1, 1, d, eta, s4)
        h = 1e-5 * max(1.0, mag)
        grad = np.array([(ps(vi + [h, 0], vj, d) - ps(vi - [h, 0], vj, d)) / (2 * h),
                         (ps(vi + [0, h], vj, d) - ps(vi - [0, h], vj, d)) / (2 * h)])
        exp = -eta / 4.0 * grad
        assert np.hypot(*(out[2:4] - vi - exp)) <= 1e-6 * np.hypot(*exp)
        checked += 1


def test_zipf_known_frequencies(oracle):  # test_rng.cpp:107-124
    s = oracle.zipf(4, 1.0, 99, 0, 1_000_000)
    freq = np.bincount(s.astype(np.int64), minlength=5)[1:] / len(s)
    assert np.all(np.abs(freq - [0.48, 0.24, 0.16, 0.12]) <= 0.005)
    assert np.all(oracle.zipf(1, 0.5, 1, 0, 1000) == 1)


def test_weighted_select_marginals(oracle):  # test_rng.cpp:210-230
    g = oracle.build([1], [[(0, 0)] * 3, [(0, 0)] * 5])
    p, s = oracle.weighted_select(g, 77, 0, 1_000_000)
    assert abs((p == 0).mean() - 0.375) <= 0.002 and abs((p == 1).mean() - 0.625) <= 0.002
    assert s[p == 0].max() == 2 and s[p == 1].max() == 4


def test_sampled_stress_perfect_layout(oracle):  # test_metrics.cpp:246-254
    g = oracle.generate(2, 80, 2, 0.0)
    f = oracle.export(g)
    lay = np.zeros(4 * g.n_nodes)
    pos = f.positions()
    lay[4 * f.step_node.astype(np.int64)] = pos[:, 0]
    lay[4 * f.step_node.astype(np.int64) + 2] = pos[:, 1]
    r = oracle.sps(g, lay, 7)
    assert (r.mean, r.std_dev, r.ci_low, r.ci_high) == (0.0, 0.0, 0.0, 0.0)
    assert r.n + r.skipped == 100 * 2 * 80
    rc = oracle.sps_counter(g, lay, 7)
    assert rc.mean == 0.0 and rc.n + rc.skipped == 100 * 2 * 80


def test_counter_estimator_is_unbiased(oracle):
    """The counter-based estimator (the GPU's) and the reference stream agree
    in distribution: z-test over seeds (test_metrics.cpp:308-327)."""
    g = oracle.generate(31, 120, 2, 0.1)
    lay, _ = oracle.run_layout(g, make_cfg(n_iters=6))
    agree = 0
    for k in range(60):
        a, b = oracle.sps_counter(g, lay, 1000 + k), oracle.sps(g, lay, 1000 + k)
        se = math.hypot(a.std_dev / math.sqrt(a.n), b.std_dev / math.sqrt(b.n))
        agree += abs(a.mean - b.mean) <= 1.96 * se
    assert agree >= 52


def test_counter_ci_formula(oracle):  # test_metrics.cpp:297-306
    g = oracle.generate(6, 80, 2, 0.1)
    r = oracle.sps_counter(g, oracle.init_layout(g, 6), 11)
    half = 1.96 * r.std_dev / math.sqrt(r.n)
    assert abs((r.ci_high - r.mean) - half) <= 1e-12 * half
    assert abs((r.mean - r.ci_low) - half) <= 1e-12 * half
