"""Multi-GPU shard scheduler (pgl_shard_plan / pgl_layout_shards, SURVEY.md
§8e): independent graphs (the 24 chromosomes of config 4) spread over
devices by LPT, no collective.

CPU tests check the plan against a plain restatement of LPT and its
error behaviour; the GPU test drives the threaded scheduler with two
"devices" that are both cuda:0 (one host thread and stream each) in replay
mode, where every graph's layout is bit-exact with the oracle whichever
worker ran it."""
import numpy as np
import pytest

from oracle_ffi import make_cfg

ARGS = [(11, 60, 2, 0.1), (3, 50, 4, 0.3), (5, 30, 3, 0.3), (12, 50, 2, 0.1), (7, 200, 3, 0.05),
        (8, 120, 1, 0.0)]


def lpt(work, n_dev):
    order = sorted(range(len(work)), key=lambda k: -work[k])  # stable: ties keep index order
    load = [0.0] * n_dev
    out = [0] * len(work)
    for k in order:
        d = min(range(n_dev), key=lambda i: (load[i], i))
        load[d] += work[k]
        out[k] = d
    return out, load


@pytest.mark.parametrize("n_dev", [1, 2, 3, 8])
def test_plan_is_lpt_over_update_counts(pgl, n_dev):
    graphs = [pgl.generate_synthetic_pangenome(*a) for a in ARGS]
    cfgs = [pgl.LayoutConfig(n_iters=10 + k, drf=1 + (k % 2), srf=1) for k in range(len(graphs))]
    assign, work, load = pgl.shard_plan(graphs, cfgs, n_dev)
    want_work = [g.total_steps() * c.n_iters * c.drf / c.srf for g, c in zip(graphs, cfgs)]
    assert np.array_equal(work, want_work)
    want, want_load = lpt(want_work, n_dev)
    assert assign == want
    assert np.allclose(load, want_load)
    assert sum(load) == pytest.approx(sum(want_work))
    # LPT's bound: makespan <= 4/3 OPT, and OPT >= max(mean load, heaviest graph)
    assert max(load) <= 4 / 3 * max(sum(want_work) / n_dev, max(want_work)) + 1e-9


def test_plan_chromosome_like_sizes(pgl):
    """24 graphs of decreasing size on 8 devices (the config-4 shape)."""
    graphs = [pgl.generate_synthetic_pangenome(100 + k, 40 * (25 - k), 2, 0.05) for k in range(24)]
    cfgs = [pgl.LayoutConfig()] * 24
    assign, work, load = pgl.shard_plan(graphs, cfgs, 8)
    assert sorted(set(assign)) == list(range(8))
    assert max(load) / (sum(load) / 8) < 1.1


def test_plan_errors(pgl):
    g = pgl.generate_synthetic_pangenome(*ARGS[0])
    with pytest.raises(pgl.InvalidParameter):
        pgl.shard_plan([g], [pgl.LayoutConfig()], 0)
    with pytest.raises(pgl.InvalidParameter):
        pgl.shard_plan([g], [pgl.LayoutConfig(n_iters=0)], 2)
    assert pgl.shard_plan([], [], 4)[0] == []


@pytest.mark.gpu
def test_shards_threaded_replay_bit_exact(pgl, oracle, gpu):
    graphs = [pgl.generate_synthetic_pangenome(*a) for a in ARGS]
    kws = [dict(n_iters=3 + k, global_seed=50 + k) for k in range(len(ARGS))]
    cfgs = [pgl.LayoutConfig(**kw) for kw in kws]
    outs, secs, assign = pgl.layout_shards(graphs, cfgs, [0, 0],
                                           ext=pgl.LayoutExt(mode=pgl.MODE_REPLAY))
    assert assign == pgl.shard_plan(graphs, cfgs, 2)[0]
    assert set(assign) == {0, 1} and all(s > 0 for s in secs)
    for a, kw, out in zip(ARGS, kws, outs):
        ref, _ = oracle.run_layout(oracle.generate(*a), make_cfg(**kw))
        assert np.array_equal(out, ref)


@pytest.mark.gpu
def test_shards_hogwild_and_errors(pgl, gpu):
    graphs = [pgl.generate_synthetic_pangenome(*a) for a in ARGS[:3]]
    cfgs = [pgl.LayoutConfig()] * 3
    outs, _, assign = pgl.layout_shards(graphs, cfgs, [0, 0, 0])
    assert sorted(assign) == [0, 1, 2]
    for g, out in zip(graphs, outs):
        assert out.shape == (4 * g.n_nodes,) and np.isfinite(out).all()
    with pytest.raises(pgl.Error):
        pgl.layout_shards(graphs, cfgs, [pgl.device_count() + 5])
