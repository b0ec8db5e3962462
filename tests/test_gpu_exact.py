"""GPU exact path stress (pgl_exact_path_stress) against the reference's
exact_path_stress (metrics.cpp:75-106) and its C restatement.

Bars: n and skipped identical; mean within 1e-12 relative (1e-10 at config
1's 3.7e8 pairs, where the reference's own serial double sum drifts by
~1e-12; the device sums the reference's bit-identical per-pair terms in
double-double with a fixed fold order); sigma and CI within 1e-9 relative;
the device result is bit-reproducible run to run."""
import numpy as np
import pytest

from test_gpu_parity import C1, SMALL, both, revisit_graph

pytestmark = pytest.mark.gpu

MID = (4, 2000, 4, 0.05)


def check(got, want, rtol_mean=1e-12, rtol_sd=1e-9):
    assert got.n == want.n and got.skipped == want.skipped, (got, want)
    assert got.mean == pytest.approx(want.mean, rel=rtol_mean, abs=1e-300)
    assert got.std_dev == pytest.approx(want.std_dev, rel=rtol_sd, abs=1e-300)
    assert got.ci_low == pytest.approx(want.ci_low, rel=rtol_sd, abs=1e-300)
    assert got.ci_high == pytest.approx(want.ci_high, rel=rtol_sd, abs=1e-300)


@pytest.mark.parametrize("args", SMALL + [MID])
def test_exact_stress_matches_reference_init_and_layout(pgl, oracle, ref, gpu, args):
    g, go = both(pgl, oracle, args)
    gr = ref.generate(*args)
    for lay in (ref.init_layout(gr, 7), pgl.run_layout(g, pgl.LayoutConfig(global_seed=3))):
        want = ref.exact(gr, lay)
        check(pgl.exact_path_stress(g, lay), want)
        o = oracle.exact(go, lay)
        assert (o.n, o.skipped) == (want.n, want.skipped)


def test_exact_stress_revisits_and_degenerate_pairs(pgl, oracle, gpu):
    """Reverse steps and revisits give zero-d_ref endpoint combinations,
    which drop out of a pair's average (metrics.cpp:59-73). (A whole pair is
    never skipped: two distinct steps of positive length always have a
    combination with a nonzero reference distance.)"""
    g, go = revisit_graph(pgl, oracle)
    lay = pgl.init_layout(g, 5)
    want = oracle.exact(go, lay)
    got = pgl.exact_path_stress(g, lay)
    check(got, want)


def test_exact_stress_perfect_layout_is_zero(pgl, gpu):
    """One straight path laid out at its own positions: every term is 0
    (test_metrics.cpp:246-254 for the sampled metric)."""
    lens = [4, 6, 3, 5]
    g = pgl.build_graph(lens, [[(0, 0), (1, 0), (2, 0), (3, 0)]])
    x = np.cumsum([0] + lens)
    lay = np.zeros(16)
    for k in range(4):
        lay[4 * k + 0], lay[4 * k + 2] = x[k], x[k + 1]
    r = pgl.exact_path_stress(g, lay)
    assert r.mean == 0.0 and r.n == 6 and r.skipped == 0


def test_exact_stress_resident_layout_and_determinism(pgl, oracle, gpu):
    g, go = both(pgl, oracle, MID)
    with pgl.DeviceGraph(g) as dg:
        lay = dg.layout(pgl.LayoutConfig(global_seed=11))
        a = dg.exact_stress()            # the resident layout
        b = dg.exact_stress(lay)         # the same layout from the host
        c = dg.exact_stress(lay)
    assert (a.mean, a.n, a.std_dev, a.skipped) == (b.mean, b.n, b.std_dev, b.skipped)
    assert (b.mean, b.n, b.std_dev, b.ci_low, b.ci_high) == (c.mean, c.n, c.std_dev, c.ci_low, c.ci_high)
    check(b, oracle.exact(go, lay))


@pytest.mark.slow
def test_exact_stress_config1(pgl, ref, gpu):
    """Config 1 (3.8e8 step pairs): the reference's single-threaded exact metric."""
    g = pgl.generate_synthetic_pangenome(*C1)
    gr = ref.generate(*C1)
    lay = pgl.run_layout(g, pgl.LayoutConfig(global_seed=101))
    # the reference sums 3.7e8 terms serially in double: its own rounding is
    # ~sqrt(n) * eps ~ 1e-12 relative (measured up to 1.1e-12), so the bar is
    # 1e-10 here; the device sum is double-double
    check(pgl.exact_path_stress(g, lay), ref.exact(gr, lay), rtol_mean=1e-10, rtol_sd=1e-9)
