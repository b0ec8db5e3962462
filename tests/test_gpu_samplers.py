"""The production samplers on the device, counted inside the kernels.

Every number here comes from the Hogwild kernels while they run (DevStats
and pgl_layout_diag), not from host formulas:
  * RunStats accounting (engine.cpp:114-131, test_engine.cpp:257-312): the
    device counts primary steps, attempts, applied and skipped updates
    separately; the reference's identities must hold between them, and the
    applied fraction must sit at the reference's (0.9757 at configs 1-3,
    SURVEY.md §8 a15);
  * primary-step visits: the tile sampler enumerates the N = 10*S/srf picks
    of an iteration; with srf not dividing 10 the N mod S extra visits must
    rotate over the steps (no step favoured across iterations);
  * Zipf hops drawn by the kernels follow the pmf k^-theta / H(n, theta)
    (test_rng.cpp:107-171: known answers at n=4 theta=1, chi-square at
    n=1000 theta=0.99, merged tail at theta=2);
  * outcome frequencies on a two-step path: P(applied) = 9/16 for uniform
    selections and 3/4 for cooling ones (test_engine.cpp:210-240).
Each runs through k_sgd_tiles (register pipeline = variant 1, async
pipeline = variant 6, FP64 and anchored stores) and k_sgd_hogwild (i.i.d.).
"""
import numpy as np
import pytest
from scipy import stats as sst

pytestmark = pytest.mark.gpu

C1 = (1, 9680, 8, 0.05)

# (sampling, kernel_variant, coord_precision): the kernels the library runs
KERNELS = [
    pytest.param(0, 1, 0, id="tiles-v1-f32"),
    pytest.param(0, 1, 1, id="tiles-v1-f64"),
    pytest.param(0, 6, 1, id="tiles-v6-f64"),
    pytest.param(0, 6, 2, id="tiles-v6-anch"),
    pytest.param(0, 7, 1, id="tiles-v7-f64"),
    pytest.param(0, 7, 2, id="tiles-v7-anch"),
    pytest.param(0, 8, 1, id="tiles-v8-f64"),
    pytest.param(0, 8, 2, id="tiles-v8-anch"),
    pytest.param(0, 9, 1, id="tiles-v9-f64"),
    pytest.param(0, 9, 2, id="tiles-v9-anch"),
    pytest.param(0, 13, 1, id="tiles-v13-f64"),
    pytest.param(0, 13, 2, id="tiles-v13-anch"),
    pytest.param(1, 0, 1, id="iid-f64"),
    pytest.param(1, 0, 2, id="iid-anch"),
    pytest.param(1, 2, 1, id="iid-d3-f64"),
    pytest.param(1, 4, 2, id="iid-d4-anch"),
    pytest.param(1, 5, 1, id="iid-d4-3cta-f64"),
    pytest.param(1, 7, 2, id="iid-d4pf-anch"),
    pytest.param(1, 8, 1, id="iid-d2-f64"),
]


def ext_for(pgl, samp, variant, prec, **kw):
    return pgl.LayoutExt(sampling=samp, kernel_variant=variant, coord_precision=prec, **kw)


# ---- accounting ------------------------------------------------------------------

@pytest.mark.parametrize("samp,variant,prec", KERNELS)
def test_device_accounting_config1(pgl, gpu, samp, variant, prec):
    """Config 1, LayoutConfig{} defaults: every enumerated pick reaches the
    update stage (primary = n_iters * floor(10 S / srf)), attempted = drf per
    primary, applied + skipped = attempted from independent counters, and the
    applied fraction matches the reference's 0.9757 (skips are d_ref = 0: a
    cooling hop k=1 onto the abutting endpoint combination)."""
    g = pgl.generate_synthetic_pangenome(*C1)
    st = pgl.RunStats()
    pgl.run_layout(g, pgl.LayoutConfig(global_seed=101), stats=st, ext=ext_for(pgl, samp, variant, prec))
    spi = 10 * g.total_steps()
    assert st.primary_steps == 30 * spi
    assert st.updates_attempted == st.primary_steps
    assert st.updates_applied + st.updates_skipped == st.updates_attempted
    frac = st.updates_applied / st.updates_attempted
    assert 0.970 <= frac <= 0.981, frac


@pytest.mark.parametrize("samp,variant,prec", KERNELS)
@pytest.mark.parametrize("drf,srf", [(2, 2), (4, 4), (2, 3), (4, 1)])
def test_device_accounting_reuse(pgl, gpu, samp, variant, prec, drf, srf):
    if samp == 0 and 7 <= variant <= 14:
        pytest.skip("the lean kernel covers drf 1 only (the host picks variant 6 for reuse runs)")
    g = pgl.generate_synthetic_pangenome(3, 400, 3, 0.05)
    st = pgl.RunStats()
    cfg = pgl.LayoutConfig(n_iters=6, drf=drf, srf=srf)
    pgl.run_layout_reuse(g, cfg, stats=st, ext=ext_for(pgl, samp, variant, prec))
    assert st.primary_steps == 6 * (10 * g.total_steps() // srf)
    assert st.updates_attempted == st.primary_steps * drf
    assert st.updates_applied + st.updates_skipped == st.updates_attempted
    assert st.updates_applied > 0.9 * st.updates_attempted


def test_device_accounting_reuse_shuffle(pgl, gpu):
    g = pgl.generate_synthetic_pangenome(3, 400, 3, 0.05)
    for variant in (1, 6):
        st = pgl.RunStats()
        cfg = pgl.LayoutConfig(n_iters=6, drf=4, srf=4)
        pgl.run_layout_reuse(g, cfg, stats=st, ext=pgl.LayoutExt(reuse_shuffle=1, kernel_variant=variant))
        assert st.primary_steps == 6 * (10 * g.total_steps() // 4)
        assert st.updates_attempted == 4 * st.primary_steps
        assert st.updates_applied + st.updates_skipped == st.updates_attempted


def test_device_accounting_invalid_selections(pgl, gpu):
    """One-step paths can never form a pair: every pick landing there skips
    all drf updates (engine.cpp:128-131), counted on the device."""
    g = pgl.build_graph([3] * 12, [[(k, 0) for k in range(10)], [(10, 0)], [(11, 0)]])
    for samp in (0, 1):
        d = pgl.LayoutDiag(total_steps=g.total_steps())
        st = pgl.RunStats()
        pgl.run_layout_reuse(g, pgl.LayoutConfig(n_iters=8, drf=2, srf=1), stats=st,
                             ext=pgl.LayoutExt(sampling=samp, diag=d))
        lone = int(d.primary_visits[10:].sum())  # picks of the two one-step paths
        assert st.primary_steps == 8 * 120 == int(d.primary_visits.sum())
        assert st.updates_skipped >= 2 * lone
        assert st.updates_applied + st.updates_skipped == st.updates_attempted == 2 * st.primary_steps


# ---- primary visits ----------------------------------------------------------------

@pytest.mark.parametrize("variant", [1, 6, 8, 13])
@pytest.mark.parametrize("srf", [1, 3, 4, 7])
def test_tile_visits_rotate(pgl, gpu, variant, srf):
    """The tile sampler's enumeration: in every iteration each step is the
    primary step floor(N/S) or ceil(N/S) times (N = floor(10 S / srf)); the
    start of the enumeration moves every iteration, so over a run no part of
    the graph collects the N mod S extra visits (without the rotation the
    first N mod S steps -- the first paths -- would get them every time)."""
    g = pgl.generate_synthetic_pangenome(4, 3000, 4, 0.05)
    S = g.total_steps()
    n_iters = 2000
    d = pgl.LayoutDiag(total_steps=S)
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=n_iters, srf=srf), ext=pgl.LayoutExt(kernel_variant=variant, diag=d))
    v = d.primary_visits.astype(np.int64)
    N = 10 * S // srf
    assert v.sum() == n_iters * N
    lo, hi = N // S, -(-N // S)
    assert v.min() >= n_iters * lo and v.max() <= n_iters * hi
    per = v / n_iters
    want = N / S
    # the extra visits spread evenly: head, middle and tail of the step range
    # agree. A step takes the extra visit of an iteration when it falls in the
    # rotated stretch of N mod S steps: Bernoulli(f), f = (N mod S) / S, so a
    # part's mean visit rate has sd sqrt(f (1 - f) / n_iters) (the stretch is
    # longer than a part, which therefore moves as one step does); 5 sd. A
    # fixed start would put f on the first parts and 0 on the rest.
    f = (N % S) / S
    tol = 5 * np.sqrt(f * (1 - f) / n_iters) + 1e-12
    assert tol < 0.25 * max(f, 1e-9) or f == 0
    for part in np.array_split(per, 8):
        assert abs(part.mean() - want) <= tol, (part.mean(), want, tol)


@pytest.mark.parametrize("srf", [1, 4])
def test_iid_visits_are_uniform(pgl, gpu, srf):
    """weighted_step_select (graph.hpp:123-138): i.i.d. picks, each step with
    probability 1/S -- chi-square over the steps."""
    g = pgl.generate_synthetic_pangenome(4, 800, 3, 0.05)
    S = g.total_steps()
    d = pgl.LayoutDiag(total_steps=S)
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=100, srf=srf), ext=pgl.LayoutExt(sampling=pgl.SAMPLING_IID, diag=d))
    v = d.primary_visits.astype(np.float64)
    n = v.sum()
    assert n == 100 * (10 * S // srf)
    chi2 = ((v - n / S) ** 2 / (n / S)).sum()
    assert sst.chi2.sf(chi2, S - 1) > 1e-3


# ---- Zipf hops drawn by the kernels -------------------------------------------------

def zipf_pmf(n, theta):
    k = np.arange(1, n + 1, dtype=np.float64)
    w = k ** -theta
    return w / w.sum()


SAMPLER_KERNELS = [pytest.param(0, 1, id="tiles-v1"), pytest.param(0, 6, id="tiles-v6"),
                   pytest.param(0, 7, id="tiles-v7"), pytest.param(0, 8, id="tiles-v8"),
                   pytest.param(0, 9, id="tiles-v9"), pytest.param(0, 13, id="tiles-v13"),
                   pytest.param(1, 0, id="iid")]


@pytest.mark.parametrize("samp,variant", SAMPLER_KERNELS)
def test_zipf_draws_known_answer_n4(pgl, gpu, samp, variant):
    """test_rng.cpp:107-124: Zipf over {1..4} at theta 1 = {.48,.24,.16,.12}
    +- .005, drawn by the kernels' cooling selections (five-step paths with
    zipf_space_max 4: every path's support is 4, the speculated zdef one)."""
    walks = [[(5 * p + k, 0) for k in range(5)] for p in range(400)]
    g = pgl.build_graph([7] * 2000, walks)
    d = pgl.LayoutDiag(zipf_len=8)
    cfg = pgl.LayoutConfig(n_iters=40, zipf_space_max=4, zipf_theta=1.0)
    pgl.run_layout(g, cfg, ext=pgl.LayoutExt(sampling=samp, kernel_variant=variant, diag=d))
    c = d.zipf_draws.astype(np.float64)
    assert c[0] == 0 and c[5:].sum() == 0
    n = c.sum()
    assert n > 200_000
    np.testing.assert_allclose(c[1:5] / n, [0.48, 0.24, 0.16, 0.12], atol=0.005)


@pytest.mark.parametrize("samp,variant", SAMPLER_KERNELS)
def test_zipf_draws_chi2_n1000(pgl, gpu, samp, variant):
    """test_rng.cpp:126-147: goodness of fit at n=1000, theta=0.99 (paths of
    20k steps: support min(|p|-1, 1000) = 1000)."""
    g = pgl.generate_synthetic_pangenome(8, 20000, 4, 0.0)
    d = pgl.LayoutDiag(zipf_len=1002)
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=24), ext=pgl.LayoutExt(sampling=samp, kernel_variant=variant, diag=d))
    c = d.zipf_draws.astype(np.float64)
    assert c[0] == 0 and c[1001] == 0
    obs = c[1:1001]
    n = obs.sum()
    exp = zipf_pmf(1000, 0.99) * n
    assert exp.min() >= 5.0
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert sst.chi2.sf(chi2, 999) > 1e-3, (n, chi2)


@pytest.mark.parametrize("samp,variant", SAMPLER_KERNELS)
def test_zipf_draws_steep_merged_tail(pgl, gpu, samp, variant):
    """test_rng.cpp:149-171: theta 2, cells 1..20 individually, 21..1000 merged."""
    g = pgl.generate_synthetic_pangenome(9, 20000, 4, 0.0)
    d = pgl.LayoutDiag(zipf_len=1002)
    cfg = pgl.LayoutConfig(n_iters=12, zipf_theta=2.0)
    pgl.run_layout(g, cfg, ext=pgl.LayoutExt(sampling=samp, kernel_variant=variant, diag=d))
    c = d.zipf_draws.astype(np.float64)[1:1001]
    pmf = zipf_pmf(1000, 2.0)
    obs = np.append(c[:20], c[20:].sum())
    p = np.append(pmf[:20], pmf[20:].sum())
    exp = p * obs.sum()
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert sst.chi2.sf(chi2, 20) > 1e-3, chi2


def test_zipf_draws_mixed_supports(pgl, gpu):
    """Paths of different lengths use different supports (zipf_params_for,
    engine.cpp:36-39): the zdef speculation must not leak the most common
    support into other paths. Two-path graph: the draws are the mixture of
    Zipf(1000) and Zipf(9), weighted by the paths' cooling selections."""
    walks = [[(k, 0) for k in range(30000)], [(30000 + k, 0) for k in range(10)]] + \
            [[(30010 + 10 * p + k, 0) for k in range(10)] for p in range(300)]
    g = pgl.build_graph([5] * (30010 + 3000), walks)
    for samp, variant in [(0, 1), (0, 6), (0, 8), (1, 0)]:
        d = pgl.LayoutDiag(zipf_len=1002)
        pgl.run_layout(g, pgl.LayoutConfig(n_iters=16), ext=pgl.LayoutExt(sampling=samp, kernel_variant=variant,
                                                                          diag=d))
        c = d.zipf_draws.astype(np.float64)
        # the short paths' support is 9: their draws k in 1..9; the long path's
        # cells 10..1000 carry only its own Zipf(1000) mass
        tail = c[10:1001]
        long_n = tail.sum() / zipf_pmf(1000, 0.99)[9:].sum()
        short_n = c[1:1001].sum() - long_n
        head = c[1:10] - long_n * zipf_pmf(1000, 0.99)[:9]
        np.testing.assert_allclose(head / short_n, zipf_pmf(9, 0.99), atol=0.01)


# ---- selection outcome frequencies (test_engine.cpp:210-240) -------------------------

@pytest.mark.parametrize("samp,variant", SAMPLER_KERNELS)
def test_outcome_frequencies_two_step_path(pgl, gpu, samp, variant):
    """Two abutting steps of length 5: an endpoint combination collides at
    the shared position with probability 1/4; a uniform selection abandons
    1/4 of its draws (two collisions on a two-step path). So P(applied) =
    9/16 for uniform selections and 3/4 for cooling ones, +-0.02. (The lean
    kernels need >= 32 steps: 64 disjoint two-step paths, same frequencies.)"""
    n_paths, n_iters = (64, 200) if samp == 0 and 7 <= variant <= 14 else (1, 8000)
    g = pgl.build_graph([5] * (2 * n_paths), [[(2 * p, 0), (2 * p + 1, 0)] for p in range(n_paths)])
    d = pgl.LayoutDiag()
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=n_iters, global_seed=9),
                   ext=pgl.LayoutExt(sampling=samp, kernel_variant=variant, diag=d))
    ua, uap, ca, cap = d.outcomes
    assert ua + ca == n_iters * 20 * n_paths
    assert ua > 15000 and ca > 15000
    assert abs(uap / ua - 9 / 16) <= 0.02, uap / ua
    assert abs(cap / ca - 3 / 4) <= 0.02, cap / ca


# ---- the lean kernel's preconditions ---------------------------------------------------

def test_lean_kernel_preconditions(pgl, gpu):
    """Variants 7/8 (k_sgd_lean) cover batch 32, drf 1, pair_window 3 and
    32 <= S < 2^30 only; asked for anything else they refuse loudly, and the
    auto choice never picks them there."""
    g = pgl.generate_synthetic_pangenome(3, 400, 3, 0.05)
    tiny = pgl.build_graph([4] * 6, [[(k, 0) for k in range(6)]])
    for gg, cfg, ext in [(g, dict(batch_size=7), {}), (g, {}, dict(pair_window=2)), (tiny, {}, {}),
                         (g, {}, dict(kernel_variant=8 | 16))]:
        with pytest.raises(pgl.InvalidParameter):
            pgl.run_layout(gg, pgl.LayoutConfig(n_iters=2, **cfg),
                           ext=pgl.LayoutExt(**{"kernel_variant": 8, **ext}))
    with pytest.raises(pgl.InvalidParameter):
        pgl.run_layout_reuse(g, pgl.LayoutConfig(n_iters=2, drf=2, srf=2), ext=pgl.LayoutExt(kernel_variant=7))
    # unit length / random order: a power of two, below 32 only with the random order, lean kernel only
    for ext in [dict(kernel_variant=7, unit_len=3, unit_order=pgl.ORDER_RANDOM),
                dict(kernel_variant=7, unit_len=8),
                dict(kernel_variant=6, unit_order=pgl.ORDER_RANDOM),
                dict(sampling=pgl.SAMPLING_IID, unit_order=pgl.ORDER_RANDOM)]:
        with pytest.raises(pgl.InvalidParameter):
            pgl.run_layout(g, pgl.LayoutConfig(n_iters=2), ext=pgl.LayoutExt(**ext))


@pytest.mark.parametrize("variant", [7, 9, 13])
@pytest.mark.parametrize("unit_len", [1, 4, 32])
def test_lean_random_units_visit_uniformly(pgl, gpu, variant, unit_len):
    """PGL_ORDER_RANDOM with unit_len picks: every step's primary-visit count
    is Binomial-like around N/S (no step range favoured: chi-square over 16
    stretches of the step range), the device RunStats identities hold."""
    g = pgl.generate_synthetic_pangenome(4, 3000, 4, 0.05)
    S = g.total_steps()
    d = pgl.LayoutDiag(total_steps=S)
    st = pgl.RunStats()
    n_iters = 200
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=n_iters), stats=st,
                   ext=pgl.LayoutExt(kernel_variant=variant, unit_order=pgl.ORDER_RANDOM, unit_len=unit_len,
                                     pair_window=1, diag=d))
    v = d.primary_visits.astype(np.float64)
    assert v.sum() == n_iters * 10 * S == st.primary_steps
    assert st.updates_applied + st.updates_skipped == st.updates_attempted
    parts = np.array([p.sum() for p in np.array_split(v, 16)])
    exp = np.array([len(p) for p in np.array_split(v, 16)]) * v.sum() / S
    # unit starts are i.i.d.: counts of a stretch are sums of unit_len-step runs
    chi2 = ((parts - exp) ** 2 / (exp * unit_len)).sum()
    assert sst.chi2.sf(chi2, 15) > 1e-4, chi2


@pytest.mark.parametrize("variant", [7, 8, 13, 14])
@pytest.mark.parametrize("prec", [0, 1, 2])
def test_lean_kernel_batches_and_tail(pgl, gpu, variant, prec):
    """Every unit is one batch of 32 picks opened by lane 0, the partial last
    unit included (engine.cpp:115-124 with batch 32): the device's batch
    counters equal ceil(N/32) per iteration, split between the halves, and
    the first half's cooling batches are ~Bernoulli(1/2)."""
    g = pgl.generate_synthetic_pangenome(5, 3000, 5, 0.05)
    S = g.total_steps()
    N = 10 * S
    assert N % 32 != 0 or S % 32 != 0
    st = pgl.RunStats()
    pgl.run_layout(g, pgl.LayoutConfig(n_iters=30, global_seed=3), stats=st,
                   ext=pgl.LayoutExt(kernel_variant=variant, coord_precision=prec))
    units = -(-N // 32)
    assert st.batches_first_half == 15 * units
    assert st.batches_second_half == st.batches_second_half_cooling == 15 * units
    frac = st.batches_first_half_cooling / st.batches_first_half
    assert abs(frac - 0.5) < 5 / np.sqrt(st.batches_first_half), frac
    assert st.primary_steps == st.updates_attempted == 30 * N
    assert st.updates_applied + st.updates_skipped == st.updates_attempted


@pytest.mark.parametrize("base,rec8", [(10, 13), (9, 14)])
@pytest.mark.parametrize("prec", [1, 2])
def test_lean_rec8_matches_16_byte_records(pgl, gpu, base, rec8, prec):
    """Variants 13/14 read 8-byte records {node | reverse << 31, offset}
    (offset(k+1) = the far end of step k, a sentinel after each path)
    instead of the 16-byte records; with one warp the kernel is
    deterministic, so on a nested graph (reverse steps, revisits, path ends
    inside units) both record formats must give the identical layout and
    RunStats."""
    g = pgl.generate_nested_pangenome(7, 600, 12, 3, 0.05)
    outs, stats = [], []
    for v in (base, rec8):
        st = pgl.RunStats()
        outs.append(pgl.run_layout(g, pgl.LayoutConfig(n_iters=6, global_seed=11), stats=st,
                                   ext=pgl.LayoutExt(kernel_variant=v, coord_precision=prec, max_warps=1)))
        stats.append((st.primary_steps, st.updates_applied, st.updates_skipped))
    assert stats[0] == stats[1]
    assert np.array_equal(outs[0], outs[1])
