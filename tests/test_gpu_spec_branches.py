"""Device tests of the SPEC branches of fit_em / select_k_bic / detect that the
headline workloads never take, each through the C-ABI and against the oracle:

  collapse reseed and RepeatedCollapse
  SingularCovariance after an M-step        SPEC.md:265 (reg disabled)
  mixture-density detect / calibrate mode
  select_k_bic, full covariance             SPEC.md:301-309 (its three examples + BIC values)
  acceptance #1 (EM monotonicity)           SPEC.md:543 (>= 20 seeded fits, 3 datasets, d in {1,2,3})
  acceptance #2 (parameter recovery)
"""
import numpy as np
import pytest

from test_gpu_parity import BAND, LL_TOL, assert_params

pytestmark = pytest.mark.gpu


def _blobs(seed, centers, n_each, d):
    rng = np.random.default_rng(seed)
    return np.concatenate([rng.normal(c, 1.0, size=(n_each, d)) for c in centers])


def _given(pi, mu, cov):
    return np.asarray(pi, float), np.asarray(mu, float), np.asarray(cov, float)


# ------------------------------------------------------------- collapse
def test_collapse_reseed_matches_oracle(es, oracle):
    """A component placed far from every event gets responsibility exactly 0 (N_k = 0 < 1):
    its mean is reseeded at a uniformly drawn event, its covariance reset to the data
    covariance (+ reg), its weight to 1/K before renormalisation; the fit then continues."""
    X = _blobs(1, [(-4, 0, 0), (4, 0, 0), (0, 5, 0)], 3000, 3)
    pi, mu, cov = _given([0.3, 0.3, 0.3, 0.1], [(-4, 0, 0), (4, 0, 0), (0, 5, 0), (1e3, 1e3, 1e3)],
                         np.repeat(np.eye(3)[None], 4, 0))
    init = es.GmmModel(pi, mu, cov)
    m = es.fit_em(X, 4, init_params=init, tol=0.0, max_iter=12, seed=5)
    opi, omu, ocov, rep = oracle.fit_em(X, 4, init_params=(pi, mu, cov), tol=0.0, max_iter=12, seed=5)
    assert rep["collapses"] == 1 and m.fit_report.collapses == 1
    assert_params(m, opi, omu, ocov)
    assert np.allclose(m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"],
                       rtol=LL_TOL, atol=0)
    assert abs(m.weights.sum() - 1) < 1e-12


def test_repeated_collapse_raises(es, oracle):
    """Three components with no events collapse in the first M-step: the third reseed is
    refused with RepeatedCollapse (kind Numeric), at most twice per fit."""
    X = _blobs(2, [(-4, 0), (4, 0)], 2000, 2)
    far = [(1e3, 1e3), (-1e3, 1e3), (1e3, -1e3)]
    pi, mu, cov = _given([0.25, 0.25, 0.5 / 3, 0.5 / 3, 0.5 / 3], [(-4, 0), (4, 0)] + far,
                         np.repeat(np.eye(2)[None], 5, 0))
    with pytest.raises(oracle.OracleError) as eo:
        oracle.fit_em(X, 5, init_params=(pi, mu, cov), tol=0.0, max_iter=5, seed=1)
    assert eo.value.name == "RepeatedCollapse"
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(X, 5, init_params=es.GmmModel(pi, mu, cov), tol=0.0, max_iter=5, seed=1)
    assert e.value.name == "RepeatedCollapse" and e.value.kind == "Numeric"


def test_two_collapses_are_allowed(es, oracle):
    X = _blobs(3, [(-4, 0), (4, 0)], 2000, 2)
    pi, mu, cov = _given([0.3, 0.3, 0.2, 0.2], [(-4, 0), (4, 0), (1e3, 1e3), (-1e3, 1e3)],
                         np.repeat(np.eye(2)[None], 4, 0))
    m = es.fit_em(X, 4, init_params=es.GmmModel(pi, mu, cov), tol=0.0, max_iter=8, seed=2)
    opi, omu, ocov, rep = oracle.fit_em(X, 4, init_params=(pi, mu, cov), tol=0.0, max_iter=8, seed=2)
    assert m.fit_report.collapses == rep["collapses"] == 2
    assert_params(m, opi, omu, ocov)


# -------------------------------------------------- post-update SingularCovariance
def test_singular_covariance_after_m_step(es, oracle):
    """reg disabled; a component that captures exactly two events (N_k = 2 >= 1, no collapse)
    has a rank-1 covariance after the M-step: SingularCovariance (kind Numeric) on both sides."""
    X = np.concatenate([_blobs(4, [(0, 0, 0), (50, 0, 0)], 300, 3), [[0, 100, 0], [0, 100, 1]]])
    pi, mu, cov = _given([0.45, 0.45, 0.1], [(0, 0, 0), (50, 0, 0), (0, 100, 0.5)], np.repeat(np.eye(3)[None], 3, 0))
    with pytest.raises(oracle.OracleError) as eo:
        oracle.fit_em(X, 3, init_params=(pi, mu, cov), tol=0.0, max_iter=3, reg=0.0)
    assert eo.value.name == "SingularCovariance"
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(X, 3, init_params=es.GmmModel(pi, mu, cov), tol=0.0, max_iter=3, reg=0.0)
    assert e.value.name == "SingularCovariance" and e.value.kind == "Numeric"
    # with the default reg the same fit is well posed and matches the oracle
    m = es.fit_em(X, 3, init_params=es.GmmModel(pi, mu, cov), tol=0.0, max_iter=3)
    opi, omu, ocov, _ = oracle.fit_em(X, 3, init_params=(pi, mu, cov), tol=0.0, max_iter=3)
    assert_params(m, opi, omu, ocov)


# ------------------------------------------------------- mixture-density mode
def test_mixture_mode_detect_and_calibrate(es, oracle):
    n, D, K = 300_000, 8, 4
    ds = es.Dataset.generate(21, n, D, K)
    X = ds.read_rows()
    pi, mu, cov, _ = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=10, seed=4)
    m = es.GmmModel(pi, mu, cov)
    d, ld = es.calibrate_threshold(m, ds, 0.02, mode="mixture", n_train=n // 2, return_log=True)
    od, old = oracle.calibrate(X[: n // 2], pi, mu, cov, 0.02, mode=1)
    assert abs(ld - old) <= 1e-9 * max(1.0, abs(old))
    r = es.detect(m, ds, log_delta=old, mode="mixture")
    of, obk, obl, on = oracle.detect(X, pi, mu, cov, old, mode=1)
    ll = oracle.score(X, pi, mu, cov)["ll"]
    mism = np.nonzero(r.flags != of)[0]
    assert np.all(np.abs(ll[mism] - old) < BAND), "mixture-mode flag mismatches away from the threshold"
    assert np.array_equal(of.astype(bool), ll < old)  # the oracle's mixture mode is ll < log delta
    assert np.array_equal(r.anomaly_indices, np.nonzero(r.flags)[0])
    # the component-mode report fields are still the unweighted best component
    assert np.max(np.abs(r.log_density - obl) / np.maximum(1, np.abs(obl))) <= LL_TOL
    # calibration guarantee in mixture mode: at most ceil(q n_train) training events flagged
    assert r.flags[: n // 2].sum() <= int(np.ceil(0.02 * (n // 2)))
    # the mode switch changes the decision (mixture density >= best-component density)
    rc = es.detect(m, ds, log_delta=old, mode="component")
    assert not np.array_equal(rc.flags, r.flags)


# ------------------------------------------------------------ select_k_bic
def test_select_k_bic_spec_examples_full_covariance(es, oracle):
    rng = np.random.default_rng(1)
    blob = rng.normal(0, 1, size=(600, 2))
    best, bic = es.select_k_bic(blob, [1, 2, 3], init="kmeans++", seed=3)
    ob, obic = oracle.select_k_bic(blob, [1, 2, 3], init="kmeans++", seed=3)
    assert best == ob == 1
    assert np.allclose(bic, obic, rtol=LL_TOL, atol=0)
    two = np.concatenate([rng.normal(-10, 1, size=(300, 2)), rng.normal(10, 1, size=(300, 2))])
    best, bic = es.select_k_bic(two, [1, 2, 3], init="kmeans++", seed=3)
    ob, obic = oracle.select_k_bic(two, [1, 2, 3], init="kmeans++", seed=3)
    assert best == ob == 2
    assert np.allclose(bic, obic, rtol=LL_TOL, atol=0)
    best, bic = es.select_k_bic(two, [1], seed=3)
    assert best == 1 and len(bic) == 1


def test_select_k_bic_full_covariance_large(es, oracle):
    """BIC values through the mixed tcgen05 fit (>= 2^14 events per component) against the
    oracle's: -2 logL + p ln N with p = K-1 + K d + K d(d+1)/2."""
    n, D = 1 << 20, 16
    ds = es.Dataset.generate(42, n, D, 8)
    X = ds.read_rows()
    kr = [4, 8]
    best, bic = es.select_k_bic(ds, kr, init="random", tol=0.0, max_iter=6, seed=7)
    ob, obic = oracle.select_k_bic(X, kr, init="random", tol=0.0, max_iter=6, seed=7)
    assert best == ob
    assert np.all(np.abs(bic - obic) <= 2 * LL_TOL * np.abs(obic))


def test_select_k_bic_skips_failed_k(es):
    X = _blobs(5, [(-3, 0), (3, 0)], 20, 2)
    best, bic = es.select_k_bic(X, [2, 100], init="random", seed=1)  # K = 100 > N = 40: TooFewPoints, skipped
    assert best == 2 and np.isfinite(bic[0]) and np.isnan(bic[1])
    with pytest.raises(es.EventscopeError) as e:
        es.select_k_bic(X, [100], init="random", seed=1)
    assert e.value.name == "TooFewPoints"


# ------------------------------------------------------ acceptance #1 / #2 on the device
@pytest.mark.parametrize("d", [1, 2, 3])
def test_acceptance1_em_monotone_on_device(es, oracle, d):
    """>= 20 seeded fits over >= 3 datasets per d; every per-iteration logL
    sequence nondecreasing within 1e-8, and equal to the oracle's within 1e-6."""
    fits = 0
    for dsi in range(3):
        rng = np.random.default_rng(100 * d + dsi)
        X = np.concatenate([rng.normal(c, 1.0, size=(200, d)) for c in (-3, 0, 4)])
        for seed in range(4):
            for init in ("random", "kmeans++"):
                m = es.fit_em(X, 3, init=init, seed=seed, max_iter=60)
                t = m.fit_report.per_iteration_log_likelihoods
                assert np.all(np.diff(t) >= -1e-8), t
                assert abs(m.weights.sum() - 1) < 1e-12
                assert np.allclose(m.covariances, np.transpose(m.covariances, (0, 2, 1)), atol=1e-12)
                _, _, _, rep = oracle.fit_em(X, 3, init=init, seed=seed, max_iter=60)
                to = rep["per_iteration_log_likelihoods"]
                assert len(t) == len(to) and np.all(np.abs(t - to) <= LL_TOL * np.abs(to))
                fits += 1
    assert fits >= 20


def test_acceptance2_parameter_recovery_on_device(es):
    rng = np.random.default_rng(2026)
    X = np.concatenate([rng.normal(-5, 1, 1000), rng.normal(5, 1, 1000)])[:, None]
    m = es.fit_em(X, 2, seed=7)
    order = np.argsort(m.means[:, 0])
    assert np.all(np.abs(m.means[order, 0] - [-5, 5]) < 0.2)
    assert np.all(np.abs(m.weights[order] - 0.5) < 0.05)


def test_dataset_outlives_context(es):
    """A dataset destroyed after its context frees its own planes (no use-after-free); reading it
    in between fails with ContextDestroyed."""
    import ctypes as C
    lib = es.load_library()
    h = C.c_void_p()
    assert lib.es_ctx_create(0, C.byref(h)) == 0
    d = C.c_void_p()
    assert lib.es_dataset_generate(h, C.c_uint64(1), C.c_int64(10_000), 4, 2, C.byref(d)) == 0
    assert lib.es_ctx_destroy(h) == 0
    out = np.empty((10, 4))
    assert lib.es_dataset_read_rows(d, C.c_int64(0), C.c_int64(10), C.c_void_p(out.ctypes.data)) != 0
    assert lib.es_last_error_name().decode() == "ContextDestroyed"
    assert lib.es_dataset_destroy(d) == 0
    # the Python layer closes a context's datasets first
    ctx = es.Context(0)
    ds = es.Dataset.generate(1, 10_000, 4, 2, ctx=ctx)
    ctx.close()
    assert ds.handle is None
