"""GPU parity: the CUDA path (C-ABI via ctypes) against the CPU oracle.

Tolerances are the north star's (BASELINE.json): per-event log-likelihood
within 1e-6 relative (absolute floor 1e-6 * max(1, |ll|)), fitted
weights/means/covariances within 1e-5 relative (floor: 1e-5 * max|entry| of
the component), labels/flags identical except events within 1e-9 of a tie or
of the threshold, which are counted and must be rare.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LL_TOL = 1e-6
PAR_TOL = 1e-5
BAND = 1e-9


@pytest.fixture(params=["mixed", "fp64"])
def prec(request, es):
    """Both arithmetic modes of the product path."""
    ctx = es.default_context()
    ctx.set_precision(request.param)
    yield request.param
    ctx.set_precision("mixed")


def syn(es, oracle, n, D, K, seed=42):
    ds = es.Dataset.generate(seed, n, D, K)
    return ds, ds.read_rows()


def assert_ll(a, b):
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max() <= LL_TOL, f"max rel ll err {err.max():.3e}"


def assert_params(model, pi, mu, cov):
    assert np.all(np.abs(model.weights - pi) <= PAR_TOL * np.maximum(np.abs(pi), 1e-3))
    for k in range(len(pi)):
        sm = np.abs(mu[k]).max()
        assert np.all(np.abs(model.means[k] - mu[k]) <= PAR_TOL * np.maximum(np.abs(mu[k]), sm)), k
        sc = np.abs(cov[k]).max()
        assert np.all(np.abs(model.covariances[k] - cov[k]) <= PAR_TOL * np.maximum(np.abs(cov[k]), sc)), k


def labels_match(a, b, w):
    """a, b label arrays; w (N,K) log-scores used to find ties within BAND."""
    diff = np.nonzero(a != b)[0]
    if len(diff) == 0:
        return 0
    s = np.sort(w[diff], axis=1)
    gap = s[:, -1] - s[:, -2]
    assert np.all(gap < BAND), f"{len(diff)} label mismatches, not ties"
    return len(diff)


# ----------------------------------------------------------- golden values
def test_golden_densities_through_cabi(es):
    m1 = es.GmmModel(np.array([1.0]), np.array([[0.0]]), np.array([[[1.0]]]))
    assert abs(es.component_log_density(m1, [0.0], 0) - (-0.9189385332046727)) < 1e-9
    m2 = es.GmmModel(np.array([1.0]), np.zeros((1, 2)), np.eye(2)[None])
    assert abs(es.component_log_density(m2, [0.0, 0.0], 0) - (-1.8378770664093453)) < 1e-9
    m3 = es.GmmModel(np.array([1.0]), np.array([[0.0]]), np.array([[[4.0]]]))
    assert abs(es.component_log_density(m3, [2.0], 0) - (-2.112085713764618)) < 1e-9
    mm = es.GmmModel(np.array([0.5, 0.5]), np.array([[-1.0], [1.0]]), np.ones((2, 1, 1)))
    assert abs(es.mixture_density(mm, [0.0]) - 0.24197072451914337) < 1e-12
    g = es.responsibilities(es.GmmModel(np.array([0.5, 0.5]), np.array([[0.0], [4.0]]), np.ones((2, 1, 1))),
                            np.array([[1.0]]))
    assert abs(g[0, 0] - 0.9820137900379085) < 1e-12
    with pytest.raises(es.EventscopeError) as e:
        es.component_log_density(m2, [0.0], 0)
    assert e.value.name == "DimensionMismatch" and e.value.kind == "Data"


def test_detect_examples_through_cabi(es):
    m = es.GmmModel(np.array([1.0]), np.array([[0.0]]), np.array([[[1.0]]]))
    ld3 = es.component_log_density(m, [3.0], 0)
    r = es.detect(m, np.array([[0.0], [4.0], [3.0]]), log_delta=ld3)
    assert list(r.flags) == [0, 1, 0] and list(r.anomaly_indices) == [1] and r.n_flagged == 1
    r = es.detect(m, np.array([[0.0], [4.0], [3.0]]), delta=math.inf)
    assert r.flags.sum() == 3


def test_calibrate_examples_through_cabi(es, oracle):
    m = es.GmmModel(np.array([1.0]), np.array([[0.0]]), np.array([[[1.0]]]))
    xs = np.sqrt(-2 * np.log(np.array([0.1, 0.2, 0.3]) * np.sqrt(2 * np.pi)))[:, None]
    assert abs(es.calibrate_threshold(m, xs, 0.5) - 0.2) < 1e-12
    rng = np.random.default_rng(8)
    Xt = rng.normal(size=(10_000, 1))
    d, ld = es.calibrate_threshold(m, Xt, 0.01, return_log=True)
    od, old = oracle.calibrate(Xt, [1.0], [[0.0]], [[[1.0]]], 0.01)
    assert d == od and ld == old
    assert es.detect(m, Xt, log_delta=ld).flags.sum() <= math.ceil(0.01 * len(Xt))
    d0, ld0 = es.calibrate_threshold(m, Xt, 1e-300, return_log=True)
    assert es.detect(m, Xt, log_delta=ld0).flags.sum() == 0
    with pytest.raises(es.EventscopeError) as e:
        es.calibrate_threshold(m, Xt, 0.1, n_train=0)
    assert e.value.name == "EmptyTraining"


# ------------------------------------------------------ c1-shaped parity
def _fit_both(es, oracle, ds, X, K, iters, init="random", seed=7):
    model = es.fit_em(ds, K, init=init, tol=0.0, max_iter=iters, seed=seed)
    pi, mu, cov, rep = oracle.fit_em(X, K, init=init, tol=0.0, max_iter=iters, seed=seed)
    return model, (pi, mu, cov, rep)


@pytest.mark.parametrize("D,K,n,iters", [(8, 4, 1 << 20, 100), (16, 8, 1 << 17, 12), (3, 5, 100_003, 40),
                                         (20, 3, 30_011, 10), (2, 40, 20_000, 8), (32, 32, 40_000, 5),
                                         (48, 3, 20_000, 4), (64, 2, 10_007, 3)])
def test_fit_score_detect_parity(es, oracle, prec, D, K, n, iters):
    ds, X = syn(es, oracle, n, D, min(K, 8))
    model, (pi, mu, cov, rep) = _fit_both(es, oracle, ds, X, K, iters)
    assert_params(model, pi, mu, cov)
    per_g, per_o = model.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"]
    assert len(per_g) == len(per_o) == iters
    assert np.all(np.abs(per_g - per_o) <= LL_TOL * np.abs(per_o))
    assert abs(model.fit_report.final_log_likelihood - rep["final_log_likelihood"]) <= LL_TOL * abs(
        rep["final_log_likelihood"])
    assert model.fit_report.iterations == rep["iterations"]
    # score on the oracle's parameters (same model both sides)
    om = es.GmmModel(pi, mu, cov)
    ll = np.empty(ds.n_local)
    pr = np.empty(ds.n_local, np.int32)
    bk = np.empty(ds.n_local, np.int32)
    bl = np.empty(ds.n_local)
    tot = es.score(om, ds, ll=ll, predict=pr, best_k=bk, best_logdens=bl)
    o = oracle.score(X, pi, mu, cov, gamma=True)
    assert_ll(ll, o["ll"])
    assert_ll(bl, o["best_logdens"])
    assert abs(tot - o["ll"].sum()) <= 1e-9 * abs(o["ll"].sum())
    w = np.log(np.maximum(o["gamma"], 1e-300))
    labels_match(pr, o["predict"], w)
    lnk = w + o["ll"][:, None] - np.log(pi)[None]  # component log densities (up to rounding)
    labels_match(bk, o["best_k"], lnk)
    # detect at the calibrated threshold
    d, ld = es.calibrate_threshold(om, ds, 0.01, n_train=n // 2, return_log=True)
    od, old = oracle.calibrate(X[: n // 2], pi, mu, cov, 0.01)
    assert abs(ld - old) <= 1e-9 * max(1.0, abs(old))
    r = es.detect(om, ds, log_delta=old)
    of, obk, obl, on = oracle.detect(X, pi, mu, cov, old)
    mism = np.nonzero(r.flags != of)[0]
    assert np.all(np.abs(obl[mism] - old) < BAND), "flag mismatches away from the threshold"
    assert np.array_equal(r.anomaly_indices, np.nonzero(r.flags)[0])
    assert r.n_flagged == r.flags.sum()


def test_responsibilities_rows_sum_to_one(es, oracle, prec):
    ds, X = syn(es, oracle, 50_000, 16, 8)
    pi, mu, cov, _ = oracle.fit_em(X, 8, init="random", tol=0.0, max_iter=5, seed=3)
    g = es.responsibilities(es.GmmModel(pi, mu, cov), ds)
    o = oracle.score(X, pi, mu, cov, gamma=True)["gamma"]
    assert np.abs(g.sum(1) - 1).max() < 1e-9
    assert np.abs(g - o).max() < 1e-6


def test_kmeanspp_init_parity(es, oracle, prec):
    ds, X = syn(es, oracle, 200_000, 8, 4)
    model, (pi, mu, cov, rep) = _fit_both(es, oracle, ds, X, 4, 20, init="kmeans++", seed=11)
    assert_params(model, pi, mu, cov)


def test_k1_closed_form_and_convergence(es, oracle):
    ds, X = syn(es, oracle, 10_007, 5, 3)
    m = es.fit_em(ds, 1, seed=0)
    pi, mu, cov, rep = oracle.fit_em(X, 1, seed=0)
    assert np.allclose(m.means[0], X.mean(0), atol=1e-9)
    assert np.allclose(m.covariances[0], np.cov(X.T, bias=True) + rep["reg"] * np.eye(5), atol=1e-9)
    assert m.fit_report.converged and rep["converged"]
    assert m.fit_report.iterations == rep["iterations"]


def test_converged_fit_parity(es, oracle, prec):
    ds, X = syn(es, oracle, 100_000, 4, 3, seed=5)
    m = es.fit_em(ds, 3, init="kmeans++", seed=2, tol=1e-6, max_iter=200)
    pi, mu, cov, rep = oracle.fit_em(X, 3, init="kmeans++", seed=2, tol=1e-6, max_iter=200)
    assert m.fit_report.converged == rep["converged"]
    assert m.fit_report.iterations == rep["iterations"]
    assert_params(m, pi, mu, cov)
    t = m.fit_report.per_iteration_log_likelihoods
    assert np.all(np.diff(t) >= -1e-8 * np.abs(t[1:]))


def test_errors_through_cabi(es):
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(np.zeros((2, 1)), 3)
    assert e.value.name == "TooFewPoints" and e.value.kind == "Data"
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(np.ones((10, 2)), 2)
    assert e.value.name == "DegenerateData"
    X = np.ones((10, 2))
    X[3, 1] = np.nan
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(X + np.arange(10)[:, None], 1)
    assert e.value.name == "NonFiniteInput"
    t = np.linspace(0, 1, 50)
    with pytest.raises(es.EventscopeError) as e:
        es.fit_em(np.stack([t, 2 * t], 1), 1, reg=0.0)
    assert e.value.name == "SingularCovariance" and e.value.kind == "Numeric"


def test_determinism_bitwise(es, prec):
    ds = es.Dataset.generate(9, 300_000, 16, 8)
    a = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=5, seed=1)
    b = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=5, seed=1)
    assert np.array_equal(a.covariances, b.covariances) and np.array_equal(a.means, b.means)
    assert np.array_equal(a.fit_report.per_iteration_log_likelihoods, b.fit_report.per_iteration_log_likelihoods)


def test_layouts_and_generator(es, oracle):
    rng = np.random.default_rng(0)
    X = rng.normal(size=(1001, 7))
    for arr in (X, np.asfortranarray(X), X[:, ::1].copy()):
        ds = es.Dataset.from_array(arr)
        assert np.array_equal(ds.read_rows(), X)
    # device generator vs host restatement of SYN-v1 (same Philox counters; libm ulps)
    ds = es.Dataset.generate(42, 4096, 8, 4)
    model = oracle.syn_model(42, 8, 4)
    Xo, _, _ = oracle.syn_rows(42, 8, 4, model, 0, 4096)
    assert np.abs(ds.read_rows() - Xo).max() < 1e-12 * max(1.0, np.abs(Xo).max())


# ------------------------------------------------- diagonal covariance (a11)
@pytest.mark.parametrize("D,K,n,iters", [(16, 16, 1 << 18, 15), (5, 3, 50_001, 30), (24, 8, 40_000, 8)])
def test_diag_fit_parity(es, oracle, D, K, n, iters):
    ds, X = syn(es, oracle, n, D, min(K, 8), seed=3)
    m = es.fit_em(ds, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    assert_params(m, pi, mu, cov)
    off = m.covariances - np.array([np.diag(np.diag(c)) for c in m.covariances])
    assert np.all(off == 0.0)
    assert np.allclose(m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"],
                       rtol=LL_TOL)
    best, bic = es.select_k_bic(ds, [K], init="random", max_iter=3, seed=5, covariance_type="diag")
    assert best == K and np.isfinite(bic[0])


# ------------------------------------------- full-size fused-kernel parity
def test_full_size_one_pass_records_vs_fp64(es):
    """At N = 2^25 every component has >= 2^20 events, so the fused tcgen05 pass
    uses its single-fp16-record precision.  The strict FP64
    kernel (itself pinned to the oracle above) is the reference at this size: the
    oracle would need minutes per iteration here."""
    n, D, K, iters = 1 << 25, 16, 8, 6
    fits = {}
    for prec in ("mixed", "fp64"):
        ctx = es.Context(0, precision=prec)
        ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
        em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=7)
        em.step(iters)
        passes = em.record_passes
        fits[prec] = (em.finish(), passes)
        em.close()
        ds.close()
    (m, passes), (r, _) = fits["mixed"], fits["fp64"]
    assert passes == 1
    assert_params(m, r.weights, r.means, r.covariances)
    per_m, per_r = m.fit_report.per_iteration_log_likelihoods, r.fit_report.per_iteration_log_likelihoods
    assert np.all(np.abs(per_m - per_r) <= LL_TOL * np.abs(per_r))


def test_two_pass_records_small_components(es, oracle):
    """Below 2^20 events per component the fused pass switches to hi + lo records."""
    ds, X = syn(es, oracle, 1 << 20, 16, 8)
    em = es.EM(ds, 8, init="random", tol=0.0, max_iter=6, seed=7)
    em.step(6)
    assert em.record_passes == 2
    m = em.finish()
    em.close()
    pi, mu, cov, rep = oracle.fit_em(X, 8, init="random", tol=0.0, max_iter=6, seed=7)
    assert_params(m, pi, mu, cov)


def test_small_components_use_strict_passes(es, oracle):
    """With fewer than 2^14 events in some component the iteration runs on the strict FP64
    kernel (the tensor-core whitening's per-event rounding would not average out)."""
    ds, X = syn(es, oracle, 1000, 16, 8)
    em = es.EM(ds, 8, init="random", tol=0.0, max_iter=10, seed=7)
    em.step(10)
    assert em.record_passes == 0
    m = em.finish()
    em.close()
    pi, mu, cov, rep = oracle.fit_em(X, 8, init="random", tol=0.0, max_iter=10, seed=7)
    assert_params(m, pi, mu, cov)
    assert np.all(np.abs(m.fit_report.per_iteration_log_likelihoods - rep["per_iteration_log_likelihoods"])
                  <= LL_TOL * np.abs(rep["per_iteration_log_likelihoods"]))


# ------------------------------------------------ run_pipeline
def test_run_pipeline_parity(es, oracle):
    """run_pipeline on the device vs the oracle composition: train split =
    first half of the (time-ordered) rows, z-scored with its mean and population std; fit;
    q-quantile threshold on the train split; detect over all rows."""
    n, D, K = 200_000, 8, 4
    ds, X = syn(es, oracle, n, D, K, seed=11)
    r = es.run_pipeline(ds, K, train_window=0.5, quantile_q=0.01, init="random", tol=0.0, max_iter=25, seed=3)
    n_train = n // 2
    m, s = X[:n_train].mean(0), X[:n_train].std(0)
    assert r.n_train == n_train
    assert np.allclose(r.mean, m, rtol=1e-12, atol=1e-12) and np.allclose(r.scale, s, rtol=1e-12)
    Z = (X - m) / s
    pi, mu, cov, rep = oracle.fit_em(Z[:n_train], K, init="random", tol=0.0, max_iter=25, seed=3)
    assert_params(r.model, pi, mu, cov)
    # threshold and flags on the pipeline's own model (identical model on both sides)
    od, old = oracle.calibrate(Z[:n_train], r.model.weights, r.model.means, r.model.covariances, 0.01)
    assert abs(r.report.log_delta - old) <= 1e-9 * max(1.0, abs(old))
    of, obk, obl, on = oracle.detect(Z, r.model.weights, r.model.means, r.model.covariances, r.report.log_delta)
    mism = np.nonzero(r.report.flags != of)[0]
    assert np.all(np.abs(obl[mism] - r.report.log_delta) < BAND)
    assert np.array_equal(r.report.anomaly_indices, np.nonzero(r.report.flags)[0])
    assert_ll(r.report.log_density, obl)
    # the calibration guarantee on the training split
    assert r.report.flags[:n_train].sum() <= math.ceil(0.01 * n_train)


def test_run_pipeline_errors_and_fixed_delta(es, oracle):
    ds, X = syn(es, oracle, 60, 2, 2, seed=5)
    with pytest.raises(es.EventscopeError) as e:
        es.run_pipeline(ds, 4, train_window=0.5)  # 30 training rows < 10 K
    assert e.value.name == "InsufficientTraining" and e.value.kind == "Data"
    # fixed delta, no standardization: detect runs on the raw features with that delta
    ds2, X2 = syn(es, oracle, 50_000, 3, 2, seed=6)
    r = es.run_pipeline(ds2, 2, train_window=0.4, quantile_q=None, delta=1e-3, standardize=False, init="random",
                        tol=0.0, max_iter=10, seed=1)
    assert np.all(r.mean == 0) and np.all(r.scale == 1) and abs(r.report.delta - 1e-3) < 1e-18
    of, _, obl, _ = oracle.detect(X2, r.model.weights, r.model.means, r.model.covariances, np.log(1e-3))
    mism = np.nonzero(r.report.flags != of)[0]
    assert np.all(np.abs(obl[mism] - np.log(1e-3)) < BAND)


@pytest.mark.parametrize("n", [1 << 16, 1 << 24])
def test_em_monotone_on_device(es, prec, n):
    """SPEC.md:299,312 (acceptance #1): the logL trajectory is nondecreasing within 1e-8
    (relative), through the default mixed path and the strict FP64 path, small and large N."""
    ctx = es.Context(0, precision=prec)
    ds = es.Dataset.generate(11, n, 16, 8, ctx=ctx)
    m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=12, seed=3, ctx=ctx)
    per = m.fit_report.per_iteration_log_likelihoods
    assert np.all(np.diff(per) >= -1e-8 * np.abs(per[1:])), np.diff(per)


def test_detect_properties_full_size(es):
    """At 2^24 events (size-independent properties): anomaly sets are nested in delta
    (acceptance #7) and the calibrated threshold flags the q-quantile of the
    train split: #{train: log p < log delta} = floor(h) + 1 or so."""
    n, q = 1 << 24, 0.01
    ds = es.Dataset.generate(5, n, 16, 8)
    m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=5, seed=1)
    d, ld = es.calibrate_threshold(m, ds, q, n_train=n // 2, return_log=True)
    r = es.detect(m, ds, log_delta=ld, indices=False)
    bl = r.log_density
    ntr = int(np.sum(bl[: n // 2] < ld))
    h = (n // 2 - 1) * q
    assert int(np.floor(h)) <= ntr <= int(np.floor(h)) + 1
    prev = None
    for lds in np.linspace(ld - 5.0, ld + 5.0, 10):
        f = es.detect(m, ds, log_delta=float(lds), indices=False).flags.astype(bool)
        assert np.array_equal(f, bl < lds)
        if prev is not None:
            assert np.all(f[prev])  # A(delta_i) subset of A(delta_i+1)
        prev = f


@pytest.mark.parametrize("mode,kernel,n,D,K", [("1", "k_em_diag_tc", 1 << 23, 16, 4),
                                               ("0", "k_em_diag_mixed", 1 << 23, 16, 4),
                                               ("1", "k_em_diag_tc", (1 << 24) + 77, 16, 4),
                                               ("1", "k_em_diag_tc", 1 << 24, 10, 5)])
def test_diag_mixed_pass_parity(es, oracle, mode, kernel, n, D, K, monkeypatch):
    """Diagonal covariances, every component >= 2^20 events: the default tcgen05 pass
    (k_em_diag_tc, E-step quadratic form and M-step moments on the tensor cores) and the FP32
    SIMT pass (k_em_diag_mixed, ES_EM_DIAG_TC=0) against the oracle (c3's kernels at a
    parity-testable size; 2^24 + 77 events: a ragged last tile and every component >= 2^20
    events from the first iteration on; D = 10, K = 5: padded features and components)."""
    monkeypatch.setenv("ES_EM_DIAG_TC", mode)
    iters = 8
    ds, X = syn(es, oracle, n, D, K, seed=3)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    em.step(iters)
    assert em.last_kernel == kernel
    m = em.finish()
    em.close()
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    assert_params(m, pi, mu, cov)
    assert np.all(m.covariances[:, ~np.eye(D, dtype=bool)] == 0.0)
    per_g, per_o = m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"]
    assert np.all(np.abs(per_g - per_o) <= LL_TOL * np.abs(per_o))
    assert abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) <= LL_TOL * abs(
        rep["final_log_likelihood"])


def test_diag_tc_c3_shape_parity(es, oracle, monkeypatch):
    """k_em_diag_tc at c3's K = D = 16 against the oracle.  At a parity-testable N the smallest
    SYN-v1 component (weight 1/136) holds fewer than the 2^20 events the default path requires,
    so the pass is forced (ES_EM_DIAG_TC=2): a harder case than the default regime."""
    monkeypatch.setenv("ES_EM_DIAG_TC", "2")
    n, D, K, iters = 1 << 24, 16, 16, 6
    ds, X = syn(es, oracle, n, D, K, seed=3)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    kern = []
    for _ in range(iters):
        em.step(1)
        kern.append(em.last_kernel)
    m = em.finish()
    em.close()
    assert kern.count("k_em_diag_tc") >= iters - 1, kern
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    assert_params(m, pi, mu, cov)
    per_g, per_o = m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"]
    assert np.all(np.abs(per_g - per_o) <= LL_TOL * np.abs(per_o))


@pytest.mark.parametrize("n,D,K,iters", [(1 << 24, 32, 32, 4), (1 << 22, 24, 12, 6)])
def test_full_mixed_pass_parity(es, oracle, n, D, K, iters, monkeypatch):
    """Full covariances beyond k_em_mma's shapes (the c5 shape D = K = 32 and an odd one), every
    component >= 2^14 events, with the wide tensor-core pass switched off (ES_EM_WIDE=0): the
    FP32 k_em_full_mixed pass against the oracle."""
    monkeypatch.setenv("ES_EM_WIDE", "0")
    ds, X = syn(es, oracle, n, D, K, seed=13)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=2)
    em.step(iters)
    assert em.last_kernel == "k_em_full_mixed"
    m = em.finish()
    em.close()
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=2)
    assert_params(m, pi, mu, cov)
    per_g, per_o = m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"]
    assert np.all(np.abs(per_g - per_o) <= LL_TOL * np.abs(per_o))
    assert abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) <= LL_TOL * abs(
        rep["final_log_likelihood"])


@pytest.mark.parametrize("n,D,K,iters", [(1 << 24, 32, 32, 3), (1 << 22, 24, 12, 4), (1 << 24, 32, 4, 4),
                                         ((1 << 22) + 45, 20, 6, 3)])
def test_wide_pass_parity(es, oracle, n, D, K, iters):
    """The default full-covariance pass beyond k_em_mma's shapes (D, K <= 32; BASELINE c5 is
    D = K = 32): k_em_wide, E-step whitening and M-step Gram on tcgen05, against the oracle.
    hi + lo records in the first iteration and while some component holds < 2^20 events; the
    D = 32, K = 4 case reaches one-fp16 records (SYN-v1 weights are (k + 1) / 10, so the
    smallest component holds ~1.7e6 > 2^20 events at N = 2^24).  2^22 + 45 events: a ragged
    last tile (and an early trajectory that amplified the pass's Gram bias before the lo
    products were issued first: weights margin 1.006 -> 0.33)."""
    ds, X = syn(es, oracle, n, D, K, seed=13)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=2)
    kern = []
    for _ in range(iters):
        em.step(1)
        kern.append(em.last_kernel)
    m = em.finish()
    em.close()
    assert kern[0] == "k_em_wide<2>", kern
    if K == 32:  # c5's shape at 2^24 events: the wide pass except after the Random init's first
        # M-step (one component left with ~3k < 2^14 events takes the strict kernel)
        assert sum(k.startswith("k_em_wide") for k in kern) >= iters - 1, kern
    if K == 4:
        assert "k_em_wide<1>" in kern, kern
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=2)
    assert_params(m, pi, mu, cov)
    per_g, per_o = m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"]
    assert np.all(np.abs(per_g - per_o) <= LL_TOL * np.abs(per_o))
    assert abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) <= LL_TOL * abs(
        rep["final_log_likelihood"])
