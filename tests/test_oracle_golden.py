"""Pins the CPU oracle (the parity checker) before it is trusted.

Sources: every closed-form example in SPEC.md gmm-core / anomaly-detect
(SPEC.md:267-269, 277-279, 287-289, 297-299, 307-309, 312-316, 363-365,
373-375, 388-391), the acceptance criteria SPEC.md:543-550, Random123's
Philox4x32-10 known-answer vectors, and the committed scikit-learn fixtures
(tests/golden/make_sklearn_golden.py).  CPU only.
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def one(mu, var):
    return [1.0], [[mu]], [[[var]]]


# ------------------------------------------------------------ densities
def test_component_log_density_examples(oracle):
    # SPEC.md:267-269 (acceptance #4: within 1e-9)
    assert abs(oracle.component_log_density(*one(0.0, 1.0), [0.0], 0) - (-0.9189385332046727)) < 1e-9
    assert abs(oracle.component_log_density([1.0], [[0.0, 0.0]], [np.eye(2)], [0, 0], 0) - (-1.8378770664093453)) < 1e-9
    assert abs(oracle.component_log_density(*one(0.0, 4.0), [2.0], 0) - (-2.112085713764618)) < 1e-9


def test_mixture_density_examples(oracle):
    # SPEC.md:277-279
    pi, mu, cov = one(0.3, 2.0)
    x = [1.1]
    assert math.isclose(math.exp(oracle.mixture_log_density(pi, mu, cov, x)),
                        math.exp(oracle.component_log_density(pi, mu, cov, x, 0)), rel_tol=1e-14)
    same = oracle.mixture_log_density([0.5, 0.5], [[0.3], [0.3]], [[[2.0]], [[2.0]]], x)
    assert math.isclose(same, oracle.mixture_log_density(pi, mu, cov, x), rel_tol=1e-14)
    v = math.exp(oracle.mixture_log_density([0.5, 0.5], [[-1.0], [1.0]], [[[1.0]], [[1.0]]], [0.0]))
    assert abs(v - 0.24197072451914337) < 1e-12


def test_responsibility_examples(oracle):
    # SPEC.md:287-289
    X = np.array([[0.3], [2.0]])
    g = oracle.score(X, *one(0.0, 1.0), gamma=True)["gamma"]
    assert np.all(g == 1.0)
    g = oracle.score(np.array([[0.0]]), [0.5, 0.5], [[-2.0], [2.0]], [[[1.0]], [[1.0]]], gamma=True)["gamma"]
    assert np.allclose(g, 0.5, atol=1e-15)
    g = oracle.score(np.array([[1.0]]), [0.5, 0.5], [[0.0], [4.0]], [[[1.0]], [[1.0]]], gamma=True)["gamma"]
    assert abs(g[0, 0] - 0.9820137900379085) < 1e-12


def test_one_d_mixture_integrates_to_one(oracle):
    # SPEC.md:314, acceptance #4
    rng = np.random.default_rng(5)
    X = np.concatenate([rng.normal(-2, 0.5, 300), rng.normal(3, 1.5, 700)])[:, None]
    pi, mu, cov, _ = oracle.fit_em(X, 2, seed=1, max_iter=50)
    s = np.sqrt(cov.ravel().max())
    grid = np.linspace(mu.min() - 10 * s, mu.max() + 10 * s, 10_000)
    ll = oracle.score(grid[:, None], pi, mu, cov)["ll"]
    assert abs(np.trapezoid(np.exp(ll), grid) - 1.0) < 1e-3


# ------------------------------------------------------------------- EM
def test_fit_k1_closed_form(oracle):
    # SPEC.md:297, acceptance #3: mean, biased covariance + reg I within 1e-9
    rng = np.random.default_rng(3)
    X = rng.normal(size=(500, 3)) @ np.array([[1, 0.2, 0], [0, 1, 0.4], [0, 0, 0.5]]) + 2.0
    pi, mu, cov, rep = oracle.fit_em(X, 1, seed=0)
    reg = rep["reg"]
    assert np.allclose(pi, 1.0)
    assert np.allclose(mu[0], X.mean(0), atol=1e-9)
    assert np.allclose(cov[0], np.cov(X.T, bias=True) + reg * np.eye(3), atol=1e-9)
    assert abs(reg - 1e-6 * np.trace(np.cov(X.T, bias=True)) / 3) < 1e-18


def test_parameter_recovery(oracle):
    # SPEC.md:298, acceptance #2
    rng = np.random.default_rng(2026)
    X = np.concatenate([rng.normal(-5, 1, 1000), rng.normal(5, 1, 1000)])[:, None]
    pi, mu, cov, rep = oracle.fit_em(X, 2, seed=7)
    order = np.argsort(mu[:, 0])
    assert np.all(np.abs(mu[order, 0] - [-5, 5]) < 0.2)
    assert np.all(np.abs(pi[order] - 0.5) < 0.05)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_em_monotone(oracle, d):
    # SPEC.md:299,312; acceptance #1 (>= 20 seeded fits over >= 3 datasets)
    for ds in range(3):
        rng = np.random.default_rng(100 * d + ds)
        X = np.concatenate([rng.normal(c, 1.0, size=(200, d)) for c in (-3, 0, 4)])
        for seed in range(3):
            for init in ("random", "kmeans++"):
                pi, mu, cov, rep = oracle.fit_em(X, 3, init=init, seed=seed, max_iter=60)
                t = rep["per_iteration_log_likelihoods"]
                assert np.all(np.diff(t) >= -1e-8), t
                assert abs(pi.sum() - 1) < 1e-12
                assert np.allclose(cov, np.transpose(cov, (0, 2, 1)), atol=1e-12)


def test_fit_reproducible(oracle):
    # SPEC.md:316
    rng = np.random.default_rng(9)
    X = rng.normal(size=(777, 2))
    a = oracle.fit_em(X, 3, seed=4, max_iter=30, nthreads=1)
    b = oracle.fit_em(X, 3, seed=4, max_iter=30, nthreads=8)
    for u, v in zip(a[:3], b[:3]):
        assert np.array_equal(u, v)
    assert np.array_equal(a[3]["per_iteration_log_likelihoods"], b[3]["per_iteration_log_likelihoods"])


def test_fit_errors(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_em(np.zeros((2, 1)), 3)
    assert e.value.name == "TooFewPoints"
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_em(np.ones((10, 2)), 2)
    assert e.value.name == "DegenerateData"
    X = np.ones((10, 2))
    X[3, 1] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_em(X, 1)
    assert e.value.name == "NonFiniteInput"
    # reg disabled on rank-deficient data -> SingularCovariance
    t = np.linspace(0, 1, 50)
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_em(np.stack([t, 2 * t], 1), 1, reg=0.0)
    assert e.value.name == "SingularCovariance"


# ------------------------------------------------------------------ BIC
def test_select_k_bic(oracle):
    # SPEC.md:307-309
    rng = np.random.default_rng(1)
    blob = rng.normal(0, 1, size=(600, 2))
    assert oracle.select_k_bic(blob, [1, 2, 3], init="kmeans++", seed=3)[0] == 1
    two = np.concatenate([rng.normal(-10, 1, size=(300, 2)), rng.normal(10, 1, size=(300, 2))])
    assert oracle.select_k_bic(two, [1, 2, 3], init="kmeans++", seed=3)[0] == 2
    assert oracle.select_k_bic(two, [1], seed=3)[0] == 1


# --------------------------------------------------------------- detect
def test_detect_examples(oracle):
    # SPEC.md:363-365 (x=3 has density exactly delta: strict '<' keeps it normal)
    pi, mu, cov = one(0.0, 1.0)
    X = np.array([[0.0], [4.0], [3.0]])
    ld3 = oracle.component_log_density(pi, mu, cov, [3.0], 0)
    flags, bk, bl, n = oracle.detect(X, pi, mu, cov, ld3)
    assert list(flags) == [0, 1, 0] and n == 1
    assert abs(math.exp(ld3) - 0.0044318484119380075) < 1e-15
    flags, *_ = oracle.detect(X, pi, mu, cov, bl.min() - 1.0)
    assert flags.sum() == 0
    flags, *_ = oracle.detect(X, pi, mu, cov, math.inf)
    assert flags.sum() == 3


def test_detect_monotone_and_log_linear_equivalence(oracle):
    # SPEC.md:388-389, acceptance #7
    rng = np.random.default_rng(4)
    X = rng.normal(size=(2000, 2))
    pi, mu, cov, _ = oracle.fit_em(X, 2, seed=2, max_iter=30)
    _, _, bl, _ = oracle.detect(X, pi, mu, cov, 0.0)
    prev = None
    for ld in np.linspace(bl.min(), bl.max(), 10):
        flags, *_ = oracle.detect(X, pi, mu, cov, ld)
        lin = (np.exp(bl) < np.exp(ld)).astype(np.uint8)
        assert np.array_equal(flags, (bl < ld).astype(np.uint8))
        assert np.array_equal(flags == 1, lin == 1) or np.all((flags == lin) | (np.abs(bl - ld) < 1e-12))
        if prev is not None:
            assert np.all(flags >= prev)
        prev = flags


def test_calibrate_examples(oracle):
    # SPEC.md:373-375
    rng = np.random.default_rng(8)
    Xt = rng.normal(size=(10_000, 1))
    pi, mu, cov = one(0.0, 1.0)
    d, ld = oracle.calibrate(Xt, pi, mu, cov, 1e-300)
    flags, *_ = oracle.detect(Xt, pi, mu, cov, ld)
    assert flags.sum() == 0
    # N=3 densities {0.1, 0.2, 0.3}, q = 0.5 -> 0.2: points whose N(x|0,1) are those values
    xs = np.sqrt(-2 * np.log(np.array([0.1, 0.2, 0.3]) * np.sqrt(2 * np.pi)))[:, None]
    d, ld = oracle.calibrate(xs, pi, mu, cov, 0.5)
    assert abs(d - 0.2) < 1e-12
    d, ld = oracle.calibrate(Xt, pi, mu, cov, 0.01)
    fresh = rng.normal(size=(10_000, 1))
    frac = oracle.detect(fresh, pi, mu, cov, ld)[0].mean()
    assert 0.004 <= frac <= 0.02
    flags, *_ = oracle.detect(Xt, pi, mu, cov, ld)
    assert flags.sum() <= math.ceil(0.01 * len(Xt))
    with pytest.raises(oracle.OracleError) as e:
        oracle.calibrate(np.zeros((0, 1)), pi, mu, cov, 0.1)
    assert e.value.name == "EmptyTraining"


# ------------------------------------------------------- sklearn fixtures
@pytest.mark.parametrize("name", ["sklearn_d3k3.npz", "sklearn_d8k4.npz", "sklearn_diag_d6k5.npz"])
def test_oracle_matches_sklearn(oracle, name):
    g = np.load(os.path.join(GOLD, name))
    X = g["X"]
    iters = int(g["iters"])
    ct = str(g["covariance_type"]) if "covariance_type" in g else "full"
    pi, mu, cov, rep = oracle.fit_em(X, len(g["w0"]), init_params=(g["w0"], g["mu0"], g["cov0"]), tol=0.0,
                                     max_iter=iters, reg=float(g["reg"]), covariance_type=ct)
    assert np.allclose(pi, g["weights"], rtol=1e-9, atol=1e-12)
    assert np.allclose(mu, g["means"], rtol=1e-9, atol=1e-9)
    assert np.allclose(cov, g["covariances"], rtol=1e-8, atol=1e-10)
    per = rep["per_iteration_log_likelihoods"] / len(X)
    assert np.allclose(per, g["lower_bounds"], rtol=1e-10, atol=1e-10)
    s = oracle.score(X, pi, mu, cov)
    assert np.allclose(s["ll"], g["score"], rtol=1e-9, atol=1e-9)
    assert np.array_equal(s["predict"], g["predict"])


# -------------------------------------------------------------- SYN-v1
def test_philox_known_answers(oracle):
    # Random123 kat_vectors, philox4x32_10
    assert oracle.philox4x32([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox4x32([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert oracle.philox4x32([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_syn_v1_shape_and_ratio(oracle):
    model = oracle.syn_model(42, 8, 4)
    X, comp, anom = oracle.syn_rows(42, 8, 4, model, 0, 60_000)
    assert X.shape == (60_000, 8) and np.isfinite(X).all()
    assert abs(anom.mean() - 1 / 6) < 0.01           # SPEC.md:186 / PAPER.md:209 5:1
    pi_true = model[0]
    assert np.allclose(np.bincount(comp, minlength=4) / len(comp), pi_true, atol=0.01)
    # counter-based: any sub-range regenerates identically
    X2, _, _ = oracle.syn_rows(42, 8, 4, model, 1234, 10)
    assert np.array_equal(X2, X[1234:1244])


def test_em_step_is_one_fit_iteration(oracle):
    # bench.py --impl reference times eso_em_step: one iteration of eso_fit_em exactly
    model = oracle.syn_model(42, 4, 3)
    X, _, _ = oracle.syn_rows(42, 4, 3, model, 0, 20_000)
    pi, mu, cov, reg = oracle.random_init(X, 3, 7)
    p2, m2, c2, rep = oracle.fit_em(X, 3, init_params=(pi, mu, cov), tol=0.0, max_iter=2, reg=reg)
    lls = []
    for _ in range(2):
        ll, nc = oracle.em_step(X, pi, mu, cov, reg)
        lls.append(ll)
        assert nc == 0
    assert np.array_equal(pi, p2) and np.array_equal(mu, m2) and np.array_equal(cov, c2)
    assert lls == list(rep["per_iteration_log_likelihoods"])
