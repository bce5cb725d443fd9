"""eval-bench: confusion / metrics / kmeans_baseline / sensitivity_sweep.

CPU tests pin the oracle and the host metrics to the SPEC examples; GPU tests compare the
device k-means baseline and confusion counts with the oracle through the C-ABI."""
import numpy as np
import pytest


def blobs(n, D, K, seed=5, spread=12.0, outliers=0):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-spread, spread, size=(K, D))
    lab = rng.integers(0, K, size=n)
    X = centres[lab] + rng.normal(size=(n, D))
    y = np.zeros(n, np.uint8)
    if outliers:
        idx = rng.choice(n, outliers, replace=False)
        X[idx] += rng.normal(scale=8.0, size=(outliers, D))
        y[idx] = 1
    return X, y


# ------------------------------------------------------------------ CPU: oracle + host logic
def test_confusion_examples_oracle(oracle):
    assert oracle.confusion([1, 1, 0, 0], [1, 0, 1, 0]) == (1, 1, 1, 1)
    lab = np.array([0, 1, 1, 0, 1], np.uint8)
    tp, fp, tn, fn = oracle.confusion(lab, lab)
    assert fp == 0 and fn == 0 and tp + tn == 5
    assert oracle.confusion(np.zeros(7, np.uint8), np.ones(7, np.uint8)) == (0, 7, 0, 0)
    with pytest.raises(oracle.OracleError):
        oracle.confusion([1, 0], [1])


def test_metrics_examples():
    # host arithmetic of the product API (no GPU involved)
    from paper_2506_02007_b200 import ConfusionMatrix, EventscopeError, metrics
    m = metrics(ConfusionMatrix(tp=80, fp=10, tn=90, fn=20))
    assert m.accuracy == pytest.approx(0.85) and m.recall == pytest.approx(0.80)
    assert m.precision == pytest.approx(8 / 9) and m.f1 == pytest.approx(0.8421052631578947)
    m = metrics(ConfusionMatrix(tp=0, fp=0, tn=5, fn=3))
    assert m.precision == 0.0 and m.f1 == 0.0
    m = metrics(ConfusionMatrix(tp=4, fp=0, tn=6, fn=0))
    assert (m.accuracy, m.precision, m.recall, m.f1) == (1.0, 1.0, 1.0, 1.0)
    with pytest.raises(EventscopeError):
        metrics(ConfusionMatrix(0, 0, 0, 0))


def test_kmeans_examples_oracle(oracle):
    # duplicated rows, K = 1: all scores 0, no flags for any q < 1
    X = np.tile(np.array([[1.5, -2.0, 0.25]]), (64, 1))
    for q in (0.01, 0.5, 0.99):
        cen, thr, fl, sc, nf, it = oracle.kmeans_baseline(X, 1, q=q, seed=3)
        assert nf == 0 and np.all(sc == 0.0) and thr == 0.0
        assert np.array_equal(cen[0], X[0])
    # a tight cluster plus a point 100 sigma away, K = 1, q = 0.01 -> the outlier is flagged
    rng = np.random.default_rng(1)
    X = rng.normal(scale=0.01, size=(400, 2))
    X[300] = [1.0, 1.0]
    cen, thr, fl, sc, nf, it = oracle.kmeans_baseline(X, 1, q=0.01, seed=0)
    assert fl[300] == 1 and sc[300] > 20 * thr
    with pytest.raises(oracle.OracleError):
        oracle.kmeans_baseline(X[:3], 4, q=0.01)  # TooFewPoints


def test_kmeans_oracle_recovers_blobs(oracle):
    X, y = blobs(3000, 3, 4, outliers=60)
    cen, thr, fl, sc, nf, it = oracle.kmeans_baseline(X, 4, q=0.02, seed=11)
    assert it >= 2
    tp, fp, tn, fn = oracle.confusion(y, fl)
    assert tp / (tp + fn) > 0.8


# ------------------------------------------------------------------ GPU: device vs oracle
@pytest.mark.gpu
@pytest.mark.parametrize("n,D,K", [(20000, 4, 3), (50001, 16, 8), (4096, 33, 5)])
def test_kmeans_parity(es, oracle, n, D, K):
    X, _ = blobs(n, D, K, seed=n, outliers=n // 50)
    r = es.kmeans_baseline(X, K, q=0.02, seed=9)
    cen, thr, fl, sc, nf, it = oracle.kmeans_baseline(X, K, q=0.02, seed=9)
    assert r.iterations == it
    np.testing.assert_allclose(r.centroids, cen, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(r.scores, sc, rtol=1e-10, atol=1e-12)
    assert abs(r.threshold - thr) <= 1e-10 * max(1.0, abs(thr))
    near = np.abs(sc - thr) <= 1e-9 * max(1.0, thr)
    assert np.array_equal(r.flags[~near], fl[~near])
    assert abs(r.n_flagged - nf) <= int(near.sum())


@pytest.mark.gpu
def test_kmeans_examples_device(es):
    X = np.tile(np.array([[1.5, -2.0, 0.25]]), (64, 1))
    r = es.kmeans_baseline(X, 1, q=0.5, seed=3)
    assert r.n_flagged == 0 and np.all(r.scores == 0.0)
    rng = np.random.default_rng(1)
    X = rng.normal(scale=0.01, size=(400, 2))
    X[300] = [1.0, 1.0]
    r = es.kmeans_baseline(X, 1, q=0.01, seed=0)
    assert r.flags[300] == 1
    with pytest.raises(es.EventscopeError) as e:
        es.kmeans_baseline(X[:3], 4, q=0.01)
    assert e.value.name == "TooFewPoints"


@pytest.mark.gpu
def test_confusion_device(es, oracle):
    import torch
    rng = np.random.default_rng(4)
    for n in (0, 1, 1000, 1 << 20):
        lab = rng.integers(0, 2, n).astype(np.uint8)
        fl = rng.integers(0, 2, n).astype(np.uint8)
        want = oracle.confusion(lab, fl)
        cm = es.confusion(lab, fl)
        assert (cm.tp, cm.fp, cm.tn, cm.fn) == want
        if n:
            cm = es.confusion(torch.from_numpy(lab).cuda(), torch.from_numpy(fl).cuda())
            assert (cm.tp, cm.fp, cm.tn, cm.fn) == want
    with pytest.raises(es.EventscopeError):
        es.confusion(np.zeros(3, np.uint8), np.zeros(4, np.uint8))


@pytest.mark.gpu
def test_sensitivity_sweep(es, tmp_path):
    X, y = blobs(6000, 3, 3, seed=2, outliers=120)
    # singleton sweep == one direct run_pipeline cell
    rows = es.sensitivity_sweep(X, y, [3], [0.02], seeds=[0], csv_path=str(tmp_path / "grid.csv"))
    r = es.run_pipeline(X, 3, quantile_q=0.02, seed=0)
    m = es.metrics(es.confusion(y, r.report.flags))
    assert len(rows) == 1 and rows[0]["status"] == "ok" and rows[0]["seed_count"] == 1
    assert rows[0]["f1"] == pytest.approx(m.f1, abs=1e-12) and rows[0]["recall"] == pytest.approx(m.recall, abs=1e-12)
    assert (tmp_path / "grid.csv").read_text().splitlines()[0] == "layer,K,q,seed_count,accuracy,precision,recall,f1,status"
    # full grid; a failing cell (K too large for the train split) is recorded, not raised
    rows = es.sensitivity_sweep(X[:40], y[:40], [2, 3000], [1e-3, 1e-2], seeds=[0, 1])
    assert [(c["K"], c["q"]) for c in rows] == [(2, 1e-3), (2, 1e-2), (3000, 1e-3), (3000, 1e-2)]
    assert rows[0]["status"] == "ok" and rows[2]["status"] != "ok" and rows[2]["seed_count"] == 0


@pytest.mark.gpu
def test_empty_inputs(es):
    """Empty event matrices: scoring / detect are no-ops, fits and calibration raise the
    SPEC's data errors."""
    X0 = np.empty((0, 4))
    rng = np.random.default_rng(0)
    m = es.GmmModel(np.array([0.5, 0.5]), rng.normal(size=(2, 4)), np.tile(np.eye(4), (2, 1, 1)))
    assert es.score(m, X0, ll=np.empty(0)) == 0.0
    r = es.detect(m, X0, log_delta=-5.0)
    assert r.n_flagged == 0 and len(r.flags) == 0
    with pytest.raises(es.EventscopeError):
        es.fit_em(X0, 2)
    with pytest.raises(es.EventscopeError):
        es.calibrate_threshold(m, X0, 0.01, n_train=0)
    with pytest.raises(es.EventscopeError):
        es.kmeans_baseline(X0, 2)
    with pytest.raises(es.EventscopeError):
        es.run_pipeline(X0, 2)


def test_lloyd_oracle_matches_sklearn(oracle):
    """The oracle's Lloyd loop (nearest centroid, ties -> lowest k, stop when no assignment
    changes) against scikit-learn's KMeans(algorithm="lloyd", tol=0) from the same start."""
    from sklearn.cluster import KMeans
    X, _ = blobs(4000, 5, 6, seed=21, spread=4.0)
    rng = np.random.default_rng(3)
    init = X[rng.choice(len(X), 6, replace=False)]
    cen, it = oracle.lloyd(X, init, max_iter=300)
    km = KMeans(n_clusters=6, init=init, n_init=1, max_iter=300, tol=0.0, algorithm="lloyd").fit(X)
    np.testing.assert_allclose(cen, km.cluster_centers_, rtol=1e-12, atol=1e-12)
