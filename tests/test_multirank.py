"""world_size-2 coverage of the sharded path.

CPU: the gloo exchange callbacks used by es_ctx_create_exchange (rank-ordered
all-gather; sum/min/max in f64 and i64) through real ctypes function pointers.
GPU: two ranks sharing cuda:0 run fit / calibrate / detect / k-means++ on the row
shards of one SYN-v1 matrix and must reproduce the single-rank results.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mp_worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(args, world=2, timeout=600):
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r), WORLD_SIZE=str(world),
                   LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, WORKER, *args], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=timeout)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o


def test_gloo_exchange_callbacks(tmp_path):
    out = str(tmp_path / "ex")
    launch(["exchange", out])
    for r in range(2):
        z = np.load(out + f".{r}.npz")
        assert np.array_equal(z["gather"], np.concatenate([np.arange(5), np.arange(5) + 10]))
        base = np.array([3, -1, 7])
        assert np.array_equal(z["r00"], base * 3) and np.array_equal(z["r10"], base * 3)
        assert np.array_equal(z["r01"], np.minimum(base, base * 2))
        assert np.array_equal(z["r02"], np.maximum(base, base * 2))
        assert z["r10"].dtype == np.int64


@pytest.mark.gpu
def test_two_ranks_match_single_rank(tmp_path):
    import paper_2506_02007_b200 as es
    n = 200_003
    out = str(tmp_path / "fit")
    launch(["fit", out, str(n)])
    z0, z1 = np.load(out + ".0.npz"), np.load(out + ".1.npz")
    # identical model on every rank (rank-ordered reduction)
    for key in ("w", "mu", "cov", "per", "kmu"):
        assert np.array_equal(z0[key], z1[key]), key
    assert z1["off"] == n // 2
    ds = es.Dataset.generate(42, n, 16, 8)
    m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=8, seed=7)
    # mixed precision: FP32 per-lane partials group differently per CTA/rank layout and
    # EM amplifies that along slow directions; the contract tolerance is 1e-5
    assert np.allclose(z0["w"], m.weights, rtol=1e-5, atol=1e-8)
    for k in range(len(m.weights)):  # same floor rule as the oracle parity tests
        assert np.all(np.abs(z0["mu"][k] - m.means[k]) <= 1e-5 * np.maximum(np.abs(m.means[k]),
                                                                         np.abs(m.means[k]).max()))
        assert np.all(np.abs(z0["cov"][k] - m.covariances[k]) <= 1e-5 * np.maximum(np.abs(m.covariances[k]),
                                                                                np.abs(m.covariances[k]).max()))
    assert np.allclose(z0["per"], m.fit_report.per_iteration_log_likelihoods, rtol=1e-7)
    d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)
    assert abs(ld - float(z0["ld"])) <= 1e-6 * abs(ld)
    both = np.concatenate([z0["idx"], z1["idx"]])
    assert int(z0["nflag"]) == int(z1["nflag"]) == len(both)
    # the ranks' own model and threshold on the single-rank context: the same flags, except
    # events within 1e-9 of the threshold (counted from the best-component densities)
    mr = es.GmmModel(z0["w"], z0["mu"], z0["cov"])
    bl = np.empty(n)
    r = es.detect(mr, ds, log_delta=float(z0["ld"]), best_logdens=bl)
    band = np.abs(bl - float(z0["ld"])) <= 1e-9 * max(1.0, abs(float(z0["ld"])))
    diff = np.setxor1d(both, r.anomaly_indices)
    assert np.all(band[diff]), (len(diff), int(band.sum()))
    mk = es.fit_em(ds, 4, init="kmeans++", tol=0.0, max_iter=3, seed=5)
    assert np.allclose(z0["kmu"], mk.means, rtol=1e-5, atol=1e-6)
    # k-means baseline: rank-ordered Lloyd sums -> the same centroids / threshold on both ranks
    kb = es.kmeans_baseline(ds, 4, q=0.02, seed=3)
    for key in ("kbc", "kbt", "kbn", "kbi"):
        assert np.array_equal(z0[key], z1[key]), key
    assert int(z0["kbi"]) == kb.iterations
    np.testing.assert_allclose(z0["kbc"], kb.centroids, rtol=1e-10, atol=1e-12)
    assert abs(float(z0["kbt"]) - kb.threshold) <= 1e-10 * kb.threshold
    both = np.concatenate([z0["kbf"], z1["kbf"]])
    assert np.sum(both != kb.flags) <= 2 and abs(int(z0["kbn"]) - kb.n_flagged) <= 2
    # run_pipeline over the shards (the train split is rank 0's rows)
    pr = es.run_pipeline(ds, 4, quantile_q=0.02, seed=1, max_iter=10)
    for key in ("pmu", "pmean", "pscale", "pdelta", "pn"):
        assert np.array_equal(z0[key], z1[key]), key
    np.testing.assert_allclose(z0["pmean"], pr.mean, rtol=1e-12)
    np.testing.assert_allclose(z0["pmu"], pr.model.means, rtol=1e-5, atol=1e-6)
    pf = np.concatenate([z0["pf"], z1["pf"]])
    assert np.sum(pf != pr.report.flags) <= 1e-4 * n


@pytest.mark.gpu
def test_nccl_exchange_one_rank(monkeypatch):
    """The NCCL exchange path (stat all-gather, histogram all-reduce, k-means++ / Lloyd host
    sums) on a one-rank NCCL communicator reproduces the single-context results bitwise."""
    import ctypes as C

    import paper_2506_02007_b200 as es
    monkeypatch.setenv("ES_FORCE_NCCL", "1")
    lib = es.load_library()
    h = C.c_void_p()
    idb = (C.c_ubyte * 128).from_buffer_copy(es.Context.nccl_unique_id())
    assert lib.es_ctx_create_nccl(0, 0, 1, idb, C.byref(h)) == 0
    nc = es.Context.__new__(es.Context)
    nc._lib, nc._keep, nc.handle, nc.device, nc.rank, nc.world = lib, None, h, 0, 0, 1
    nc.set_precision("mixed")
    ref = es.Context(0)
    out = []
    for ctx in (nc, ref):
        ds = es.Dataset.generate(42, 100_003, 16, 8, ctx=ctx)
        m = es.fit_em(ds, 8, init="kmeans++", tol=0.0, max_iter=4, seed=3, ctx=ctx)
        d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=50_000, return_log=True)
        kb = es.kmeans_baseline(ds, 4, q=0.02, seed=1)
        out.append((m.means, m.covariances, m.fit_report.per_iteration_log_likelihoods, ld, kb.centroids,
                    kb.threshold))
        ds.close()
    for a, b in zip(*out):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    # the exchanges really went through NCCL (stat all-gathers, histogram / row all-reduces)
    assert nc.collective_count > 4 and ref.collective_count == 0
