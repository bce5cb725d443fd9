"""Device tests of host-runtime behaviour that must not change results: the speculative EM
loop (iteration t + 1 enqueued before t's record is read) and the derived-model cache of the
scoring entry points."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_FIT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2506_02007_b200 as es
ds = es.Dataset.generate(42, 1 << 26, 16, 8)
m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=12, seed=7)
np.save(sys.argv[1], np.concatenate([m.weights.ravel(), m.means.ravel(), m.covariances.ravel(),
                                     m.fit_report.per_iteration_log_likelihoods]))
"""


def test_speculative_loop_is_bitwise_neutral(tmp_path):
    """The same fit with ES_EM_SPEC=0 (status read before the next iteration is enqueued) and
    the default speculative loop: bit-identical parameters and per-iteration logL.  The bench
    trajectory (N = 2^26) switches record precision between iterations, so the rule that does
    not speculate near a path threshold is on the path."""
    outs = []
    for spec in ("0", "1"):
        out = str(tmp_path / f"fit{spec}.npy")
        env = dict(os.environ, ES_EM_SPEC=spec)
        r = subprocess.run([sys.executable, "-c", _FIT.format(root=ROOT), out], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


def test_model_cache_tracks_parameter_changes(es):
    """detect / score on a model, on a different model, on the first one mutated in place, and
    on it restored: each result is that of the parameters passed (the cache keys on contents)."""
    ds = es.Dataset.generate(42, 1 << 18, 16, 8)
    m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=6, seed=7)
    d, ld = es.calibrate_threshold(m, ds, 0.05, n_train=1 << 17, return_log=True)
    r1 = es.detect(m, ds, log_delta=ld)
    ll1 = np.empty(ds.n_local)
    es.score(m, ds, ll=ll1)
    m2 = es.GmmModel(m.weights.copy(), m.means + 0.25, m.covariances.copy())
    r2 = es.detect(m2, ds, log_delta=ld)
    assert not np.array_equal(r1.anomaly_indices, r2.anomaly_indices)
    saved = m.covariances.copy()
    m.covariances *= 1.5  # in place: same arrays, new contents
    ll3 = np.empty(ds.n_local)
    es.score(m, ds, ll=ll3)
    assert np.max(np.abs(ll3 - ll1)) > 1e-3
    m.covariances[...] = saved
    ll4 = np.empty(ds.n_local)
    es.score(m, ds, ll=ll4)
    r4 = es.detect(m, ds, log_delta=ld)
    assert np.array_equal(ll4, ll1) and np.array_equal(r4.anomaly_indices, r1.anomaly_indices)


def test_bench_two_ranks_functional():
    """`bench.py --gpus 2` without a launcher re-runs itself as two ranks (torch.distributed.run on
    127.0.0.1); on a one-GPU box both ranks share it through the host exchange (a functional
    check of the multi-rank bench path, not a scaling number).  Rank 0 prints one JSON line."""
    import json
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup",
                          "3", "--rows", str(1 << 20), "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["N"] == 1 << 20 and "exchange" in d["config"]
