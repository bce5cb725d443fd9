"""Parity diagnostics (test infrastructure, not collected): fit the same SYN-v1
data with the CUDA path and the CPU oracle and print the error metrics the
parity tests bound, as margins (error / tolerance; < 1 passes).

    python tests/parity_report.py [n D K iters]...   (defaults: the c1 shape and a c2-like shape)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_02007_b200 as es  # noqa: E402
from oracle import oracle  # noqa: E402


def margins(model, pi, mu, cov, per_g, per_o, tol=1e-5, ll_tol=1e-6):
    w = np.max(np.abs(model.weights - pi) / (tol * np.maximum(np.abs(pi), 1e-3)))
    m = c = 0.0
    for k in range(len(pi)):
        sm = np.abs(mu[k]).max()
        m = max(m, np.max(np.abs(model.means[k] - mu[k]) / (tol * np.maximum(np.abs(mu[k]), sm))))
        sc = np.abs(cov[k]).max()
        c = max(c, np.max(np.abs(model.covariances[k] - cov[k]) / (tol * np.maximum(np.abs(cov[k]), sc))))
    ll = np.abs(np.asarray(per_g) - np.asarray(per_o)) / (ll_tol * np.abs(per_o))
    return w, m, c, ll


def run(n, D, K, iters, seed=42):
    ds = es.Dataset.generate(seed, n, D, min(K, 8))
    X = ds.read_rows()
    model = es.fit_em(ds, K, init="random", tol=0.0, max_iter=iters, seed=7)
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=7)
    w, m, c, ll = margins(model, pi, mu, cov, model.fit_report.per_iteration_log_likelihoods,
                          rep["per_iteration_log_likelihoods"])
    print(f"n={n} D={D} K={K} iters={iters} kernel={os.environ.get('ES_EM_KERNEL', 'default')}: "
          f"margins weights {w:.3f} means {m:.3f} cov {c:.3f} | per-iter logL max {ll.max():.3f} "
          f"(iter {int(ll.argmax())}), last {ll[-1]:.3f}", flush=True)


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]]
    cfgs = [tuple(a[i:i + 4]) for i in range(0, len(a), 4)] or [(1 << 20, 8, 4, 100), (1 << 17, 16, 8, 12),
                                                                 (1 << 20, 16, 8, 30)]
    for cfg in cfgs:
        run(*cfg)
