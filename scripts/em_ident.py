"""Isolation test: K identical components (gamma = 1/K exactly) vs K = 1, one EM iteration,
default kernel vs strict FP64: any K-dependence of the error is in the M-step path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
D = 16
for K in (1, 8):
    res = {}
    for prec in ("mixed", "fp64"):
        ctx = es.Context(0, precision=prec)
        ds = es.Dataset.generate(42, n, D, 8, ctx=ctx)
        X0 = ds.read_rows()[:4096]
        mu0 = X0.mean(0) + 0.3
        cov0 = np.cov(X0.T) * 1.5
        init = es.GmmModel(np.full(K, 1.0 / K), np.tile(mu0, (K, 1)), np.tile(cov0, (K, 1, 1)))
        m = es.fit_em(ds, K, tol=0.0, max_iter=1, init_params=init, ctx=ctx)
        res[prec] = m
    a, b = res["mixed"], res["fp64"]
    for k in (0, K - 1):
        dd = (np.diag(a.covariances[k]) - np.diag(b.covariances[k])) / np.diag(b.covariances[k])
        dm = (a.means[k] - b.means[k]) / np.sqrt(np.diag(b.covariances[k]))
        print(f"K={K} k={k}: cov diag rel err mean {dd.mean():+.2e} max|.| {np.abs(dd).max():.2e}; "
              f"mean err / sigma max {np.abs(dm).max():.2e}")
