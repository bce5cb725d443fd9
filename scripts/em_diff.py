"""One EM iteration with the default (mixed) kernel vs the strict FP64 kernel on the same data:
per-component weight / mean / covariance errors in units of the parity tolerance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
it = int(sys.argv[4]) if len(sys.argv) > 4 else 1
res = {}
for prec in ("mixed", "fp64"):
    ctx = es.Context(0, precision=prec)
    ds = es.Dataset.generate(42, n, D, min(K, 8), ctx=ctx)
    m = es.fit_em(ds, K, init="random", tol=0.0, max_iter=it, seed=7)
    res[prec] = (m.weights, m.means, m.covariances)
w, mu, cov = res["mixed"]
w0, mu0, cov0 = res["fp64"]
for k in range(K):
    sm = np.abs(mu0[k]).max()
    sc = np.abs(cov0[k]).max()
    em = np.abs(mu[k] - mu0[k]) / (1e-5 * np.maximum(np.abs(mu0[k]), sm))
    ec = np.abs(cov[k] - cov0[k]) / (1e-5 * np.maximum(np.abs(cov0[k]), sc))
    ia = np.unravel_index(ec.argmax(), ec.shape)
    print(f"k={k} N_k={w0[k] * n:10.0f} w_err {abs(w[k] - w0[k]) / (1e-5 * max(w0[k], 1e-3)):.3f} "
          f"mean_err {em.max():.3f} (a={em.argmax()}) cov_err {ec.max():.3f} at {ia} "
          f"sigma_diag [{np.sqrt(np.diag(cov0[k])).min():.3f},{np.sqrt(np.diag(cov0[k])).max():.3f}] "
          f"dcov_diag_rel {np.max(np.abs(np.diag(cov[k]) - np.diag(cov0[k])) / np.diag(cov0[k])):.2e}")
