"""D = 32, K = 32 (config c5 shape): which public call fails (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

n, D, K = 40000, int(sys.argv[1]) if len(sys.argv) > 1 else 32, int(sys.argv[2]) if len(sys.argv) > 2 else 32
ds = es.Dataset.generate(42, n, D, 8)
X = ds.read_rows()
rng = np.random.default_rng(0)
mu = X[rng.choice(n, K, replace=False)]
cov = np.tile(np.cov(X.T)[None], (K, 1, 1))
m = es.GmmModel(np.full(K, 1.0 / K), mu, cov)
calls = [("score_ll", lambda: es.score(m, ds, ll=np.empty(n))),
         ("score_all", lambda: es.score(m, ds, ll=np.empty(n), predict=np.empty(n, np.int32),
                                        best_k=np.empty(n, np.int32), best_logdens=np.empty(n))),
         ("calibrate", lambda: es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)),
         ("detect", lambda: es.detect(m, ds, log_delta=-40.0)),
         ("resp", lambda: es.responsibilities(m, ds)),
         ("fit", lambda: es.fit_em(ds, K, init="random", tol=0.0, max_iter=2, seed=7))]
for prec in ("mixed", "fp64"):
    es.default_context().set_precision(prec)
    for name, f in calls:
        try:
            f()
            print(prec, name, "ok", flush=True)
        except Exception as e:  # noqa: BLE001
            print(prec, name, "FAIL", e, flush=True)
