"""A/B: tcgen05 EM pass vs SIMT FP32 EM pass vs FP64 on the same data (one process per kernel choice)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
prec = sys.argv[4] if len(sys.argv) > 4 else "mixed"
ctx = es.Context(0, precision=prec)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
m = es.fit_em(ds, K, init="random", tol=0.0, max_iter=5, seed=7)
np.savez(f"gpurun_out/ab_{os.environ.get('ES_EM_KERNEL', 'ws')}_{prec}.npz", w=m.weights, mu=m.means,
         cov=m.covariances, per=m.fit_report.per_iteration_log_likelihoods)
print(os.environ.get("ES_EM_KERNEL", "ws"), prec, m.fit_report.per_iteration_log_likelihoods)
