"""Small driver for ncu captures: one EM iteration + one detect pass at N (default 2^23)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
em = es.EM(ds, K, init="random", tol=0.0, max_iter=4, seed=7)
em.step(2)
m = em.finish()
r = es.detect(m, ds, log_delta=-40.0)
print("ok", m.fit_report.per_iteration_log_likelihoods, r.n_flagged)
