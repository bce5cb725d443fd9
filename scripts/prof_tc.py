"""ncu driver: EM at N (default 2^23) for `warm` iterations, the profiled launch is the next one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=warm + 3, seed=7)
em.step(warm + 1)
m = em.finish()
r = es.detect(m, ds, log_delta=-40.0)
print("ok", r.n_flagged)
