import os, sys
sys.path.insert(0, "/root/repo")
import paper_2506_02007_b200 as es
ctx = es.Context(0)
ds = es.Dataset.generate(42, 1 << 26, 16, 16, ctx=ctx)
em = es.EM(ds, 16, init="random", tol=0.0, max_iter=4, seed=7, covariance_type="diag")
em.step(3)
print(em.last_kernel)
