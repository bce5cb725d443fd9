"""ncu driver: the k_em_full_mixed pass at the c5 shape (D = K = 32), N = 2^24."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
ds = es.Dataset.generate(42, 1 << 24, 32, 32, ctx=ctx)
em = es.EM(ds, 32, init="random", tol=0.0, max_iter=4, seed=7)
em.step(3)
print(em.last_kernel)
