"""ncu driver for the scorer at the bench model: fit 20 EM iterations at N = 2^26 (the bench's
model), then one detect pass (the first k_score_mma launch of the process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
ds = es.Dataset.generate(42, 1 << 26, 16, 8, ctx=ctx)
m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=20, seed=7, ctx=ctx)
r = es.detect(m, ds, log_delta=-40.0, indices=False)
print("flagged", r.n_flagged)
