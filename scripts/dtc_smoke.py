"""k_em_diag_tc smoke run (diagnostics, e.g. under compute-sanitizer): a small forced diagonal fit."""
import os
import sys

os.environ.setdefault("ES_EM_DIAG_TC", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
ds = es.Dataset.generate(3, int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21, 16, 4, ctx=ctx)
em = es.EM(ds, 4, init="random", tol=0.0, max_iter=3, seed=5, covariance_type="diag")
for _ in range(3):
    em.step(1)
    print(em.last_kernel, flush=True)
print(em.finish().weights)
