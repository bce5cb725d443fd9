"""Small fits and scoring on every pass kernel (diagnostics, run under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
os.environ["ES_EM_DIAG_TC"] = "2"  # the diagonal tensor-core pass at a small N
for (n, D, K, cov) in ((1 << 20, 16, 8, "full"), (1 << 19, 24, 12, "full"), (1 << 20, 16, 4, "diag")):
    ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=3, seed=7, covariance_type=cov)
    kern = []
    for _ in range(3):
        em.step(1)
        kern.append(em.last_kernel.split(" ")[0])
    m = em.finish()
    em.close()
    if cov == "full" and D <= 16 and K <= 8:
        d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)
        r = es.detect(m, ds, log_delta=ld)
        kern.append(f"detect {r.n_flagged}")
    ds.close()
    print(n, D, K, cov, kern, flush=True)
