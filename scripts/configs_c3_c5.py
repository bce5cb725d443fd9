"""BASELINE.json configs c3 (diagonal covariance, K = 16, D = 16, 2^28 events) and c5 (full
covariance, K = 32, D = 32) on one B200: EM iterations/s with the data resident in HBM."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402


def run(tag, n, D, K, cov, iters):
    ctx = es.Context(0)
    ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters + 3, seed=7, covariance_type=cov)
    em.step(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    em.step(iters)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / iters
    kern = em.last_kernel
    em.close()
    ds.close()
    ctx.close()
    print(f"{tag}: N={n} D={D} K={K} {cov} [{kern}]: {1 / t:.2f} EM iters/s ({t * 1e3:.1f} ms/iter), "
          f"{n * D * 8 / t / 1e9:.0f} GB/s of the FP64 matrix ({n * D * 8 / t / 6547.2e9 * 100:.1f}% of 6.55 TB/s)",
          flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("c3", "both"):
    run("c3", 1 << 28, 16, 16, "diag", 5)
if which in ("c5", "both"):
    run("c5", 1 << 26, 32, 32, "full", 3)
