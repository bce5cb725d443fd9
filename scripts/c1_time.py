"""BASELINE c1 (the reference's CPU-runnable case): full covariance K = 4, D = 8, 2^20 events,
100 EM iterations (tol 0, Random init seed 7) + score + flags, on the device (default mixed path)
and on the CPU oracle (all host threads), wall time of the whole fit + detect."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402
from oracle import oracle  # noqa: E402

n, D, K = 1 << 20, 8, 4
oracle.build()
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
X = ds.read_rows()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = es.fit_em(ds, K, init="random", tol=0.0, max_iter=100, seed=7)
    d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)
    r = es.detect(m, ds, log_delta=ld)
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
print(f"c1 device: {tg * 1e3:.1f} ms for 100 EM iterations + calibrate + detect ({100 / tg:.0f} iters/s incl. "
      f"scoring), flagged {r.n_flagged}", flush=True)
t0 = time.perf_counter()
pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=100, seed=7)
to = time.perf_counter() - t0
print(f"c1 oracle (C++ FP64, {os.cpu_count()} threads): {to:.2f} s for the 100-iteration fit alone; "
      f"device / oracle speed-up {to / tg:.0f}x", flush=True)
