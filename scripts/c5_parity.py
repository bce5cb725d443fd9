"""BASELINE c5 parity at the config itself: full covariance, N = 2^28, D = 32, K = 32, SYN-v1
seed 42, Random init seed 7, tol 0, `iters` iterations on the default path (k_em_wide: hi + lo records
while some component holds < 2^20 events, one fp16 record after) against the CPU oracle on the
same 68.7 GB matrix (host RAM: X + the oracle's N x K responsibilities, ~140 GB).

    python scripts/c5_parity.py [iters]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2506_02007_b200 as es  # noqa: E402
from oracle import oracle  # noqa: E402
from parity_report import margins  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n, D, K = 1 << 28, 32, 32
oracle.build()
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
t0 = time.time()
em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=7)
kern = []
for _ in range(iters):
    em.step(1)
    kern.append(em.last_kernel.split(" ")[0])
m = em.finish()
em.close()
print(f"gpu: {time.time() - t0:.1f} s, kernels {kern}", flush=True)
X = ds.read_rows()
ds.close()
t0 = time.time()
pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=7)
print(f"oracle: {time.time() - t0:.1f} s (16 threads); min N_k {n * pi.min():.0f}", flush=True)
w, mm, c, ll = margins(m, pi, mu, cov, m.fit_report.per_iteration_log_likelihoods, rep["per_iteration_log_likelihoods"])
fl = abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) / (1e-6 * abs(rep["final_log_likelihood"]))
print(f"c5 n={n} D={D} K={K} iters={iters}: margins weights {w:.3f} means {mm:.3f} cov {c:.3f} final logL {fl:.3f} | "
      f"per-iter logL {' '.join(f'{v:.3f}' for v in ll)}", flush=True)
