"""k_em_wide (D, K <= 32 full covariance on tcgen05) diagnostics: parity margins against the
CPU oracle and against the FP32 k_em_full_mixed pass, and the EM pass time.

    ES_EM_WIDE=2 python scripts/wide_check.py parity [n] [iters] [D] [K]
    python scripts/wide_check.py time [n] [D] [K]        (ES_EM_WIDE=0 times k_em_full_mixed)
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2506_02007_b200 as es  # noqa: E402

mode = sys.argv[1]
ctx = es.Context(0)
if mode == "parity":
    from oracle import oracle
    from parity_report import margins
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    D = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    K = int(sys.argv[5]) if len(sys.argv) > 5 else 32
    oracle.build()
    ds = es.Dataset.generate(13, n, D, K, ctx=ctx)
    X = ds.read_rows()
    t0 = time.time()
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=2)
    print(f"oracle: {time.time() - t0:.1f} s; min N_k {n * pi.min():.0f}", flush=True)
    for var in (os.environ.get("WIDE_VARIANTS") or "2,0").split(","):
        os.environ["ES_EM_WIDE"] = var
        em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=2)
        kern = []
        for _ in range(iters):
            em.step(1)
            kern.append(em.last_kernel.split(" ")[0])
        m = em.finish()
        em.close()
        w, mm, c, ll = margins(m, pi, mu, cov, m.fit_report.per_iteration_log_likelihoods,
                               rep["per_iteration_log_likelihoods"])
        print(f"ES_EM_WIDE={var} n={n} D={D} K={K} iters={iters} {kern}: margins weights {w:.3f} means {mm:.3f} "
              f"cov {c:.3f} | per-iter logL {' '.join(f'{v:.3f}' for v in ll)}", flush=True)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 26
    D = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    K = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    ds = es.Dataset.generate(13, n, D, K, ctx=ctx)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=40, seed=2)
    em.step(3)
    ctx._lib.es_ctx_set_timing(ctx.handle, 1)
    t0 = time.perf_counter()
    em.step(3)
    dt = (time.perf_counter() - t0) / 3
    ms, nn = C.c_double(), C.c_int64()
    ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(nn))
    print(f"time n={n} D={D} K={K} [{em.last_kernel}]: pass {ms.value / max(nn.value, 1):.2f} ms, "
          f"step {dt * 1e3:.2f} ms", flush=True)
    em.close()
