"""k_em_diag_tc (diagonal covariances on tcgen05) diagnostics: parity margins against the CPU
oracle (ES_EM_DIAG_TC variants: 1 default, 0 the FP32 SIMT pass, 2 forced below 2^20 events per
component) and the EM pass time at BASELINE c3 (N = 2^28, D = 16, K = 16).

    python scripts/diag_check.py parity n D K iters [variants]
    python scripts/diag_check.py time [n] [D] [K]
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
    n, D, K, iters = (int(v) for v in sys.argv[2:6])
    variants = (sys.argv[6] if len(sys.argv) > 6 else "1,0").split(",")
    oracle.build()
    ds = es.Dataset.generate(3, n, D, K, ctx=ctx)
    X = ds.read_rows()
    t0 = time.time()
    pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
    print(f"oracle: {time.time() - t0:.1f} s; min N_k {n * pi.min():.0f}", flush=True)
    for var in variants:
        os.environ["ES_EM_DIAG_TC"] = var
        em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=5, covariance_type="diag")
        kern = []
        for _ in range(iters):
            em.step(1)
            kern.append(em.last_kernel.split(" ")[0])
        m = em.finish()
        em.close()
        w, mm, c, ll = margins(m, pi, mu, cov, m.fit_report.per_iteration_log_likelihoods,
                               rep["per_iteration_log_likelihoods"])
        fl = abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) / (1e-6 * abs(rep["final_log_likelihood"]))
        print(f"ES_EM_DIAG_TC={var} n={n} D={D} K={K} iters={iters} {kern}: margins weights {w:.3f} means {mm:.3f} "
              f"cov {c:.3f} final logL {fl:.3f} | per-iter logL {' '.join(f'{v:.3f}' for v in ll)}", flush=True)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    D = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    K = int(sys.argv[4]) if len(sys.argv) > 4 else 16
    ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
    for var in (os.environ.get("DIAG_VARIANTS") or "1,0").split(","):
        os.environ["ES_EM_DIAG_TC"] = var
        em = es.EM(ds, K, init="random", tol=0.0, max_iter=40, seed=7, covariance_type="diag")
        em.step(6)
        ctx._lib.es_ctx_set_timing(ctx.handle, 1)
        em.step(2)
        ms0, n0 = C.c_double(), C.c_int64()
        ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms0), C.byref(n0))
        t0 = time.perf_counter()
        em.step(5)
        dt = (time.perf_counter() - t0) / 5
        ms, nn = C.c_double(), C.c_int64()
        ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(nn))
        ctx._lib.es_ctx_set_timing(ctx.handle, 0)
        pm = (ms.value - ms0.value) / max(nn.value - n0.value, 1)
        gbs = n * D * 8 / (pm * 1e-3) / 1e9
        print(f"ES_EM_DIAG_TC={var} n={n} D={D} K={K} [{em.last_kernel}]: pass {pm:.3f} ms ({gbs:.0f} GB/s), "
              f"step {dt * 1e3:.3f} ms", flush=True)
        em.close()
