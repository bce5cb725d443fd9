"""Headline-config parity margins (diagnostic): the bench's EM fit (SYN-v1 seed 42,
Random init seed 7, tol 0, `iters` iterations) on the device in both precisions
against the CPU oracle, then score/detect of the fitted model over all N.

    python scripts/headline_parity.py [n] [iters]
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
D, K = 16, 8
oracle.build()
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
X = ds.read_rows()
fits = {}
for prec in ("mixed", "fp64"):
    ctx.set_precision(prec)
    t0 = time.time()
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=iters, seed=7)
    em.step(iters)
    fits[prec] = (em.finish(), em.record_passes)
    em.close()
    print(f"gpu {prec}: {time.time() - t0:.1f} s, record passes {fits[prec][1]}", flush=True)
ctx.set_precision("mixed")
t0 = time.time()
pi, mu, cov, rep = oracle.fit_em(X, K, init="random", tol=0.0, max_iter=iters, seed=7)
print(f"oracle: {time.time() - t0:.1f} s ({os.cpu_count()} threads)", flush=True)
per_o = rep["per_iteration_log_likelihoods"]
for prec, (m, npass) in fits.items():
    w, mm, c, ll = margins(m, pi, mu, cov, m.fit_report.per_iteration_log_likelihoods, per_o)
    fl = abs(m.fit_report.final_log_likelihood - rep["final_log_likelihood"]) / (1e-6 * abs(rep["final_log_likelihood"]))
    print(f"n={n} iters={iters} {prec}: margins weights {w:.3f} means {mm:.3f} cov {c:.3f} | per-iter logL max "
          f"{ll.max():.3f} (iter {int(ll.argmax())}) last {ll[-1]:.3f} | final logL {fl:.3f}", flush=True)
    print("   per-iter logL margins:", " ".join(f"{v:.2f}" for v in ll), flush=True)
# score / detect of the oracle's model over all N
t0 = time.time()
om = es.GmmModel(pi, mu, cov)
ll = np.empty(n)
pr = np.empty(n, np.int32)
bk = np.empty(n, np.int32)
bl = np.empty(n)
es.score(om, ds, ll=ll, predict=pr, best_k=bk, best_logdens=bl)
o = oracle.score(X, pi, mu, cov)
err = np.abs(ll - o["ll"]) / np.maximum(1.0, np.abs(o["ll"]))
errb = np.abs(bl - o["best_logdens"]) / np.maximum(1.0, np.abs(o["best_logdens"]))
print(f"score: ll margin {err.max() / 1e-6:.4f} best_ld margin {errb.max() / 1e-6:.4f} predict mism "
      f"{int((pr != o['predict']).sum())} best_k mism {int((bk != o['best_k']).sum())} ({time.time() - t0:.1f} s)")
d, ld = es.calibrate_threshold(om, ds, 0.01, n_train=n // 2, return_log=True)
od, old = oracle.calibrate(X[: n // 2], pi, mu, cov, 0.01)
r = es.detect(om, ds, log_delta=old)
of, obk, obl, on = oracle.detect(X, pi, mu, cov, old)
mism = np.nonzero(r.flags != of)[0]
band = int(np.sum(np.abs(obl - old) < 1e-9))
print(f"calibrate: log delta gpu {ld!r} oracle {old!r}; detect flag mism {len(mism)} "
      f"(outside band {int(np.sum(np.abs(obl[mism] - old) >= 1e-9))}), band count {band}, flagged {r.n_flagged}/{on}")
