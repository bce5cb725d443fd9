"""Scorer timing + quick parity (diagnostic): c2 model (25 EM iterations), then detect
passes over N = 2^26 timed with CUDA events (kernel time from the library's own events),
and score parity against the oracle on the first 2^22 events.

    python scripts/score_ab.py [steps]
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_02007_b200 as es  # noqa: E402
from oracle import oracle  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
N, D, K = 1 << 26, 16, 8
ctx = es.Context(0)
lib = ctx._lib
ds = es.Dataset.generate(42, N, D, K, ctx=ctx)
em = es.EM(ds, K, init="random", tol=0.0, max_iter=25, seed=7)
em.step(25)
model = em.finish()
em.close()
d, ld = es.calibrate_threshold(model, ds, 0.01, n_train=N // 2, return_log=True)
flags = torch.empty(N, dtype=torch.uint8, device="cuda")
bk = torch.empty(N, dtype=torch.int32, device="cuda")
bl = torch.empty(N, dtype=torch.float64, device="cuda")
idx = torch.empty(N, dtype=torch.int64, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    es.detect(model, ds, log_delta=ld, flags=flags, best_k=bk, best_logdens=bl, indices=idx)
torch.cuda.synchronize()
cnt = getattr(lib, "es_debug_score_pairs", None)
if cnt is not None:
    cnt.restype = C.c_ulonglong
    cnt()
    es.detect(model, ds, log_delta=ld, flags=flags, best_k=bk, best_logdens=bl, indices=idx)
    print(f"refined pairs per event: {cnt() / N:.3f}")
lib.es_ctx_set_timing(ctx.handle, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
t0 = time.perf_counter()
for _ in range(steps):
    r = es.detect(model, ds, log_delta=ld, flags=flags, best_k=bk, best_logdens=bl, indices=idx)
e1.record(stream)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / steps * 1e3
ms, n = C.c_double(), C.c_int64()
lib.es_ctx_kernel_time(ctx.handle, 1, C.byref(ms), C.byref(n))
lib.es_ctx_set_timing(ctx.handle, 0)
kern = ms.value / max(n.value, 1)
ev_ms = e0.elapsed_time(e1) / steps
byt = N * (D * 8 + 13)
print(f"detect: stream {ev_ms:.3f} ms/pass, host wall {wall:.3f} ms, kernel {kern:.3f} ms "
      f"({byt / kern / 1e6:.0f} GB/s = {byt / kern / 1e6 / 6547.2:.3f} of 6547), flagged {r.n_flagged}")
# parity on a prefix
M = 1 << 22
X = ds.read_rows(0, M)
ll = np.empty(N)
pr = np.empty(N, np.int32)
bkk = np.empty(N, np.int32)
bll = np.empty(N)
es.score(model, ds, ll=ll, predict=pr, best_k=bkk, best_logdens=bll)
o = oracle.score(X, model.weights, model.means, model.covariances)
e = np.abs(ll[:M] - o["ll"]) / np.maximum(1, np.abs(o["ll"]))
eb = np.abs(bll[:M] - o["best_logdens"]) / np.maximum(1, np.abs(o["best_logdens"]))
print(f"parity on 2^22: ll margin {e.max() / 1e-6:.4f}, best_ld margin {eb.max() / 1e-6:.5f}, "
      f"predict mism {int((pr[:M] != o['predict']).sum())}, best_k mism {int((bkk[:M] != o['best_k']).sum())}")
fl = flags.cpu().numpy()
of, _, obl, _ = oracle.detect(X, model.weights, model.means, model.covariances, ld)
print(f"flags mism on 2^22: {int((fl[:M] != of).sum())}")
