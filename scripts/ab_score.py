"""Score-pass A/B + timing: tensor-core scorer vs oracle-exact FP64 team scorer on the same model."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=6, seed=7)
out = {}
for prec in ("mixed", "fp64"):
    ctx.set_precision(prec)
    ll = np.empty(n); pr = np.empty(n, np.int32); bk = np.empty(n, np.int32); bl = np.empty(n)
    es.score(m, ds, ll=ll, predict=pr, best_k=bk, best_logdens=bl)
    out[prec] = (ll, pr, bk, bl)
    ctx._lib.es_ctx_set_timing(ctx.handle, 1)
    for _ in range(3):
        r = es.detect(m, ds, log_delta=-40.0, indices=False)
    ms, cnt = C.c_double(), C.c_int64()
    ctx._lib.es_ctx_kernel_time(ctx.handle, 1, C.byref(ms), C.byref(cnt))
    print(prec, "score kernel ms", ms.value / max(cnt.value, 1), "flagged", r.n_flagged)
a, b = out["mixed"], out["fp64"]
rel = np.abs(a[0] - b[0]) / np.maximum(1, np.abs(b[0]))
print("ll max rel", rel.max(), "best_ld max rel", (np.abs(a[3] - b[3]) / np.maximum(1, np.abs(b[3]))).max())
print("predict mismatches", int((a[1] != b[1]).sum()), "best_k mismatches", int((a[2] != b[2]).sum()))
