"""Per-iteration fixed cost of the EM loop (diagnostic): step time - EM pass time over 20
timed iterations after 5 warm-up ones, at the bench config and at a small N where the fixed
cost dominates; prints a digest of the fitted parameters (bitwise A/B across loop modes)."""
import ctypes as C
import hashlib
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
for n, D, K in ((1 << 26, 16, 8), (1 << 20, 16, 8), (1 << 22, 8, 4)):
    ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
    em = es.EM(ds, K, init="random", tol=0.0, max_iter=40, seed=7)
    em.step(5)
    torch.cuda.synchronize()
    ctx._lib.es_ctx_set_timing(ctx.handle, 1)
    ms0, n0 = C.c_double(), C.c_int64()
    ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms0), C.byref(n0))
    t0 = time.perf_counter()
    em.step(20)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    ms, nn = C.c_double(), C.c_int64()
    ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(nn))
    ctx._lib.es_ctx_set_timing(ctx.handle, 0)
    kp = (ms.value - ms0.value) / max(nn.value - n0.value, 1)
    m = em.finish()
    em.close()
    ds.close()
    h = hashlib.sha1(np.concatenate([m.weights.ravel(), m.means.ravel(), m.covariances.ravel()]).tobytes()).hexdigest()[:12]
    print(f"spec={os.environ.get('ES_EM_SPEC', '1')} N={n} D={D} K={K}: pass {kp * 1e3:.1f} us, step {dt * 1e6:.1f} us, "
          f"fixed {dt * 1e6 - kp * 1e3:.1f} us, params {h}", flush=True)
