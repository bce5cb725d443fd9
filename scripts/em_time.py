"""EM pass timing (diagnostic A/B): bench config, 5 warm-up + 20 timed iterations, prints the
average k_em_mma launch and the step time from the library's own CUDA events."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
ds = es.Dataset.generate(42, 1 << 26, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=40, seed=7)
em.step(5)
torch.cuda.synchronize()
ctx._lib.es_ctx_set_timing(ctx.handle, 1)
t0 = time.perf_counter()
em.step(20)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 20
ms, n = C.c_double(), C.c_int64()
ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(n))
tag = os.environ.get("ES_LIB_OVERRIDE", "default").split("/")[-2] if os.environ.get("ES_LIB_OVERRIDE") else "default"
print(f"{tag}: pass {ms.value / n.value:.4f} ms, step {dt * 1e3:.4f} ms", flush=True)
