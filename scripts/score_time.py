"""Scoring-pass timing (diagnostic A/B): detect over the bench data with a fixed 10-iteration
model, 10 timed passes, the library's own CUDA events for the kernel."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

N = 1 << 26
ctx = es.Context(0)
ds = es.Dataset.generate(42, N, 16, 8, ctx=ctx)
m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=10, seed=7, ctx=ctx)
fl = torch.empty(N, dtype=torch.uint8, device="cuda")
bk = torch.empty(N, dtype=torch.int32, device="cuda")
bl = torch.empty(N, dtype=torch.float64, device="cuda")
idx = torch.empty(N, dtype=torch.int64, device="cuda")
for _ in range(2):
    es.detect(m, ds, log_delta=-40.0, flags=fl, best_k=bk, best_logdens=bl, indices=idx)
ctx._lib.es_ctx_set_timing(ctx.handle, 1)
for _ in range(10):
    es.detect(m, ds, log_delta=-40.0, flags=fl, best_k=bk, best_logdens=bl, indices=idx)
ms, n = C.c_double(), C.c_int64()
ctx._lib.es_ctx_kernel_time(ctx.handle, 1, C.byref(ms), C.byref(n))
tag = os.environ.get("ES_LIB_OVERRIDE", "x/default/x").split("/")[-2]
print(f"{tag}: score kernel {ms.value / n.value:.4f} ms", flush=True)
