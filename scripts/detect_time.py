"""detect() wall time per call vs the scoring kernel (bench model, N = 2^26): the overhead a
detect call adds around k_score_mma (model upload, compaction, count read)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
n = 1 << 26
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=6, seed=7)
d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)
flags = torch.empty(n, dtype=torch.uint8, device="cuda")
bk = torch.empty(n, dtype=torch.int32, device="cuda")
bl = torch.empty(n, dtype=torch.float64, device="cuda")
idx = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(3):
    r = es.detect(m, ds, log_delta=ld, flags=flags, best_k=bk, best_logdens=bl, indices=idx)
ctx._lib.es_ctx_set_timing(ctx.handle, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    r = es.detect(m, ds, log_delta=ld, flags=flags, best_k=bk, best_logdens=bl, indices=idx)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 20 * 1e3
ms, nn = C.c_double(), C.c_int64()
ctx._lib.es_ctx_kernel_time(ctx.handle, 1, C.byref(ms), C.byref(nn))
k = ms.value / nn.value
fl = flags.cpu().numpy()
ix = idx[: r.n_flagged].cpu().numpy()
assert np.array_equal(ix, np.flatnonzero(fl)), "indices != flatnonzero(flags)"
print(f"detect: {wall:.3f} ms per call, k_score_mma {k:.3f} ms ({wall / k - 1:.1%} over); n_flagged {r.n_flagged}; "
      f"indices == flatnonzero(flags)", flush=True)
