"""Where the e2e call's time goes: H2D dataset creation, EM begin (stats + init), EM
steps, finish — at the bench size (N = 2^26, D = 16, K = 8)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

n, D, K = 1 << 26, 16, 8
ctx = es.Context(0)
ds = es.Dataset.generate(42, n, D, K, ctx=ctx)
hostX = torch.empty((n, D), dtype=torch.float64, pin_memory=True)
ds.read_rows(out=hostX)
ds.close()
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    ds2 = es.Dataset.from_array(hostX.numpy(), ctx=ctx)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    em = es.EM(ds2, K, init="random", tol=0.0, max_iter=20, seed=7)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    em.step(20)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    m = em.finish()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    em.close()
    ds2.close()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"create {d[0]:.1f} ms ({n * D * 8 / d[0] / 1e6:.1f} GB/s)  begin {d[1]:.1f}  20 steps {d[2]:.1f}  "
          f"finish {d[3]:.1f}  close {d[4]:.1f}  total {sum(d[:4]):.1f} ms -> {20 / sum(d[:4]) * 1e3:.1f} it/s")
x = torch.empty((n, D), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
x.copy_(hostX, non_blocking=True); torch.cuda.synchronize()
print(f"plain pinned H2D {n * D * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
