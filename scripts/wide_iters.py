"""Per-iteration k_em_wide pass times at the c5 shape (D = K = 32): python scripts/wide_iters.py N."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.getcwd())
import paper_2506_02007_b200 as es
import torch
ctx = es.Context(0)
n = int(sys.argv[1])
ds = es.Dataset.generate(13, n, 32, 32, ctx=ctx)
em = es.EM(ds, 32, init="random", tol=0.0, max_iter=40, seed=2)
ctx._lib.es_ctx_set_timing(ctx.handle, 1)
for i in range(8):
    ms0, n0 = C.c_double(), C.c_int64(); ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms0), C.byref(n0))
    t0 = time.perf_counter(); em.step(1); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ms, nn = C.c_double(), C.c_int64(); ctx._lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(nn))
    print(f"n={n} it {i}: {em.last_kernel} pass {ms.value - ms0.value:.2f} ms step {dt*1e3:.2f} ms", flush=True)
