"""Per-iteration EM-kernel time over a fit (N default 2^26)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
prec = sys.argv[3] if len(sys.argv) > 3 else "mixed"
ctx = es.Context(0, precision=prec)
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=iters + 1, seed=7)
lib = ctx._lib
out = []
for it in range(iters):
    lib.es_ctx_set_timing(ctx.handle, 1)
    em.step(1)
    ms, cnt = C.c_double(), C.c_int64()
    lib.es_ctx_kernel_time(ctx.handle, 0, C.byref(ms), C.byref(cnt))
    out.append(ms.value)
m = em.finish()
print(os.environ.get("ES_EM_KERNEL", "ws"), prec, " ".join(f"{v:.2f}" for v in out))
print("weights", m.weights)
