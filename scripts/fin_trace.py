"""k_finalize phase timeline (diagnostic; needs the -DES_FIN_TRACE variant library via
ES_LIB_OVERRIDE, scripts/variant_build.sh es_kernels.cu -DES_FIN_TRACE): per CTA the
%globaltimer of start / reduction done / ticket won / statistics summed / M-step operands /
Cholesky done / end, in us relative to the earliest start, after EM iterations at the bench shape."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

ctx = es.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=40, seed=7)
for it in range(6):
    em.step(1)
    buf = (C.c_ulonglong * (256 * 8))()
    ctx._lib.es_debug_fin_trace(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 8).astype(np.float64)
    used = a[:, 0] > 0
    t0 = a[used, 0].min()
    rel = np.where(a > 0, (a - t0) / 1e3, np.nan)[used]
    print(f"iteration {it}: CTAs {used.sum()}, start spread {np.nanmax(rel[:, 0]):.2f} us, reduction done "
          f"max {np.nanmax(rel[:, 1]):.2f} us; last CTAs: " + "; ".join(
              " ".join(f"{v:.2f}" for v in r[2:7]) for r in rel if not np.isnan(r[2])), flush=True)
    ctx._lib.es_ctx_set_timing(ctx.handle, 0)
