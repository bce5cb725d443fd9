"""Pipeline timeline of k_em_mma CTA 0, first 128 tiles of the last pass.
Run: bash scripts/em_trace_build.sh; ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/trace/libeventscope_b200.so
python scripts/em_trace.py [N]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
ctx = es.Context()
ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=5, seed=7)
em.step(3)
tr = np.zeros((12, 128), dtype=np.int64)
assert ctx._lib.es_debug_em_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
names = ["tma", "E_iss", "G_iss", "edone", "efree", "conv", "fl_beg", "fl_end", "mready", "E_end", "G_end"]
t0 = tr[0, 0]
rel = (tr[:11] - t0).astype(np.int64)
print("tile " + " ".join(f"{x:>7s}" for x in names))
for j in range(0, 48):
    print(f"{j:4d} " + " ".join(f"{rel[e, j]:7d}" for e in range(11)))
for e, nm in enumerate(names):
    d = np.diff(tr[e, 16:112])
    print(f"{nm:7s} median period {np.median(d):7.0f}")
# per-tile latencies (steady state)
js = np.arange(16, 100)
def lat(a, b, da=0):
    return np.median(tr[b, js] - tr[a, js + da])
print("E_iss -> edone      ", lat(1, 3))
print("edone -> efree      ", lat(3, 4))
print("efree(j) -> E_iss(j+1)", np.median(tr[1, js + 1] - tr[4, js]))
print("mready -> G_iss     ", lat(8, 2))
print("G_iss(j) -> fl_end(j)", np.median(tr[7, js] - tr[2, js]))
print("edone(j) -> mready(j)", lat(3, 8))
print("conv(j) -> E_iss(j) ", lat(5, 1))
print("tma(j) -> conv(j)   ", lat(0, 5))
print("E issue duration    ", lat(1, 9))
print("G issue duration    ", lat(2, 10))
