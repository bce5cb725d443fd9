# ncu capture of k_em_wide (c5 shape D = K = 32, N = 2^24, forced) + per-iteration timing at 2^28
set -x
cat > /tmp/pw.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
os.environ["ES_EM_WIDE"] = "2"
import paper_2506_02007_b200 as es
ctx = es.Context(0)
ds = es.Dataset.generate(13, 1 << 24, 32, 32, ctx=ctx)
em = es.EM(ds, 32, init="random", tol=0.0, max_iter=10, seed=2)
em.step(3)
print(em.last_kernel)
em.close()
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_em_wide -s 1 -c 1 -o gpurun_out/wide python /tmp/pw.py > gpurun_out/pw.log 2>&1
tail -n 3 gpurun_out/pw.log
ncu -i gpurun_out/wide.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/wide_src.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/wide_src.csv 45 > gpurun_out/wide_lines.txt
python scripts/ncu_summary.py gpurun_out/wide.ncu-rep > gpurun_out/wide_summary.txt 2>&1; head -30 gpurun_out/wide_summary.txt
cat > /tmp/t28.py <<'PY'
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
PY
timeout 600 python /tmp/t28.py 268435456 > gpurun_out/t28.log 2>&1; cat gpurun_out/t28.log
