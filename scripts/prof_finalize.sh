# ncu source-level capture of k_finalize at the bench shape (N=2^20 fit, D=16, K=8)
set -x
cat > /tmp/fin.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2506_02007_b200 as es
ctx = es.Context(0)
ds = es.Dataset.generate(42, 1 << 20, 16, 8, ctx=ctx)
em = es.EM(ds, 8, init="random", tol=0.0, max_iter=10, seed=7)
em.step(8)
em.finish(); em.close()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_finalize -s 4 -c 1 -o gpurun_out/fin python /tmp/fin.py > gpurun_out/fin.log 2>&1
ncu -i gpurun_out/fin.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/fin_src.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/fin_src.csv 40 > gpurun_out/fin_lines.txt
cat gpurun_out/fin_lines.txt
ncu -i gpurun_out/fin.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[-1]
for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:
  print(k, v[h.index(k)] if k in h else '?')
"
