# k_em_mma at the bench size, three repeats (value, kernel ms, roofline fraction)
for r in 1 2 3; do
  timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bw.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bw.log').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/bw.log
done
