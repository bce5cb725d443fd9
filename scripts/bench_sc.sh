# scorer kernel time at the bench size, three repeats
for r in 1 2 3; do
  timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bs.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bs.log').read().strip().splitlines()[-1]);s=d['score'];print(round(s['events_per_s']/1e9,2), round(s['roofline']['avg_launch_ms'],3), s['n_flagged'])" || tail -5 gpurun_out/bs.log
done
