# scoring refinement rule A/B at the bench size (ES_SCORE_REFINE=all: responsibility > 1e-6)
for r in bound all; do
  ES_SCORE_REFINE=$r timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bs_$r.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bs_$r.log').read().strip().splitlines()[-1]);s=d['score'];print('$r', round(s['events_per_s']/1e9,2), round(s['roofline']['avg_launch_ms'],3), round(s['roofline']['frac'],3), s['n_flagged'])" || tail -5 gpurun_out/bs_$r.log
done
