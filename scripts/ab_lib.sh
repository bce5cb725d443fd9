# A/B of the in-tree library against paper_2506_02007_b200/lib/variant (ES_LIB_OVERRIDE):
# bench.py EM / scoring kernel times, alternating twice.
for r in 1 2; do
  for v in cur old; do
    if [ $v = old ]; then export ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/variant/libeventscope_b200.so; else unset ES_LIB_OVERRIDE; fi
    timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), round(d['roofline']['avg_launch_ms'],3), round(d['score']['roofline']['avg_launch_ms'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$v.log
  done
done
