for np in 1 2; do
  ES_EM_MMA_PASSES=$np timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bq_$np.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bq_$np.log').read().strip().splitlines()[-1]);print('npass', $np, d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
