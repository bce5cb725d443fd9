# A/B of k_em_mma launch options at the bench size: "WG POLICY" pairs
for cfg in "2 0" "3 0"; do
  set -- $cfg
  ES_EM_MMA_WG=$1 ES_EM_MMA_POLICY=$2 timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bw_$1_$2.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bw_$1_$2.log').read().strip().splitlines()[-1]);print('wg', $1, 'policy', $2, round(d['value'],1), round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/bw_$1_$2.log
done
