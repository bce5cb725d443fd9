# k_em_mma at the bench size (value, kernel ms, roofline fraction), converter warpgroup on / off
for cv in 1 0; do
  ES_EM_MMA_CV=$cv timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bw_$cv.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bw_$cv.log').read().strip().splitlines()[-1]);print('cv', $cv, round(d['value'],1), round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/bw_$cv.log
done
