# session-3 check: loop fixed cost, the wide parity case, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ES_EM_SPEC=0 timeout 600 python scripts/iter_overhead.py > gpurun_out/r3_it0.log 2>&1; cat gpurun_out/r3_it0.log
ES_EM_SPEC=1 timeout 600 python scripts/iter_overhead.py > gpurun_out/r3_it1.log 2>&1; cat gpurun_out/r3_it1.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wide_pass" > gpurun_out/r3_wide.log 2>&1; tail -5 gpurun_out/r3_wide.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3_bench.log 2> gpurun_out/r3_bench.err; tail -c 2500 gpurun_out/r3_bench.log
for c in "4194304 32 32" "67108864 32 32"; do timeout 600 python scripts/wide_check.py time $c > gpurun_out/r3_wt.log 2>&1; tail -2 gpurun_out/r3_wt.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_finalize|k_em_mma|k_reduce" -c 40 --csv --log-file gpurun_out/r3_launch.csv python scripts/iter_overhead.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/r3_launch.csv 2>/dev/null | head -20
