set -x
timeout 600 python scripts/iter_overhead.py > gpurun_out/it4.log 2>&1; cat gpurun_out/it4.log
ES_EM_WIDE=2 timeout 300 python scripts/wide_check.py time 67108864 32 32 > gpurun_out/w3_t.log 2>&1; tail -n 3 gpurun_out/w3_t.log
timeout 300 python scripts/wide_check.py time 268435456 32 32 > gpurun_out/w3_t28.log 2>&1; tail -n 3 gpurun_out/w3_t28.log
WIDE_VARIANTS=1,0 timeout 900 python scripts/wide_check.py parity 67108864 3 32 32 > gpurun_out/w3_p26.log 2>&1; tail -n 4 gpurun_out/w3_p26.log
