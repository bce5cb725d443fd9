set -x
WIDE_VARIANTS=1 timeout 300 python scripts/wide_check.py parity 4194304 4 32 32 > gpurun_out/w5_a.log 2>&1; tail -n 2 gpurun_out/w5_a.log
WIDE_VARIANTS=1 timeout 300 python scripts/wide_check.py parity 4194304 4 24 12 > gpurun_out/w5_b.log 2>&1; tail -n 2 gpurun_out/w5_b.log
WIDE_VARIANTS=3 timeout 300 python scripts/wide_check.py parity 4194304 4 16 8 > gpurun_out/w5_c.log 2>&1; tail -n 2 gpurun_out/w5_c.log
ES_EM_MMA_PASSES=1 timeout 300 python scripts/wide_check.py time 67108864 32 32 > gpurun_out/w5_t1.log 2>&1; tail -n 2 gpurun_out/w5_t1.log
WIDE_VARIANTS=1 timeout 900 python scripts/wide_check.py parity 33554432 4 32 32 > gpurun_out/w5_d.log 2>&1; tail -n 2 gpurun_out/w5_d.log
