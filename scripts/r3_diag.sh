set -x
timeout 600 python scripts/diag_check.py parity 8388608 16 4 8 1,0 > gpurun_out/r3_dp1.log 2>&1; tail -4 gpurun_out/r3_dp1.log
timeout 600 python scripts/diag_check.py parity 16777216 16 8 6 2 > gpurun_out/r3_dp2.log 2>&1; tail -3 gpurun_out/r3_dp2.log
timeout 600 python scripts/diag_check.py time 268435456 16 16 > gpurun_out/r3_dt.log 2>&1; tail -3 gpurun_out/r3_dt.log
