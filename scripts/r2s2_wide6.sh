set -x
for tau in 0 0.5 1 2; do ES_WIDE_TRUNC=$tau WIDE_VARIANTS=1 timeout 300 python scripts/wide_check.py parity 4194304 4 32 32 > gpurun_out/w6_$tau.log 2>&1; tail -n 1 gpurun_out/w6_$tau.log; done
for tau in 0 1; do ES_WIDE_TRUNC=$tau WIDE_VARIANTS=3 timeout 300 python scripts/wide_check.py parity 4194304 4 16 8 > gpurun_out/w6c_$tau.log 2>&1; tail -n 1 gpurun_out/w6c_$tau.log; done
