set -x
timeout 600 python scripts/iter_overhead.py > gpurun_out/it3.log 2>&1; cat gpurun_out/it3.log
WIDE_VARIANTS=2,0 timeout 300 python scripts/wide_check.py parity 4194304 1 32 32 > gpurun_out/w2_a.log 2>&1; tail -n 3 gpurun_out/w2_a.log
WIDE_VARIANTS=3,1 timeout 300 python scripts/wide_check.py parity 4194304 1 16 8 > gpurun_out/w2_b.log 2>&1; tail -n 3 gpurun_out/w2_b.log
WIDE_VARIANTS=3,1 timeout 300 python scripts/wide_check.py parity 4194304 4 16 8 > gpurun_out/w2_c.log 2>&1; tail -n 3 gpurun_out/w2_c.log
WIDE_VARIANTS=2,0 timeout 300 python scripts/wide_check.py parity 4194304 1 16 12 > gpurun_out/w2_d.log 2>&1; tail -n 3 gpurun_out/w2_d.log
ES_EM_WIDE=2 timeout 300 python scripts/wide_check.py time 67108864 32 32 > gpurun_out/w2_t.log 2>&1; tail -n 3 gpurun_out/w2_t.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/w2_pytest.log 2>&1; tail -n 15 gpurun_out/w2_pytest.log
