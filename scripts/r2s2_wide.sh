# wide-kernel bring-up + finalize/fixed-cost check
set -x
ES_EM_WIDE=2 timeout 300 python scripts/wide_check.py parity 4194304 4 32 32 > gpurun_out/w_par1.log 2>&1; tail -5 gpurun_out/w_par1.log
ES_EM_WIDE=2 timeout 300 python scripts/wide_check.py parity 4194304 4 24 12 > gpurun_out/w_par2.log 2>&1; tail -5 gpurun_out/w_par2.log
ES_EM_WIDE=0 timeout 300 python scripts/wide_check.py parity 4194304 4 32 32 > gpurun_out/w_par0.log 2>&1; tail -5 gpurun_out/w_par0.log
timeout 300 python scripts/wide_check.py time 67108864 32 32 > gpurun_out/w_time1.log 2>&1; tail -3 gpurun_out/w_time1.log
ES_EM_WIDE=0 timeout 300 python scripts/wide_check.py time 67108864 32 32 > gpurun_out/w_time0.log 2>&1; tail -3 gpurun_out/w_time0.log
timeout 600 python scripts/iter_overhead.py > gpurun_out/it2.log 2>&1; cat gpurun_out/it2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_finalize|k_em_mma|k_reduce" -c 40 --csv --log-file gpurun_out/it2_launch.csv python scripts/iter_overhead.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/it2_launch.csv 2>/dev/null | head -8
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/w_pytest.log 2>&1; tail -15 gpurun_out/w_pytest.log
