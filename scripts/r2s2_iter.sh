# fixed-cost A/B (speculative loop on/off) + GPU tests touching the EM loop + finalize profile
set -x
ES_EM_SPEC=0 timeout 600 python scripts/iter_overhead.py > gpurun_out/it_spec0.log 2>&1; cat gpurun_out/it_spec0.log
ES_EM_SPEC=1 timeout 600 python scripts/iter_overhead.py > gpurun_out/it_spec1.log 2>&1; cat gpurun_out/it_spec1.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; tail -15 gpurun_out/it_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_finalize|k_em_mma|k_reduce" -c 40 --csv --log-file gpurun_out/it_launch.csv python scripts/iter_overhead.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/it_launch.csv 2>/dev/null | head -20
