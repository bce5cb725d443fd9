set -x
ES_EM_DEBUG=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r3e_bench.log 2> gpurun_out/r3e_bench.err; tail -c 1500 gpurun_out/r3e_bench.log; grep -c "kept=0" gpurun_out/r3e_bench.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3e_pytest.log 2>&1; tail -5 gpurun_out/r3e_pytest.log
