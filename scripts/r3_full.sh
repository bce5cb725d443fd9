set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3f_pytest.log 2>&1; tail -4 gpurun_out/r3f_pytest.log
timeout 900 python bench.py > gpurun_out/r3f_bench.log 2> gpurun_out/r3f_bench.err; tail -c 3500 gpurun_out/r3f_bench.log
ES_EM_SPEC=1 timeout 600 python scripts/iter_overhead.py
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
