# session check on one B200: GPU tests + default bench line + smoke
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/s2_pytest.log 2>&1
tail -5 gpurun_out/s2_pytest.log
timeout 900 python bench.py > gpurun_out/s2_bench.log 2> gpurun_out/s2_bench.err
tail -c 3000 gpurun_out/s2_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; tail -2 gpurun_out/s2_smoke.log
