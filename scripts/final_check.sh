# Round-end check on one B200: CPU+GPU test suites, smoke(), default bench line, reference arm.
set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final_gpu_tests.txt 2>&1; tail -3 gpurun_out/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.txt 2>&1; tail -2 gpurun_out/final_smoke.txt
timeout 900 python bench.py > gpurun_out/final_bench.log 2> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.log 2> gpurun_out/final_ref.err
