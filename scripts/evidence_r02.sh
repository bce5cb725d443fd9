# Round-2 evidence on one B200: GPU tests, default bench line, reference arm, ncu launch list,
# ncu --set full of the two hot kernels (reports land in gpurun_out/; summaries go to profiles/).
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev2_pytest.log 2>&1
tail -3 gpurun_out/ev2_pytest.log
timeout 900 python bench.py > gpurun_out/ev2_bench.log 2> gpurun_out/ev2_bench.err
tail -c 3000 gpurun_out/ev2_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev2_ref.log 2> gpurun_out/ev2_ref.err
tail -c 1500 gpurun_out/ev2_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ev2_launch_run.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev2_smoke.log 2>&1; tail -2 gpurun_out/ev2_smoke.log
