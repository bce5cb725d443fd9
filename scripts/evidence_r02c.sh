# Round-2 final evidence (session 3, end): GPU tests, default bench line, reference arm, ncu launch
# list of the bench command, smoke.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev4_pytest.log 2>&1; tail -3 gpurun_out/ev4_pytest.log
timeout 900 python bench.py > gpurun_out/ev4_bench.log 2> gpurun_out/ev4_bench.err; tail -c 3800 gpurun_out/ev4_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev4_ref.log 2> gpurun_out/ev4_ref.err; tail -c 1500 gpurun_out/ev4_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev4_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev4_launch_run.log 2>&1
python scripts/launch_table.py gpurun_out/ev4_launches.csv > gpurun_out/ev4_launch_table.txt 2>&1; head -24 gpurun_out/ev4_launch_table.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev4_smoke.log 2>&1; tail -1 gpurun_out/ev4_smoke.log
