# Round-2 final evidence on one B200 (session 3): GPU tests, default bench line, reference arm,
# ncu launch list of the bench command, smoke, c3 timing + ncu of k_em_diag_tc.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev3_pytest.log 2>&1; tail -3 gpurun_out/ev3_pytest.log
timeout 900 python bench.py > gpurun_out/ev3_bench.log 2> gpurun_out/ev3_bench.err; tail -c 3500 gpurun_out/ev3_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev3_ref.log 2> gpurun_out/ev3_ref.err; tail -c 1500 gpurun_out/ev3_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ev3_launch_run.log 2>&1
python scripts/launch_table.py gpurun_out/ev3_launches.csv > gpurun_out/ev3_launch_table.txt 2>&1; head -20 gpurun_out/ev3_launch_table.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3_smoke.log 2>&1; tail -1 gpurun_out/ev3_smoke.log
DIAG_VARIANTS=1 timeout 300 python scripts/diag_check.py time 268435456 16 16 > gpurun_out/ev3_c3.log 2>&1; tail -1 gpurun_out/ev3_c3.log
DIAG_VARIANTS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_em_diag_tc --launch-skip 4 -c 1 -o gpurun_out/ev3_dtc python scripts/diag_check.py time 268435456 16 16 > gpurun_out/ev3_dtc_ncu.log 2>&1; tail -1 gpurun_out/ev3_dtc_ncu.log
