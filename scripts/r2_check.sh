# round-2 quick check: GPU tests (minus the 4-minute headline oracle fit), bench with and
# without iteration graphs, scorer timing + parity
python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_headline.py > gpurun_out/pt_chk.log 2>&1; tail -4 gpurun_out/pt_chk.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_chk1.log 2>&1; tail -c 300 gpurun_out/b_chk1.log | head -c 300; echo
grep -o '"value": [0-9.]*\|ms_per_step": [0-9.]*\|avg_launch_ms": [0-9.]*\|events_per_s": [0-9.]*' gpurun_out/b_chk1.log
ES_GRAPH=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_chk0.log 2>&1
grep -o '"value": [0-9.]*\|ms_per_step": [0-9.]*\|avg_launch_ms": [0-9.]*' gpurun_out/b_chk0.log
python scripts/score_ab.py 10 2>&1 | tail -4
