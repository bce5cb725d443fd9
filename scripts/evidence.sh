# Round-end evidence on one B200: default bench line, reference arm, ncu launch list,
# ncu --set full of the two hot kernels (reports land in gpurun_out/; summaries go to profiles/).
set -x
timeout 900 python bench.py > gpurun_out/ev_bench.log 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/ev_ref.log 2> gpurun_out/ev_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ev_launch_run.log 2>&1
ES_EM_MMA_PASSES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_em_mma -s 1 -c 1 \
  -f -o gpurun_out/ev_k_em_mma python scripts/prof_em.py 67108864 > gpurun_out/ev_ncu_em.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_mma -c 1 \
  -f -o gpurun_out/ev_k_score_mma python scripts/prof_em.py 67108864 > gpurun_out/ev_ncu_score.log 2>&1
