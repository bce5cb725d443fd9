# ncu --set full captures of the two hot kernels at the bench shapes (round 2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_mma -s 4 -c 1 \
  -f -o gpurun_out/r02_score python scripts/score_ab.py 2 > gpurun_out/r02_ncu_score.log 2>&1
ES_EM_MMA_PASSES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_em_mma -s 1 -c 1 \
  -f -o gpurun_out/r02_em python scripts/prof_em.py 67108864 > gpurun_out/r02_ncu_em.log 2>&1
ls -la gpurun_out/r02_*
