# ncu --set full of the round-2 scorer and diagonal pass (current builds)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_mma -s 4 -c 1 \
  -f -o gpurun_out/r02_score_final python scripts/score_ab.py 2 > gpurun_out/r02_ncu_score_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_em_diag_mixed -s 1 -c 1 \
  -f -o gpurun_out/r02_diag_final python scripts/prof_diag.py > gpurun_out/r02_ncu_diag_final.log 2>&1
ls -la gpurun_out/r02_*final*
