for v in ${VARS:-A B C}; do
  export ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/v_$v/libeventscope_b200.so
  DIAG_VARIANTS=1 timeout 300 python scripts/diag_check.py time 268435456 16 16 > gpurun_out/r3t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r3t_$v.log)"
  timeout 300 python scripts/diag_check.py parity 8388608 16 4 8 1 > gpurun_out/r3v_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r3v_$v.log)"
done
unset ES_LIB_OVERRIDE
DIAG_VARIANTS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_em_diag_tc --launch-skip 4 -c 1 -o gpurun_out/r3_dtc_full python scripts/diag_check.py time 268435456 16 16 > gpurun_out/r3_dtc_ncu.log 2>&1; tail -3 gpurun_out/r3_dtc_ncu.log
