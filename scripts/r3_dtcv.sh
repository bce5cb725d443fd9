for v in ${VARS:-A B C D E}; do
  export ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/v_$v/libeventscope_b200.so
  timeout 300 python scripts/diag_check.py parity 8388608 16 4 8 1 > gpurun_out/r3v_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r3v_$v.log)"
  timeout 300 python scripts/diag_check.py parity 16777216 16 8 6 2 > gpurun_out/r3w_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r3w_$v.log)"
  DIAG_VARIANTS=1 timeout 300 python scripts/diag_check.py time 268435456 16 16 > gpurun_out/r3t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r3t_$v.log)"
done
