for v in A B C; do
  export ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/v_$v/libeventscope_b200.so
  timeout 300 python scripts/diag_check.py parity 16777216 16 16 6 2 > gpurun_out/dab2_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/dab2_$v.log | cut -c1-250)"
  DIAG_VARIANTS=1 timeout 300 python scripts/diag_check.py time 268435456 16 16 2>&1 | tail -1
done
