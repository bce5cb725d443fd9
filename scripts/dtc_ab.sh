# k_em_diag_tc variants (scripts/dtc_variants.sh): c3 pass time and oracle margins at 2^23, K = 4
for v in ${VARS:-A B C}; do
  export ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/v_$v/libeventscope_b200.so
  DIAG_VARIANTS=1 timeout 300 python scripts/diag_check.py time 268435456 16 16 > gpurun_out/dab_t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/dab_t_$v.log)"
  timeout 300 python scripts/diag_check.py parity 8388608 16 4 8 1 > gpurun_out/dab_p_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/dab_p_$v.log | cut -c1-260)"
done
