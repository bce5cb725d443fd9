./scripts/chol_probe | tail -4
ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/variant/libeventscope_b200.so timeout 300 python scripts/fin_trace.py 2>&1 | tail -2 | cut -c1-300
ES_EM_SPEC=1 timeout 600 python scripts/iter_overhead.py
