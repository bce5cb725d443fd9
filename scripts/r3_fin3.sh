ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/variant/libeventscope_b200.so timeout 300 python scripts/fin_trace.py 2>&1 | tail -2 | cut -c1-400
ES_EM_SPEC=1 timeout 600 python scripts/iter_overhead.py
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "spec_branch or parity or multirank or determinism" > gpurun_out/r3_fin3.log 2>&1; tail -3 gpurun_out/r3_fin3.log
