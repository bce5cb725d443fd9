timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diag" > gpurun_out/r3_dtest.log 2>&1; tail -5 gpurun_out/r3_dtest.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "diag or spec_branch or multirank" > gpurun_out/r3_dtest2.log 2>&1; tail -5 gpurun_out/r3_dtest2.log
