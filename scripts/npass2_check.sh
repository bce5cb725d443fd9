# NPASS = 2 Gram order check: parity subsets + headline margins (c2, 25 iterations) + NPASS=2 forced margins
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "parity or headline or wide_pass or determinism" > gpurun_out/np2_pytest.log 2>&1; tail -3 gpurun_out/np2_pytest.log
timeout 900 python scripts/headline_parity.py 67108864 25 > gpurun_out/np2_headline.log 2>&1; grep -E "margins|score" gpurun_out/np2_headline.log | head -6
ES_EM_MMA_PASSES=2 timeout 600 python tests/parity_report.py 33554432 16 8 6 > gpurun_out/np2_forced.log 2>&1; tail -2 gpurun_out/np2_forced.log
timeout 300 python scripts/em_time.py
ES_EM_MMA_PASSES=2 timeout 300 python scripts/em_time.py
