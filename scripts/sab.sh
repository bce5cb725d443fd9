V=paper_2506_02007_b200/lib/variant/libeventscope_b200.so
for m in bound all argmax none; do echo "== $m"; ES_LIB_OVERRIDE=$V ES_SCORE_REFINE=$m python scripts/score_ab.py 10 2>&1 | grep -E "refined|detect|parity|flags"; done
for m in bound argmax none; do echo "== nocount $m"; ES_SCORE_REFINE=$m python scripts/score_ab.py 10 2>&1 | grep -E "detect"; done
