# alternate A / B library variants: $1 = script (default scripts/em_time.py), 3 rounds
S=${1:-scripts/em_time.py}
for i in 1 2 3; do for v in A B; do ES_LIB_OVERRIDE=paper_2506_02007_b200/lib/ab$v/libeventscope_b200.so python $S 2>&1 | tail -1; done; done
