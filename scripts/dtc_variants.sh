# Build paper_2506_02007_b200/lib/v_<name>/libeventscope_b200.so variants of es_em_diag_tc.cu
# (precision A/B through ES_LIB_OVERRIDE):  name:flags ...
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2506_02007_b200 import _build; _build.build()"
L=paper_2506_02007_b200/lib
src=es_em_diag_tc.cu
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  mkdir -p $L/v_$name
  nvcc $flags -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I include \
    -gencode arch=compute_100a,code=sm_100a -c paper_2506_02007_b200/csrc/$src -o $L/v_$name/$src.o &
  pids="$pids $!"
done
for p in $pids; do wait $p; done  # set -e: a failed compile stops here
for spec in "$@"; do
  name=${spec%%:*}
  objs=$(ls $L/obj/*.o | grep -v "/$src.o")
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $L/v_$name/libeventscope_b200.so $objs $L/v_$name/$src.o -ldl
  echo built $L/v_$name
done
