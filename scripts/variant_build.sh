# Build paper_2506_02007_b200/lib/variant/libeventscope_b200.so: the normal objects with one
# CUDA source ($1, e.g. es_score_mma.cu) recompiled with extra flags ($2...), for A/B runs
# through ES_LIB_OVERRIDE (scripts/ab_lib.sh).
set -e
cd "$(dirname "$0")/.."
src=$1
shift
python -c "from paper_2506_02007_b200 import _build; _build.build()"
L=paper_2506_02007_b200/lib
mkdir -p $L/variant
nvcc "$@" -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I include \
  -gencode arch=compute_100a,code=sm_100a -c paper_2506_02007_b200/csrc/$src -o $L/variant/$src.o
objs=$(ls $L/obj/*.o | grep -v "/$src.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $L/variant/libeventscope_b200.so $objs $L/variant/$src.o -ldl
echo built $L/variant/libeventscope_b200.so
