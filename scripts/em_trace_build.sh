# Build paper_2506_02007_b200/lib/trace/libeventscope_b200.so: the normal objects with
# es_em_mma.cu compiled -DES_EM_TRACE (CTA 0 pipeline timeline, see scripts/em_trace.py).
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2506_02007_b200 import _build; _build.build()"
L=paper_2506_02007_b200/lib
mkdir -p $L/trace
nvcc -DES_EM_TRACE -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I include \
  -gencode arch=compute_100a,code=sm_100a -c paper_2506_02007_b200/csrc/es_em_mma.cu -o $L/trace/es_em_mma.o
objs=$(ls $L/obj/*.o | grep -v es_em_mma)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $L/trace/libeventscope_b200.so $objs $L/trace/es_em_mma.o -ldl
echo built $L/trace/libeventscope_b200.so
