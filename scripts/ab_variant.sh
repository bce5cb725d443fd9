# Build lib/abA (sources of git revision $1 for file $2) and lib/abB (working tree) for A/B runs.
set -e
cd "$(dirname "$0")/.."
rev=$1; f=$2
python -c "from paper_2506_02007_b200 import _build; _build.build()"
L=paper_2506_02007_b200/lib
for v in A B; do mkdir -p $L/ab$v; done
git show $rev:paper_2506_02007_b200/csrc/$f > $L/abA/$f
cp paper_2506_02007_b200/csrc/$f $L/abB/$f
for v in A B; do
  nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I include -I paper_2506_02007_b200/csrc \
    -gencode arch=compute_100a,code=sm_100a -c $L/ab$v/$f -o $L/ab$v/$f.o
  objs=$(ls $L/obj/*.o | grep -v "/$f.o")
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $L/ab$v/libeventscope_b200.so $objs $L/ab$v/$f.o -ldl
done
echo built $L/abA $L/abB
