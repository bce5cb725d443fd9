set -x
ES_EM_DEBUG=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r3d_bench.log 2> gpurun_out/r3d_bench.err; tail -c 600 gpurun_out/r3d_bench.log; grep "es em" gpurun_out/r3d_bench.err | head -40
