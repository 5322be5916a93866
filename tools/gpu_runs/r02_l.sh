set -x
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3_l.json 2> gpurun_out/r02_bench_c3_l.log; echo bench rc $?
