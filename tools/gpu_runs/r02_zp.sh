set -x
timeout 900 python bench.py --steps 3 --warmup 3 --no-recovery --no-cpu-baseline > gpurun_out/r02_bench_check.json 2> gpurun_out/r02_bench_check.log; echo b rc $?
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r02_bench_ref_check.json 2> gpurun_out/r02_bench_ref_check.log; echo r rc $?
