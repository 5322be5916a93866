set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/r02_gpu_suite_d.log 2>&1; echo suite rc $?
for i in 1 2 3; do timeout 400 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider >> gpurun_out/r02_multi_loop_d.log 2>&1; echo multi $i rc $?; done
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3_d.json 2> gpurun_out/r02_bench_c3_d.log; echo bench rc $?
