set -x
export BB_WATCH=60
timeout 600 python -m pytest tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/r02_dp_tests.log 2>&1; echo dp rc $?
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k dp -p no:cacheprovider > gpurun_out/r02_dp_multi.log 2>&1; echo dpmulti rc $?
unset BB_WATCH
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_r.log 2>&1; echo suite rc $?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n1.json 2> gpurun_out/r02_bench_c3_n1.log; echo n1 rc $?
