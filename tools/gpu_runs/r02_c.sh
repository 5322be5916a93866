set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/r02_gpu_suite_c.log 2>&1; echo suite rc $?
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider >> gpurun_out/r02_multi_loop.log 2>&1; echo multi $i rc $?; done
