set -x
timeout 600 python tools/op_bench.py C3 > gpurun_out/r02_op_bench_c3_h.txt 2>&1; echo ops rc $?
timeout 1800 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/r02_gpu_suite_h.log 2>&1; echo suite rc $?
