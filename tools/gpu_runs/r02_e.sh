set -x
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 1500 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/r02_gpu_suite_e.log 2>&1; echo suite rc $?
timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3_e.json 2> gpurun_out/r02_bench_c3_e.log; echo bench rc $?
