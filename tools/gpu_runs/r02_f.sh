set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "failstop or modes" > gpurun_out/r02_failstop_f.log 2>&1; echo fs rc $?
timeout 900 python -m pytest tests/test_gpu_step.py -q -p no:cacheprovider -k "efeb or zipf or lflb" > gpurun_out/r02_efeb_f.log 2>&1; echo efeb rc $?
timeout 600 python tools/op_bench.py C3 > gpurun_out/r02_op_bench_c3.txt 2>&1; echo ops rc $?
