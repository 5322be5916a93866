set -x
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "wide_n" -p no:cacheprovider > gpurun_out/r02_mfast_optest.log 2>&1; echo op rc $?
