set -x
timeout 900 python -m pytest tests/test_gpu_dp.py -q -p no:cacheprovider > gpurun_out/r02_dp_all_modes.log 2>&1; echo dp rc $?
