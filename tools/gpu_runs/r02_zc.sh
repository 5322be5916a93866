set -x
timeout 900 python -m pytest tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/r02_dp_efeb.log 2>&1; echo dp rc $?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "dp" -p no:cacheprovider > gpurun_out/r02_dp_multi_efeb.log 2>&1; echo dpm rc $?
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "efeb" -p no:cacheprovider > gpurun_out/r02_efeb_step.log 2>&1; echo efeb rc $?
