set -x
timeout 900 python -m pytest tests/test_gpu_dp.py -q -p no:cacheprovider > gpurun_out/r02_dp_efeb2.log 2>&1; echo dp rc $?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "efeb" -p no:cacheprovider > gpurun_out/r02_dp_multi_efeb2.log 2>&1; echo dpm rc $?
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "efeb or lflb or c0_preemption" -p no:cacheprovider > gpurun_out/r02_modes_step2.log 2>&1; echo modes rc $?
