set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "dp" -p no:cacheprovider > gpurun_out/r02_failstop_dp.log 2>&1; echo fsdp rc $?
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc --launch-skip 27000 --launch-count 40 -o gpurun_out/r02_c3_gemm40 python tools/profile_step.py --config C3 --rc eflb --steps 2 > gpurun_out/r02_ncu_gemm40.log 2>&1; echo ncu rc $?
