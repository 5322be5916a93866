set -x
export BB_WATCH=20
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "gemm" -p no:cacheprovider > gpurun_out/r02_gemm_tests_p.log 2>&1; echo gemmtests rc $?
for i in 1 2 3 4; do timeout 300 python tools/profile_step.py --config C3 --rc none --steps 20 > gpurun_out/r02_watch3_off_$i.log 2>&1; echo off $i rc $?; done
for i in 1 2; do timeout 300 python tools/profile_step.py --config C3 --rc eflb --steps 15 > gpurun_out/r02_watch3_on_$i.log 2>&1; echo on $i rc $?; done
