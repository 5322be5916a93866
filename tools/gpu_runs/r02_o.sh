set -x
export BB_WATCH=20 BB_GEMM_TRACE=1
for i in 1 2 3; do timeout 300 python tools/profile_step.py --config C3 --rc none --steps 20 > gpurun_out/r02_watch2_off_$i.log 2>&1; echo off $i rc $?; done
