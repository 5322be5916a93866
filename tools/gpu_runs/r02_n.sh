set -x
export BB_WATCH=30
for i in 1 2 3; do timeout 400 python tools/profile_step.py --config C3 --rc none --steps 25 > gpurun_out/r02_watch_off_$i.log 2>&1; echo off $i rc $?; done
for i in 1 2; do timeout 400 python tools/profile_step.py --config C3 --rc eflb --steps 15 > gpurun_out/r02_watch_on_$i.log 2>&1; echo on $i rc $?; done
