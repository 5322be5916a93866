set -x
timeout 120 python tools/profile_step.py --config C1 --rc none --steps 1 > gpurun_out/r02_k_c1.log 2>&1; echo c1 rc $?
BB_DEBUG=1 timeout 150 python tools/profile_step.py --config C3 --rc none --steps 1 > gpurun_out/r02_k_c3_full.log 2>&1; echo c3 rc $?
tail -c 20000 gpurun_out/r02_k_c3_full.log > gpurun_out/r02_k_c3.log; rm gpurun_out/r02_k_c3_full.log
nvidia-smi --query-gpu=memory.used --format=csv
