set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_step.py -q -k "custom_partition or host_swap" -p no:cacheprovider > gpurun_out/r02_custom_part.log 2>&1; echo custom rc $?
timeout 900 $TR --nproc-per-node=2 --master-port=29721 bench.py --gpus 2 --steps 8 --warmup 3 --no-recovery --partition device > gpurun_out/r02_part_device_n2.json 2> gpurun_out/r02_part_device_n2.log; echo dev2 rc $?
timeout 900 $TR --nproc-per-node=2 --master-port=29722 bench.py --gpus 2 --steps 8 --warmup 3 --no-recovery --partition balanced > gpurun_out/r02_part_balanced_n2.json 2> gpurun_out/r02_part_balanced_n2.log; echo bal2 rc $?
