set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port=29751 bench.py --gpus 4 --steps 8 --warmup 3 --no-recovery --frc-persistent > gpurun_out/r02_frcpers_n4.json 2> gpurun_out/r02_frcpers_n4.log; echo pers rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29752 bench.py --gpus 4 --steps 8 --warmup 3 --no-recovery > gpurun_out/r02_frctile_n4.json 2> gpurun_out/r02_frctile_n4.log; echo tile rc $?
CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 900 $TR --nproc-per-node=4 --master-port=29753 bench.py --gpus 4 --steps 8 --warmup 3 --no-recovery > gpurun_out/r02_conn8_n4.json 2> gpurun_out/r02_conn8_n4.log; echo conn8 rc $?
