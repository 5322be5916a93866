set -x
nvidia-smi --query-gpu=index,name --format=csv
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port=29701 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n4.json 2> gpurun_out/r02_bench_c3_n4.log; echo n4 rc $?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node=2 --master-port=29702 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n2.json 2> gpurun_out/r02_bench_c3_n2.log; echo n2 rc $?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node=2 --master-port=29703 tools/xport_vs_nccl.py > gpurun_out/r02_xport_vs_nccl_n4box.json 2> gpurun_out/r02_xport_vs_nccl_n4box.log; echo xp rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29704 tools/mode_overhead.py --config C3 --steps 5 --warmup 2 > gpurun_out/r02_modes_c3_n4.json 2> gpurun_out/r02_modes_c3_n4.log; echo modes rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29705 tools/sweep_c4.py --config C3 --steps 60 --k 0 1 2 3 > gpurun_out/r02_c4_c3_n4.jsonl 2> gpurun_out/r02_c4_c3_n4.log; echo c4 rc $?
