set -x
nvidia-smi --query-gpu=index,name --format=csv
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node=2 --master-port=29703 tools/xport_vs_nccl.py > gpurun_out/r02_xport_vs_nccl_ev.json 2> gpurun_out/r02_xport_vs_nccl_ev.log; echo xp rc $?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_q.log 2>&1; echo suite rc $?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node=2 --master-port=29702 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n2.json 2> gpurun_out/r02_bench_c3_n2.log; echo n2 rc $?
