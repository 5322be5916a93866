set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port=29781 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n4_final3.json 2> gpurun_out/r02_bench_c3_n4_final3.log; echo n4 rc $?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node=2 --master-port=29782 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n2_final3.json 2> gpurun_out/r02_bench_c3_n2_final3.log; echo n2 rc $?
