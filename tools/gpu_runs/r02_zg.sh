set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port=29771 bench.py --gpus 4 --steps 10 --warmup 3 --config C2 > gpurun_out/r02_bench_c2_n4.json 2> gpurun_out/r02_bench_c2_n4.log; echo c2 rc $?
