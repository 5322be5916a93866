set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 1200 $TR --nproc-per-node=4 --master-port=29731 tools/mode_overhead.py --config C2 --steps 5 --warmup 2 > gpurun_out/r02_modes_c2_n4.json 2> gpurun_out/r02_modes_c2_n4.log; echo modesc2 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29732 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n4_final.json 2> gpurun_out/r02_bench_c3_n4_final.log; echo c3n4 rc $?
