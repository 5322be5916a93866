set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port=29791 tools/sweep_c4.py --config C3 --steps 60 --k 0 1 2 3 > gpurun_out/r02_c4_c3_n4_final.jsonl 2> gpurun_out/r02_c4_c3_n4_final.log; echo c4 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29792 tools/mode_overhead.py --config C3 --steps 5 --warmup 2 > gpurun_out/r02_modes_c3_n4_final.json 2> gpurun_out/r02_modes_c3_n4_final.log; echo modes rc $?
