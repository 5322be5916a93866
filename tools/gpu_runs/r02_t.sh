set -x
nvidia-smi --query-gpu=index,name --format=csv
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "host_swap" -p no:cacheprovider > gpurun_out/r02_swap_tests2.log 2>&1; echo swaptest rc $?
timeout 600 python -m pytest tests/test_gpu_multi.py -q -k "dp or equals_single or failstop" -p no:cacheprovider > gpurun_out/r02_multi_4gpu.log 2>&1; echo multi4 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29711 bench.py --gpus 4 --steps 6 --warmup 3 --pipelines 2 --no-cpu-baseline > gpurun_out/r02_bench_c3_d2_n4.json 2> gpurun_out/r02_bench_c3_d2_n4.log; echo c3d2 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29712 bench.py --gpus 4 --steps 10 --warmup 3 --config C1 --pipelines 2 --no-cpu-baseline > gpurun_out/r02_bench_c1_d2_n4.json 2> gpurun_out/r02_bench_c1_d2_n4.log; echo c1d2 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29713 bench.py --gpus 4 --steps 10 --warmup 3 --config C1 --no-cpu-baseline > gpurun_out/r02_bench_c1_n4.json 2> gpurun_out/r02_bench_c1_n4.log; echo c1 rc $?
timeout 900 $TR --nproc-per-node=4 --master-port=29714 tools/swap_cost.py --config C3 --keep 4 --swap-sets 4 > gpurun_out/r02_swap_c3_n4.json 2> gpurun_out/r02_swap_c3_n4.log; echo swapc3 rc $?
# partition experiment at N=4 (2 nodes per GPU): per-node balance (default) vs per-GPU sums
for v in "balanced" "lps:5,7,7,6,4,8,5,6" "device"; do
  case $v in lps:*) arg="--lps ${v#lps:}";; *) arg="--partition $v";; esac
  timeout 900 $TR --nproc-per-node=4 --master-port=29715 bench.py --gpus 4 --steps 8 --warmup 3 --no-recovery $arg > gpurun_out/r02_part_${v%%:*}_n4.json 2> gpurun_out/r02_part_${v%%:*}_n4.log; echo part $v rc $?
done
