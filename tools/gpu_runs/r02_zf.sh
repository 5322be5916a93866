set -x
# rehearsal of the driver's N=8 run on a 4-GPU box: 8 ranks, one node each,
# two ranks per GPU (gloo harness), fixed FRC budget so both fit
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 1500 $TR --nproc-per-node=8 --master-port=29761 bench.py --gpus 8 --steps 3 --warmup 3 --retain 14000000000 --no-cpu-baseline > gpurun_out/r02_rehearse_n8.json 2> gpurun_out/r02_rehearse_n8.log; echo n8 rc $?
timeout 300 $TR --nproc-per-node=8 --master-port=29762 bench.py --impl reference --gpus 8 --steps 1 --warmup 1 > gpurun_out/r02_rehearse_ref_n8.json 2> gpurun_out/r02_rehearse_ref_n8.log; echo ref8 rc $?
