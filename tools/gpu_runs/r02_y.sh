set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 300 $TR --nproc-per-node=2 --master-port=29741 tools/xport_vs_nccl.py > gpurun_out/r02_xport_vs_nccl_fixed.json 2> gpurun_out/r02_xport_vs_nccl_fixed.log; echo xp rc $?
