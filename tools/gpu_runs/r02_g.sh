set -x
export BB_DEBUG_LOSS=1
mkdir -p /tmp/o1 /tmp/o2 /tmp/o3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29611 tests/mp_worker.py --out /tmp/o1 --config C0 --stages 2 --steps 3 --failstop 1:1:9 --detect 300 > gpurun_out/r02_fs_dbg1.log 2>&1; echo fs1 rc $?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr=127.0.0.1 --master-port=29612 tests/mp_worker.py --out /tmp/o3 --config C0 --stages 3 --steps 2 --rc efeb --victim 1 --pi 12 > gpurun_out/r02_modes_dbg.log 2>&1; echo modes rc $?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29613 tests/mp_worker.py --out /tmp/o2 --config C0 --stages 2 --steps 3 --victim 1 --pi 6 > gpurun_out/r02_inj_dbg.log 2>&1; echo inj rc $?
