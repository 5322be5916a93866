set -x
mkdir -p /tmp/o1 /tmp/o3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr=127.0.0.1 --master-port=29612 tests/mp_worker.py --out /tmp/o1 --config C0 --stages 3 --steps 2 --rc efeb > gpurun_out/r02_efeb_mp0.log 2>&1; echo efeb0 rc $?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr=127.0.0.1 --master-port=29613 tests/mp_worker.py --out /tmp/o3 --config C0 --stages 3 --steps 2 --rc efeb --victim 1 --pi 12 > gpurun_out/r02_efeb_mp1.log 2>&1; echo efeb1 rc $?
