mkdir -p /tmp/o
run() { timeout 40 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 tests/mp_worker.py --out /tmp/o --config C0 --stages 4 --steps 1 "$@" > /tmp/l.log 2>&1; echo "$* rc=$?"; }
run --rc 0
BB_FRC_PRIO=0 run --rc 1
CUDA_DEVICE_MAX_CONNECTIONS=1 run --rc 0
