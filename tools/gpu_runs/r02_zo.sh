set -x
timeout 300 python tools/op_bench.py C3 > gpurun_out/r02_opb_tile_default.txt 2>&1; echo d rc $?
BB_GEMM_TILE=pair192 timeout 300 python tools/op_bench.py C3 > gpurun_out/r02_opb_tile_pair192.txt 2>&1; echo p rc $?
timeout 300 python tools/op_bench.py C3 > gpurun_out/r02_opb_tile_default2.txt 2>&1; echo d2 rc $?
BB_GEMM_TILE=pair192 timeout 300 python tools/op_bench.py C3 > gpurun_out/r02_opb_tile_pair192b.txt 2>&1; echo p2 rc $?
