set -x
timeout 600 python tools/gemm_shapes.py C3 > gpurun_out/r02_gemm_shapes_plain.log 2>&1; echo plain rc $?
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc --launch-skip 15 --launch-count 15 -o gpurun_out/r02_c3_gemm_shapes python tools/gemm_shapes.py C3 > gpurun_out/r02_gemm_shapes_ncu.log 2>&1; echo ncu rc $?
