set -x
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "gemm" -p no:cacheprovider > gpurun_out/r02_gemm_mfast_tests.log 2>&1; echo gemm rc $?
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "pt_full_width or c0_steps or c0_preemption" -p no:cacheprovider > gpurun_out/r02_mfast_step.log 2>&1; echo step rc $?
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc --launch-skip 15 --launch-count 15 -o gpurun_out/r02_c3_gemm_shapes_mfast python tools/gemm_shapes.py C3 > gpurun_out/r02_gemm_shapes_mfast.log 2>&1; echo ncu rc $?
