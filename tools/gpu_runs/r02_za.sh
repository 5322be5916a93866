set -x
for e in 0 1 2; do BB_ATTN_EMU=$e timeout 300 python tools/op_bench.py C3 > gpurun_out/r02_opb_emu$e.txt 2>&1; echo opb $e rc $?; done
for e in 0 1 2; do BB_ATTN_EMU=$e timeout 300 python tools/op_bench.py C1 > gpurun_out/r02_opb_c1_emu$e.txt 2>&1; echo opbc1 $e rc $?; done
for e in 1 2; do BB_ATTN_EMU=$e timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "attention or attn" -p no:cacheprovider > gpurun_out/r02_attn_emu$e.log 2>&1; echo attn $e rc $?; done
BB_ATTN_EMU=2 timeout 600 python -m pytest tests/test_gpu_step.py -q -k "c0_steps_match or pt1 or pt2" -p no:cacheprovider > gpurun_out/r02_step_emu2.log 2>&1; echo step2 rc $?
