set -x
for e in 0 1 2; do
  BB_ATTN_EMU=$e BB_ATTN_EMU_BWD=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:fa_|dq_reduce" --csv --log-file gpurun_out/r02_attn_c3_emu$e.csv python tools/attn_time.py C3 5 > gpurun_out/r02_attn_c3_emu$e.log 2>&1; echo c3 $e rc $?
  BB_ATTN_EMU=$e BB_ATTN_EMU_BWD=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:fa_|dq_reduce" --csv --log-file gpurun_out/r02_attn_c1_emu$e.csv python tools/attn_time.py C1 5 > gpurun_out/r02_attn_c1_emu$e.log 2>&1; echo c1 $e rc $?
done
BB_ATTN_EMU_BWD=2 timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "attention" -p no:cacheprovider > gpurun_out/r02_attnbwd_emu2.log 2>&1; echo bwdtest rc $?
