set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/parity_report.py C0 > gpurun_out/r02_parity_c0.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02_gpu_suite0.log 2>&1; echo suite rc $?
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -q -x -k "custom_partition or recovery_bitwise" > gpurun_out/r02_memcheck.log 2>&1; echo memcheck rc $?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_step.py -q -x -k "custom_partition and lps0" > gpurun_out/r02_racecheck.log 2>&1; echo racecheck rc $?
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_step.py -q -x -k "custom_partition and lps0" > gpurun_out/r02_synccheck.log 2>&1; echo synccheck rc $?
