set -x
python tools/parity_report.py gpurun_out/r02_parity_table.json > gpurun_out/r02_parity_b.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 -p no:cacheprovider > gpurun_out/r02_gpu_suite_b.log 2>&1; echo suite rc $?
