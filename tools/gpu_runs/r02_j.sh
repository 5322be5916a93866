set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/r02_gpu_suite_j.log 2>&1; echo suite rc $?
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_j.json 2> gpurun_out/r02_bench_c3_j.log; echo bench rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 51216 -c 51216 --csv --log-file gpurun_out/r02_c3_launches.csv python tools/profile_step.py --config C3 --steps 2 > gpurun_out/r02_ncu_launch.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 3000 -c 12 -o gpurun_out/r02_c3_gemm python tools/profile_step.py --config C3 --steps 1 > gpurun_out/r02_ncu_gemm.log 2>&1; echo ncu2 rc $?
timeout 900 ncu --set full --clock-control none -k regex:"ln_|fa_fwd|fa_bwd|colreduce" --launch-skip 200 -c 10 -o gpurun_out/r02_c3_misc python tools/profile_step.py --config C3 --steps 1 > gpurun_out/r02_ncu_misc.log 2>&1; echo ncu3 rc $?
