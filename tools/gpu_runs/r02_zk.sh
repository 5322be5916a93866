set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_final3.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_final3.log 2>&1; echo suite rc $?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n1_final3.json 2> gpurun_out/r02_bench_c3_n1_final3.log; echo n1 rc $?
