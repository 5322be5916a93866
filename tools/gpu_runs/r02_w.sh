set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_final.log 2>&1; echo suite rc $?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c3_n1_final.json 2> gpurun_out/r02_bench_c3_n1_final.log; echo n1 rc $?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.log; echo ref rc $?
