set -x
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k dp -p no:cacheprovider > gpurun_out/r02_dp_multi2.log 2>&1; echo dpmulti rc $?
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "host_swap or retention" -p no:cacheprovider > gpurun_out/r02_swap_tests.log 2>&1; echo swap rc $?
# stress: the round-1 flaky cases (custom partition incl. lps0, recovery) 50 times
pass=0; fail=0
for i in $(seq 1 50); do
  if timeout 120 python -m pytest tests/test_gpu_step.py -x -q -k "custom_partition or c0_preemption_recovery" -p no:cacheprovider > gpurun_out/r02_stress_last.log 2>&1; then pass=$((pass+1)); else fail=$((fail+1)); cp gpurun_out/r02_stress_last.log gpurun_out/r02_stress_fail_$i.log; fi
  echo "iter $i pass $pass fail $fail" >> gpurun_out/r02_stress.log
done
echo stress pass $pass fail $fail
timeout 300 python tools/swap_cost.py --config C1 --keep 2 > gpurun_out/r02_swap_c1_n1.json 2> gpurun_out/r02_swap_c1_n1.log; echo swapc1 rc $?
