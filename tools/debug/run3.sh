for t in test_local_group_large test_local_group_measured; do
  timeout 600 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 -k $t > gpurun_out/t_conc_$t.log 2>&1; echo "$t: $(tail -1 gpurun_out/t_conc_$t.log)"
done
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.txt)"
for v in sel1 sel2; do
  ISING_LIB=tools/exp_$v.so timeout 600 ncu --section ComputeWorkloadAnalysis --section SpeedOfLight --section WarpStateStats --section InstructionStats --clock-control none -k regex:k_halfsweep_staged -s 2 -c 1 -o gpurun_out/r02_var_$v python tools/profile_sweep.py > gpurun_out/ncu_var_$v.log 2>&1
done
echo done
