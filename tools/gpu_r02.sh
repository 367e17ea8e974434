#!/bin/bash
# Round-2 evidence pass on one B200: concurrency tests (one pytest process per group so a
# deadlock cannot poison the others), the full GPU suite, smoke, ncu captures.
mkdir -p gpurun_out
for t in test_local_group_measured_chain_load_and_heat_bath test_local_group_large test_local_group_500 test_self_exchange test_profiling; do
  timeout 600 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 -k $t > gpurun_out/t_conc_$t.log 2>&1; echo "$t: $(tail -1 gpurun_out/t_conc_$t.log)"
done
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.txt)"
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; cat gpurun_out/smoke.txt | tail -1
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-legs > gpurun_out/ncu_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halfsweep_staged -s 2 -c 1 -o gpurun_out/r02_prof_local python tools/profile_sweep.py > gpurun_out/ncu_full_local.log 2>&1
  PROF_SELF=p2p timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halfsweep_staged -s 2 -c 1 -o gpurun_out/r02_prof_p2pself python tools/profile_sweep.py > gpurun_out/ncu_full_p2p.log 2>&1
  echo "ncu rc=$?"
fi
