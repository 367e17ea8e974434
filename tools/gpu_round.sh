#!/bin/bash
# Full evidence pass on one B200: GPU tests (incl. slow), smoke, bench (default args),
# ncu launch list of the bench command's sweep driver, ncu --set full of k_halfsweep.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m "${PYTEST_MARK:-gpu}" --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_sweep.py > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halfsweep -s 2 -c 1 -o gpurun_out/prof_halfsweep python tools/profile_sweep.py > gpurun_out/ncu_full.log 2>&1
tail -25 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json
