# Round evidence pass on one B200: GPU tests, smoke, bench lines (C3 default, C4, C5, C2,
# basic layout), the reference (CPU oracle) arm, and the ncu launch list of the bench command.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config c4 --steps 64 --warmup 4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config c5 --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --config c2 --steps 2048 --warmup 64 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --layout basic --no-cpu-baseline > gpurun_out/bench_basic.json 2> gpurun_out/bench_basic.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt
for f in c3 ref c4 c5 c2 basic; do echo "== $f"; python -c "import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print(d.get('value'), d.get('vs_baseline'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'))"; done
