#!/bin/bash
# Round-end evidence pass on one B200: the GPU suite, smoke, the driver's bench command (and the
# reference arm), compute-sanitizer (four tools).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
if [ -n "$SAN" ]; then bash tools/gpu_sanitize.sh; fi
