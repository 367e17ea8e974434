bash tools/gpu_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
timeout 1200 env ISING_BENCH_SAME_DEVICE=1 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n4_samedev.json 2> gpurun_out/bench_n4_samedev.err; echo "n4 rc=$?"
