timeout 900 python -m pytest tests/test_gpu_bits.py -q --timeout 300 > gpurun_out/t_bits.log 2>&1; echo "bits: $(tail -1 gpurun_out/t_bits.log)"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1c.json 2> gpurun_out/bench_n1c.err; echo "n1 rc=$?"
