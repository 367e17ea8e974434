timeout 900 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 -k self_exchange > gpurun_out/t_self.log 2>&1; echo "self: $(tail -1 gpurun_out/t_self.log)"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1d.json 2> gpurun_out/bench_n1d.err; echo "n1 rc=$?"
