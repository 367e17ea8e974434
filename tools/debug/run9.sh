timeout 900 python -m pytest tests/test_gpu_concurrent.py tests/test_gpu_multiprocess.py tests/test_gpu_bits.py -q --timeout 300 > gpurun_out/t_p2pm.log 2>&1; echo "p2p tests: $(tail -1 gpurun_out/t_p2pm.log)"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; echo "bench rc=$?"
