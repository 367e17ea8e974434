timeout 600 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 -k trace > gpurun_out/t_trace.log 2>&1; echo "trace: $(tail -1 gpurun_out/t_trace.log)"
timeout 600 python tools/exp_variants.py paper_1906_06297_b200/libising.so tools/exp_r2d.so > gpurun_out/exp_r2d.txt 2>&1; cat gpurun_out/exp_r2d.txt
