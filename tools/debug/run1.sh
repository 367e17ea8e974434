timeout 900 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 > gpurun_out/t_conc.log 2>&1; tail -5 gpurun_out/t_conc.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -3 gpurun_out/bench_n1.err
timeout 600 python tools/exp_variants.py paper_1906_06297_b200/libising.so tools/exp_sel1.so tools/exp_sel2.so > gpurun_out/exp_sel.txt 2>&1
