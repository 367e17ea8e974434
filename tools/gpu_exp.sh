# Quick GPU experiment pass: selected parity tests, then C3 timings of experiment libraries
# (tools/exp_*.so) and env switches.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x ${EXP_TESTS} > gpurun_out/exp_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.txt
tail -3 gpurun_out/exp_tests.txt
timeout 600 python tools/exp_variants.py paper_1906_06297_b200/libising.so ${EXP_LIBS} > gpurun_out/exp.txt 2>&1
ISING_RING=0 timeout 300 python tools/exp_variants.py paper_1906_06297_b200/libising.so >> gpurun_out/exp.txt 2>&1
echo "== rules (ring)" >> gpurun_out/exp.txt; timeout 300 python tools/time_rules.py >> gpurun_out/exp.txt 2>&1
echo "== rules (staged)" >> gpurun_out/exp.txt; ISING_RING=0 timeout 300 python tools/time_rules.py >> gpurun_out/exp.txt 2>&1
cat gpurun_out/exp.txt
