cat > /tmp/gm.sh <<'X'
for c in "init-measure 2 64 128" "init-skew-measure 2 64 8192" "write-measure 4 128 8192"; do
  echo "== $c"; timeout 90 python tools/debug/group_measure.py $c 2>&1 | grep -v "^  File\|^    " | tail -4
done
X
bash /tmp/gm.sh > gpurun_out/dbg5.log 2>&1
for t in test_local_group_measured_chain_load_and_heat_bath test_self_exchange test_profiling test_local_group_500 test_local_group_large; do
  timeout 600 python -m pytest tests/test_gpu_concurrent.py -q --timeout 300 -k $t > gpurun_out/t_conc_$t.log 2>&1; echo "$t: $(tail -1 gpurun_out/t_conc_$t.log)"
done
timeout 900 env ISING_BENCH_SAME_DEVICE=1 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_samedev.json 2> gpurun_out/bench_n2_samedev.err; echo "samedev rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1b.json 2> gpurun_out/bench_n1b.err; echo "n1 rc=$?"
