# compute-sanitizer over tools/sanitize.py: memcheck (with the guided-tail lattice), racecheck,
# synccheck, initcheck.
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
out=gpurun_out/compute_sanitizer.txt
echo "# compute-sanitizer on tools/sanitize.py" > $out
echo "## memcheck (SANITIZE_BIG=1)" >> $out; SANITIZE_BIG=1 timeout 1200 $S --tool memcheck python tools/sanitize.py >> $out 2>&1
for t in racecheck synccheck initcheck; do echo "## $t" >> $out; timeout 1200 $S --tool $t python tools/sanitize.py >> $out 2>&1; done
grep -E "SUMMARY|^## " $out
