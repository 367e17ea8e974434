for l in dyn st; do ISING_LIB=tools/exp_wf_$l.so timeout 300 python - <<'X'
import os, sys
sys.path.insert(0, ".")
from paper_1906_06297_b200.ising import IsingLattice
r = []
for N, M in [(32768, 32768), (16384, 32768)]:
    lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
    lat.sweep(4); lat.sweep(64)
    r.append(round(N * M * 64 / (lat.last_sweep_ms() * 1e6), 1))
    lat.close()
print(os.environ["ISING_LIB"], r, flush=True)
X
done
