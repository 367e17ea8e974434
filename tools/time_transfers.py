import sys, time, torch
sys.path.insert(0, ".")
from paper_1906_06297_b200.ising import IsingLattice
N = M = 32768
lat = IsingLattice(N, M, 1).set_beta(0.44).init_random()
a = torch.empty((N, M), dtype=torch.int8, pin_memory=True)
lat.read_lattice(a.numpy())
for _ in range(2):
    t0 = time.perf_counter(); lat.write_lattice(a.numpy()); t1 = time.perf_counter()
    lat.read_lattice(a.numpy()); t2 = time.perf_counter()
    print(f"write_lattice {N*M/(t1-t0)/1e9:.1f} GB/s  read_lattice {N*M/(t2-t1)/1e9:.1f} GB/s")
d = torch.empty((N, M), dtype=torch.int8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    a.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"torch pinned H2D {N*M/(t1-t0)/1e9:.1f} GB/s  D2H {N*M/(t2-t1)/1e9:.1f} GB/s")
