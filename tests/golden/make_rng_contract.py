"""Regenerate tests/golden/rng_contract.txt from the oracle (calls only oracle/).

The draw contract is this build's reading R6, not the paper's, so these values
are regression fixtures of the contract as the oracle evaluates it; the contract itself is
pinned independently by the Random123 KAT (the Philox) and by
test_draw_uses_one_block_per_four_sites (the counter layout)."""
import hashlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

lines = [
    "# Golden values of the draw contract r(seed, t, c, i, j) = Philox4x32-10(ctr = {t, j>>2, c, i},",
    "# key = {lo32(seed), hi32(seed)})[j & 3]  (DESIGN.md reading R6) and of the random start",
    "# sigma = +1 iff r(seed, 0, c, i, j) < 2^31 (reading R8).  Written by",
    "# tests/golden/make_rng_contract.py, which calls only oracle/ (regression fixtures of the",
    "# contract; the contract is pinned by the Random123 KAT and the counter-layout test).",
    "# format: draw seed t c i j0 -> four hex words for j = j0..j0+3",
]
for seed, t, c, i, j0 in [(1, 0, 0, 0, 0), (1, 1, 0, 0, 0), (1, 1, 1, 5, 8), (2**40 + 7, 9, 1, 123456, 4096)]:
    w = [oracle.rand(seed, t, c, i, j0 + k) for k in range(4)]
    lines.append(f"draw {seed} {t} {c} {i} {j0} -> " + " ".join(f"{x:08x}" for x in w))
lines.append("# format: init N M seed -> up bond_energy sha256-prefix-of-row-major-int8")
for N, M, seed in [(64, 64, 1), (2048, 2048, 1)]:
    lat = oracle.Lattice(N, M, seed).init_random()
    up, E = lat.observables()
    sha = hashlib.sha256(lat.full().tobytes()).hexdigest()[:32]
    lines.append(f"init {N} {M} {seed} -> {up} {E} {sha}")
lines.append("# format: init4x4 seed -> the 4 rows of the full lattice")
rows = oracle.Lattice(4, 4, 1).init_random().full().tolist()
lines.append("init4x4 1 -> " + " | ".join(" ".join(str(v) for v in r) for r in rows))
with open(os.path.join(HERE, "rng_contract.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
