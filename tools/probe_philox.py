"""Run the live Philox-only probe once (for ncu: python tools/probe_philox.py)."""
import sys; sys.path.insert(0, ".")
from paper_1906_06297_b200.ising import ising_probe_philox
print("probe", ising_probe_philox(0))
