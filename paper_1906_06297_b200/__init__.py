"""paper_1906_06297_b200 — B200-native multi-spin checkerboard Metropolis (arXiv 1906.06297).

The product is ``libising.so`` (C ABI in ``include/ising.h``, sm_100a kernels in
``csrc/``); ``ising`` is its ctypes binding.  See DESIGN.md.
"""
from .ising import (  # noqa: F401
    RULE_HEATBATH,
    RULE_METROPOLIS,
    IsingError,
    IsingLattice,
    load,
)
