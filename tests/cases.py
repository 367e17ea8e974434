"""Seeded synthetic inputs shared by the oracle-side and GPU-side tests and the bench.

Holds no arithmetic of the method: only shapes, temperatures, seeds and plain +-1
lattices drawn from numpy's seeded generator (DESIGN.md §Input recipe)."""
import math

import numpy as np

BETA_TC = 0.4406868  # BASELINE configs[0]/[2]: beta_c rounded as the config states

# BASELINE.json configs (rows, cols, beta, sweeps)
C1 = (64, 64, BETA_TC, 1000)
C2 = (2048, 2048, (1 / 1.5, 1 / 3.0), 20000)
C3 = (32768, 32768, BETA_TC, 128)
C4 = (131072, 131072, BETA_TC, 128)
C5_ROWS_PER_GPU, C5_COLS = 131072, 1048576

# parity matrix: W = 2 (both side words wrap inside one chunk),
# odd chunk count and non power of two rows (130 x 192), non-square.
PARITY_SHAPES = [(64, 64), (66, 64), (64, 128), (130, 192), (256, 256), (2, 64)]
# 4e-11: T3 = 2^32 ("always") while T4 = 2^32 - 1, the generic kernel with mixed keep masks
PARITY_BETAS = [0.0, 0.2, BETA_TC, 0.8, math.inf, 4e-11]
PARITY_SEEDS = [1, 2]

# (rows, cols, slabs): R = 2 (every row a boundary row), 2 slabs (up = down peer)
# (SURVEY §8(c) multi-GPU additions: 16 x 64 at n = 8 (R = 2), 64 x 64 at n = 2, 4096^2 at
# n = 2, 4, 8; 4096 x 8192 at n = 8 runs the TMA-staged kernel)
SLAB_CASES = [(16, 64, 8), (64, 64, 2), (256, 256, 4), (96, 192, 3), (4096, 4096, 2),
              (4096, 4096, 4), (4096, 4096, 8), (4096, 8192, 8)]


def random_pm1(rng: np.random.Generator, N: int, M: int, p_up: float = 0.5) -> np.ndarray:
    return np.where(rng.random((N, M)) < p_up, 1, -1).astype(np.int8)


def alternating_rows(N: int, M: int) -> np.ndarray:
    """Rows alternating +1 / -1: every site has s*h = 0 (a period-2 trap, reading R21)."""
    return (np.where(np.arange(N)[:, None] % 2 == 0, 1, -1) * np.ones((1, M))).astype(np.int8)


def neel(N: int, M: int) -> np.ndarray:
    return np.where(np.add.outer(np.arange(N), np.arange(M)) % 2 == 0, 1, -1).astype(np.int8)
