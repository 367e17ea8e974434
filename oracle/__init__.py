"""CPU oracle for the checkerboard Metropolis sweep — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product package
``paper_1906_06297_b200`` never imports it, and this package imports nothing
from the product.

``ising_oracle.c`` is the plain byte-per-spin implementation of PAPER.md §2-§3.1
(see its header for the line-by-line citations); this module is ctypes
marshalling around it plus ``exact`` (closed forms and exact enumeration).
Parity status: pinned (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ising_oracle.c")
_LIB = os.path.join(_HERE, "libising_oracle.so")

RULE_METROPOLIS = 0
RULE_HEATBATH = 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C99 + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i8p = ctypes.POINTER(ctypes.c_int8)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i64p = ctypes.POINTER(ctypes.c_int64)
        I64, U64, U32, INT, DBL = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                   ctypes.c_int, ctypes.c_double)
        sig = {
            "oracle_philox4x32_10": (None, [u32p, u32p, u32p]),
            "oracle_rand": (U32, [U64, U32, U32, U32, U64]),
            "oracle_thresholds": (None, [DBL, INT, u64p]),
            "oracle_nn_sum": (INT, [i8p, INT, I64, I64, I64, I64]),
            "oracle_update_lattice": (None, [i8p, i8p, INT, I64, I64, U64, U32, u64p, INT]),
            "oracle_sweep": (None, [i8p, i8p, I64, I64, U64, U32, I64, DBL, INT]),
            "oracle_init_random": (None, [i8p, i8p, I64, I64, U64]),
            "oracle_init_cold": (None, [i8p, i8p, I64, I64]),
            "oracle_full_lattice": (None, [i8p, i8p, I64, I64, i8p]),
            "oracle_from_full": (None, [i8p, i8p, i8p, I64, I64]),
            "oracle_observables": (None, [i8p, i8p, I64, I64, i64p, i64p]),
            "oracle_chain": (None, [i8p, i8p, I64, I64, U64, U32, I64, DBL, INT, i64p, i64p]),
            "oracle_update_slab": (None, [i8p, i8p, i8p, i8p, INT, I64, I64, I64, U64, U32, u64p,
                                           INT]),
            "oracle_sample_after_one_sweep": (INT, [U64, I64, I64, DBL, INT, I64, I64]),
            "oracle_sample_row_after_one_sweep": (None, [U64, I64, I64, DBL, INT, I64, i8p]),
            "oracle_set_threads": (None, [INT]),
            "oracle_get_threads": (INT, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ct))


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c, ctypes.c_uint32), _p(k, ctypes.c_uint32),
                               _p(out, ctypes.c_uint32))
    return out


def rand(seed: int, t: int, c: int, i: int, j: int) -> int:
    return int(lib().oracle_rand(seed, t, c, i, j))


def thresholds(beta: float, rule: int = RULE_METROPOLIS) -> np.ndarray:
    """T[k] for e = 2k - 4, k = 0..4 (uint64; 2**32 means always)."""
    T = np.zeros(5, dtype=np.uint64)
    lib().oracle_thresholds(float(beta), rule, _p(T, ctypes.c_uint64))
    return T


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def update_slab(target: np.ndarray, source: np.ndarray, above: np.ndarray, below: np.ndarray,
                is_black: bool, row0: int, seed: int, t: int, beta: float,
                rule: int = RULE_METROPOLIS) -> None:
    """One colour phase on one horizontal slab, in place on ``target``."""
    T = thresholds(beta, rule)
    nrows, ny = target.shape
    for a in (target, source, above, below):
        assert a.dtype == np.int8 and a.flags["C_CONTIGUOUS"]
    lib().oracle_update_slab(_p(target, ctypes.c_int8), _p(source, ctypes.c_int8),
                             _p(above, ctypes.c_int8), _p(below, ctypes.c_int8), int(bool(is_black)),
                             row0, nrows, ny, seed, t, _p(T, ctypes.c_uint64), rule)


def sample_row_after_one_sweep(seed: int, N: int, M: int, beta: float, i: int,
                               rule: int = RULE_METROPOLIS) -> np.ndarray:
    """Row i after sweep 1 from the random start, site by site (no N x M lattice in memory)."""
    out = np.empty(M, dtype=np.int8)
    lib().oracle_sample_row_after_one_sweep(seed, N, M, float(beta), rule, i, _p(out, ctypes.c_int8))
    return out


class Lattice:
    """Byte-per-spin lattice: black and white planes of shape (N, M/2)."""

    def __init__(self, n_rows: int, n_cols: int, seed: int = 1):
        if n_rows < 2 or n_cols < 2 or n_rows % 2 or n_cols % 2:
            raise ValueError("oracle lattice needs even N, M >= 2")
        self.N, self.M, self.seed = int(n_rows), int(n_cols), int(seed)
        self.ny = self.M // 2
        self.black = np.ones((self.N, self.ny), dtype=np.int8)
        self.white = np.ones((self.N, self.ny), dtype=np.int8)
        self.t = 0
        self.beta = None
        self.rule = RULE_METROPOLIS

    def _args(self):
        return (_p(self.black, ctypes.c_int8), _p(self.white, ctypes.c_int8), self.N, self.ny)

    def init_random(self):
        b, w, nx, ny = self._args()
        lib().oracle_init_random(b, w, nx, ny, self.seed)
        self.t = 0
        return self

    def init_cold(self):
        b, w, nx, ny = self._args()
        lib().oracle_init_cold(b, w, nx, ny)
        self.t = 0
        return self

    def set_beta(self, beta: float, rule: int = RULE_METROPOLIS):
        self.beta, self.rule = float(beta), int(rule)
        return self

    def load_full(self, full: np.ndarray, t: int = 0):
        full = np.ascontiguousarray(full, dtype=np.int8)
        assert full.shape == (self.N, self.M)
        lib().oracle_from_full(_p(full, ctypes.c_int8), _p(self.black, ctypes.c_int8),
                               _p(self.white, ctypes.c_int8), self.N, self.ny)
        self.t = int(t)
        return self

    def sweep(self, n: int = 1):
        assert self.beta is not None
        b, w, nx, ny = self._args()
        lib().oracle_sweep(b, w, nx, ny, self.seed, self.t, int(n), self.beta, self.rule)
        self.t += int(n)
        return self

    def full(self) -> np.ndarray:
        out = np.empty((self.N, self.M), dtype=np.int8)
        b, w, nx, ny = self._args()
        lib().oracle_full_lattice(b, w, nx, ny, _p(out, ctypes.c_int8))
        return out

    def observables(self) -> tuple[int, int]:
        up = ctypes.c_int64()
        E = ctypes.c_int64()
        b, w, nx, ny = self._args()
        lib().oracle_observables(b, w, nx, ny, ctypes.byref(up), ctypes.byref(E))
        return int(up.value), int(E.value)

    def chain(self, nsweeps: int) -> tuple[np.ndarray, np.ndarray]:
        """Run nsweeps sweeps, returning (up, E) after each."""
        assert self.beta is not None
        ups = np.empty(int(nsweeps), dtype=np.int64)
        Es = np.empty(int(nsweeps), dtype=np.int64)
        b, w, nx, ny = self._args()
        lib().oracle_chain(b, w, nx, ny, self.seed, self.t, int(nsweeps), self.beta, self.rule,
                           _p(ups, ctypes.c_int64), _p(Es, ctypes.c_int64))
        self.t += int(nsweeps)
        return ups, Es

    def nn_sum(self, is_black: bool, i: int, j: int) -> int:
        op = self.white if is_black else self.black
        return int(lib().oracle_nn_sum(_p(op, ctypes.c_int8), int(bool(is_black)), self.N,
                                       self.ny, i, j))
