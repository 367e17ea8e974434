"""Readers for the cited text fixtures under tests/golden/ (no method arithmetic)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln


def philox_kat():
    out = []
    for ln in lines("philox4x32_10_kat.txt"):
        lhs, rhs = ln.split("->")
        w = [int(x, 16) for x in lhs.split()]
        o = [int(x, 16) for x in rhs.split()]
        out.append((w[:4], w[4:6], o))
    return out


def fig3():
    out = []
    for ln in lines("fig3_multispin_layout.txt"):
        lhs, rhs = ln.split("->")
        toks = lhs.split()
        out.append((toks[0], [int(x) for x in toks[1:]], sorted(int(x) for x in rhs.split())))
    return out


def dos4x4():
    return {int(a): int(b) for a, b in (ln.split() for ln in lines("torus4x4_exact.txt"))}


def rng_contract():
    draws, inits, init4 = [], [], []
    for ln in lines("rng_contract.txt"):
        lhs, rhs = ln.split("->")
        toks = lhs.split()
        if toks[0] == "draw":
            draws.append(([int(x) for x in toks[1:]], [int(x, 16) for x in rhs.split()]))
        elif toks[0] == "init":
            r = rhs.split()
            inits.append(([int(x) for x in toks[1:]], int(r[0]), int(r[1]), r[2]))
        elif toks[0] == "init4x4":
            rows = [[int(x) for x in row.split()] for row in rhs.split("|")]
            init4.append((int(toks[1]), rows))
    return draws, inits, init4
