"""Summarise tools/scan.py outputs (§5.3, Figs. 5 and 6 method): pairwise Binder
crossings U_L(T) = U_2L(T) near Tc (conventional U = 1 - <m^4> / (3 <m^2>^2), reading R15),
and <|m|>, E/site against Onsager's exact solution.

    python tools/scan_analysis.py gpurun_out/scan_L64.json ... > profiles/r01_scan_long.md
"""
import json
import math
import sys

from scipy.special import ellipk  # noqa: E402

TC = 2.0 / math.log(1.0 + math.sqrt(2.0))


def onsager_m(T):
    """Spontaneous magnetisation (reading R14: exact Tc as the cut-off)."""
    return 0.0 if T >= TC else (1.0 - math.sinh(2.0 / T) ** -4) ** 0.125


def onsager_u(T):
    """Energy per site of the infinite lattice, J = 1 (Onsager 1944):
    u = -coth(2b) [1 + (2/pi) (2 tanh^2(2b) - 1) K(k)], k = 2 sinh(2b) / cosh^2(2b)."""
    b = 1.0 / T
    k = 2.0 * math.sinh(2 * b) / math.cosh(2 * b) ** 2
    return -(1.0 / math.tanh(2 * b)) * (1 + 2 / math.pi * (2 * math.tanh(2 * b) ** 2 - 1) * ellipk(k * k))
U_STAR = 0.61069  # Binder cumulant at Tc for L -> inf (literature; reading R15)


def crossing(a, b):
    """Linear interpolation of the sign change of U_b - U_a over the common temperatures."""
    ta = {r["T"]: r for r in a}
    tb = {r["T"]: r for r in b}
    ts = sorted(set(ta) & set(tb))
    for t0, t1 in zip(ts, ts[1:]):
        d0 = tb[t0]["binder"] - ta[t0]["binder"]
        d1 = tb[t1]["binder"] - ta[t1]["binder"]
        if d0 > 0 >= d1:
            f = d0 / (d0 - d1)
            tc = t0 + f * (t1 - t0)
            u = ta[t0]["binder"] + f * (ta[t1]["binder"] - ta[t0]["binder"])
            return tc, u
    return None


def main(paths):
    rows = []
    for p in paths:
        rows += json.load(open(p))
    by_l = {}
    for r in rows:
        by_l.setdefault(r["L"], []).append(r)
    print("# GPU temperature scans\n")
    print(f"Tc = {TC:.6f}, U* = {U_STAR} (L -> inf). Chains: `tools/scan.py` / `tools/scan_long.sh` "
          "(cold starts, device-side measured chains).\n")
    print("## Binder cumulant U_L(T)\n")
    ts = sorted({r["T"] for r in rows if "binder" in r})
    ls = sorted(by_l)
    print("| T | " + " | ".join(f"U_{l}" for l in ls) + " |")
    print("|---|" + "---|" * len(ls))
    for t in ts:
        cells = []
        for l in ls:
            r = next((x for x in by_l[l] if x["T"] == t), None)
            if r is None:
                cells.append("")
            elif "binder_se" in r:
                cells.append(f"{r['binder']:.4f} ± {r['binder_se']:.4f}")
            else:
                cells.append(f"{r['binder']:.4f}")
        print(f"| {t} | " + " | ".join(cells) + " |")
    print("\n## Pairwise crossings\n")
    print("| L, 2L | T_cross | U at crossing | T_cross - Tc |")
    print("|---|---|---|---|")
    for l in ls:
        if 2 * l in by_l:
            c = crossing(by_l[l], by_l[2 * l])
            if c:
                print(f"| {l}, {2 * l} | {c[0]:.4f} | {c[1]:.4f} | {c[0] - TC:+.4f} |")
            else:
                print(f"| {l}, {2 * l} | no sign change in range | | |")
    big = [r for r in rows if r["L"] >= 1024]
    if big:
        print("\n## Magnetisation and energy against Onsager\n")
        print("| L | T | <\\|m\\|> | Onsager M(T) | diff | E/site | Onsager u(T) | diff |")
        print("|---|---|---|---|---|---|---|---|")
        for r in sorted(big, key=lambda x: (x["L"], x["T"])):
            m_ex = onsager_m(r["T"])
            u_ex = onsager_u(r["T"])
            print(f"| {r['L']} | {r['T']} | {r['abs_m']:.5f} | {m_ex:.5f} | {r['abs_m'] - m_ex:+.5f} | "
                  f"{r['E_site']:.5f} | {u_ex:.5f} | {r['E_site'] - u_ex:+.5f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
