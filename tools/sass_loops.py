"""Instruction mix of the innermost loops of one kernel (backward branches), from cuobjdump -sass.
python tools/sass_loops.py LIB.so MANGLED_NAME"""
import re
import subprocess
import sys
from collections import Counter

lib, fn = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
lines, on = [], False
for ln in sass.splitlines():
    if "Function :" in ln:
        on = ln.split("Function :")[1].strip() == fn
        continue
    if on and re.match(r"\s+/\*[0-9a-f]+\*/", ln):
        lines.append(ln)
addr = [int(re.search(r"/\*([0-9a-f]+)\*/", l).group(1), 16) for l in lines]
loops = []
for i, l in enumerate(lines):
    m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", l)
    if m and int(m.group(1), 16) < addr[i]:
        loops.append((int(m.group(1), 16), addr[i]))
for lo, hi in sorted(set(loops), key=lambda x: x[1] - x[0]):
    body = [l for a, l in zip(addr, lines) if lo <= a <= hi]
    c = Counter(re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", l).group(1).split(".")[0]
                for l in body)
    if c.get("IMAD", 0) < 50:
        continue
    print(f"loop {lo:#x}-{hi:#x}: {len(body)} instructions;", ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
if len(sys.argv) > 3:  # full opcodes of the innermost qualifying loop
    lo, hi = sorted(set(loops), key=lambda x: x[1] - x[0])[[i for i, (a, b) in enumerate(sorted(set(loops), key=lambda x: x[1] - x[0])) if sum(1 for ad, l in zip(addr, lines) if a <= ad <= b and "IMAD" in l) >= 50][0]]
    body = [l for a, l in zip(addr, lines) if lo <= a <= hi]
    c = Counter(re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", l).group(1) for l in body)
    print("  ", ", ".join(f"{k} {v}" for k, v in c.most_common(30)))
