"""Executed warp-instructions by opcode (and the top basic blocks) from an ncu report's SASS source page:
python scripts/ncu_ops.py rep.ncu-rep [kernel-block-index]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
rows = list(csv.reader(io.StringIO("\n".join(lines[heads[kb] + 1:heads[kb + 1]]))))
h = rows[0]
X = h.index("Instructions Executed")
ops = collections.Counter()
tot = 0
for r in rows[1:]:
    if len(r) != len(h) or not r[X]:
        continue
    n = float(r[X])
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0] if src else "?"
    ops[op] += n
    tot += n
print(f"total warp-instructions {tot:.0f}")
for op, n in ops.most_common(40):
    print(f"{100 * n / tot:5.1f}% {n:12.0f} {op}")
