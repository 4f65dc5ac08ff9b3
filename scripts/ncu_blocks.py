"""Heaviest straight-line SASS blocks (executed warp-instructions) of one kernel in an ncu report:
python scripts/ncu_blocks.py rep.ncu-rep [kernel-block-index] [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
rows = list(csv.reader(io.StringIO("\n".join(lines[heads[kb] + 1:heads[kb + 1]]))))
h = rows[0]
X = h.index("Instructions Executed")
data = [r for r in rows[1:] if len(r) == len(h)]
blocks, cur = [], None
for i, r in enumerate(data):
    c = float(r[X] or 0)
    if cur and c == cur[1]:
        cur[2] += 1
        cur[3].append(r[1].strip())
    else:
        cur = [i, c, 1, [r[1].strip()]]
        blocks.append(cur)
tot = sum(b[1] * b[2] for b in blocks)
print(f"total {tot / 1e6:.2f}M warp-instructions")
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:n]:
    print(f"idx {b[0]:5d} exec {b[1]:9.0f} x {b[2]:3d} = {b[1] * b[2] / 1e6:6.2f}M | " + " ; ".join(x[:26] for x in b[3][:5]))
