"""Top SASS lines by warp-stall samples from an ncu report:
python scripts/ncu_hot.py rep.ncu-rep [kernel-block-index] [n]   (block = n-th profiled kernel in the report)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
print(lines[heads[kb]][:120])
block = lines[heads[kb] + 1:heads[kb + 1]]
rows = list(csv.reader(io.StringIO("\n".join(block))))
h = rows[0]
S = h.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in rows[1:] if len(r) == len(h)]
tot = sum(float(r[S] or 0) for r in data)
print(f"total samples {tot:.0f}")
for k, r in sorted(enumerate(data), key=lambda kr_: -float(kr_[1][S] or 0))[:n]:
    s = float(r[S] or 0)
    top = sorted(((float(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}% {k:5d} {r[1].strip()[:60]:60s} " + " ".join(f"{nm}={v:.0f}" for v, nm in top if v > 0))
