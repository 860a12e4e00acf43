"""Per-source-line instructions per unit and stall share of one kernel in an ncu report (KREGEX, default greedy)."""
import csv, os, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 16384 * 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + os.environ.get("KREGEX", "greedy")],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = next(x for x in r if x and x[0] == "Line No")
ex, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
d = defaultdict(lambda: [0, 0])
cur = None
fname = None
for x in r:
    if x and x[0] == "File Path":
        fname = x[1].split("/")[-1]
    if len(x) <= ex or x[0] == "Line No":
        continue
    if x[0] and x[0].isdigit():
        cur = (fname, int(x[0]), x[1][:80])
        continue
    if x[2]:
        try:
            d[cur][0] += int(x[ex] or 0)
            d[cur][1] += int(x[ws] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in d.values())
st = sum(v[1] for v in d.values())
print(f"total {tot / steps:.1f} inst/step")
for k, v in sorted(d.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{k[0][:12]:12s}:{k[1]:5d} {v[0] / steps:7.1f} inst/step {100 * v[1] / st:5.1f}% stall  {k[2]}")
