"""Per-CUDA-source-line instruction / stall summary of an ncu report (kernel regex)."""
import csv, subprocess, sys
from collections import defaultdict
rep, steps = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr_idx = [i for i, x in enumerate(r) if x and x[0] == 'Line No']
file_of = {}
fname = None
per_line = defaultdict(lambda: [0, 0, ''])
for i, x in enumerate(r):
    if x and x[0] == 'File Path':
        fname = x[1].split('/')[-1]
    file_of[i] = fname
for hi_, start in enumerate(hdr_idx):
    h = r[start]
    ex = h.index('Instructions Executed'); ws = h.index('Warp Stall Sampling (All Samples)')
    end = hdr_idx[hi_ + 1] if hi_ + 1 < len(hdr_idx) else len(r)
    cur = None
    for x in r[start + 1:end]:
        if len(x) <= ex: continue
        if x[0] and x[0].isdigit():
            cur = (file_of[start], int(x[0])); per_line[cur][2] = x[1][:80]
        if cur is None: continue
        try:
            per_line[cur][0] += int(x[ex] or 0); per_line[cur][1] += int(x[ws] or 0)
        except ValueError:
            pass
tots = sum(v[1] for v in per_line.values())
for k, v in sorted(per_line.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{k[0][:14]:14s}:{k[1]:5d} {v[0]/steps:7.1f} inst/unit {100*v[1]/tots:5.1f}% stall  {v[2]}")
