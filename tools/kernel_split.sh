#!/bin/bash
# per-kernel device time of a C5 probe run (ncu launch list; run under gpurun): tools/kernel_split.sh [tasks]
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split_launches.csv \
    python tools/c5_probe.py ${1:-128} > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open("gpurun_out/split_launches.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r); H = rows[h]
ik, iv = H.index("Kernel Name"), H.index("Metric Value")
t = collections.defaultdict(float); n = collections.Counter()
for r in rows[h + 1:]:
    if len(r) > iv and r[iv]:
        t[r[ik][:50]] += float(r[iv].replace(",", "")); n[r[ik][:50]] += 1
for k, v in sorted(t.items(), key=lambda kv: -kv[1])[:12]: print(f"{k:52s} {n[k]:4d} {v / 1e6:9.3f} ms")
PY
