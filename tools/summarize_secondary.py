"""gpurun_out/sec_<kernel>.ncu-rep (tools/prof_secondary.sh) -> profiles/r2_secondary_ncu.json:
per kernel the duration, DRAM bytes, pipe activity, occupancy and issue of one launch."""
import csv
import glob
import io
import json
import os
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = []
for f in sorted(glob.glob("gpurun_out/sec_*.ncu-rep")):
    txt = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(txt)))
    if len(rd) < 3:
        continue
    h, u, r = rd[0], rd[1], rd[2]
    d = {"kernel": r[h.index("Kernel Name")], "capture": os.path.basename(f)}
    for k in KEYS:
        if k in h:
            d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
    out.append(d)
json.dump(out, open("profiles/r2_secondary_ncu.json", "w"), indent=1)
for d in out:
    print(d["kernel"][:60], "|", d.get("gpu__time_duration.sum"), "| DRAM r", d.get("dram__bytes_read.sum"),
          "w", d.get("dram__bytes_write.sum"), "| tensor", d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
          "| issue", d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"), "| L2", d.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"))
