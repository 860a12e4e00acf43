"""Turn a tools/prof_all.sh run (gpurun_out/) into the tracked profiles/ files.

    python tools/summarize_profiles.py TAG [OUT_TAG]

reads  gpurun_out/launches_TAG.csv  (ncu --metrics gpu__time_duration.sum launch list)
       gpurun_out/full_TAG.ncu-rep  (ncu --set full of the top kernels)
writes profiles/OUT_TAG_launches.csv, profiles/OUT_TAG_ncu_full_metrics.json,
       profiles/greedy_traffic.json (DRAM bytes per launch of the grouped greedy,
       read by bench.py for the roofline "traffic" field)
and prints the launch-share table (markdown) for the summary.
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def launches(tag):
    rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= iv or not r[iv]:
            continue
        name = r[ik]
        if "ns::" not in name and "k_" not in name:
            continue   # torch / flush kernels are not library kernels
        tot[name] += float(r[iv].replace(",", ""))
        cnt[name] += 1
    return tot, cnt


def full_metrics(tag):
    out = subprocess.run(["ncu", "-i", f"gpurun_out/full_{tag}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    h, units = rd[0], rd[1]
    res = []
    for r in rd[2:]:
        d = {"Kernel Name": r[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                d[m] = r[h.index(m)]
        d["units"] = {m: units[h.index(m)] for m in METRICS if m in h}
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    out_tag = sys.argv[2] if len(sys.argv) > 2 else tag
    shutil.copy(f"gpurun_out/launches_{tag}.csv", f"profiles/{out_tag}_launches.csv")
    tot, cnt = launches(tag)
    s = sum(tot.values())
    unit = "ns"
    print("| kernel | launches | total ms | share of library time |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / s:.3f} |")
    fm = full_metrics(tag)
    json.dump(fm, open(f"profiles/{out_tag}_ncu_full_metrics.json", "w"), indent=1)
    for d in fm:
        u = d["units"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        print(f"{d['Kernel Name']}: {d['gpu__time_duration.sum']} {u['gpu__time_duration.sum']}, "
              f"regs {d['launch__registers_per_thread']}, warps {float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f}%, "
              f"issue {float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f}%, "
              f"fp64 {float(d['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']):.1f}%, "
              f"dmma {float(d.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0)):.1f}%, "
              f"DRAM {dram / 1e6:.0f} MB")
    # the large-D greedy is three kernels per launch: phase 1, phase 2, replay --
    # the first consecutive triple of the capture (one beam level)
    names = [d["Kernel Name"] for d in fm]
    parts = ("k_greedy_wgrp88", "k_greedy_p2", "k_greedy_replay")
    for i in range(len(fm) - 2):
        if all(parts[k] in names[i + k] for k in range(3)):
            tot_b, per = 0.0, {}
            for d in fm[i:i + 3]:
                u = d["units"]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                b = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                per[d["Kernel Name"].split("(")[0]] = b
                tot_b += b
            json.dump({"kernel": " + ".join(parts), "bytes_per_launch": tot_b, "per_kernel": per,
                       "source": f"ncu --set full, profiles/{out_tag}_ncu_full_metrics.json "
                                 "(dram__bytes_read.sum + dram__bytes_write.sum of one launch each of the three "
                                 "kernels of one beam level of the bench's headline step)"},
                      open("profiles/greedy_traffic.json", "w"), indent=1)
            break

if __name__ == "__main__":
    main()
