#!/bin/bash
# ncu full capture of one greedy launch (bench workload, fewer tasks)
out=${1:-gpurun_out/prof_greedy}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_greedy" -s 1 -c 1 -o $out \
  python bench.py --steps 1 --warmup 1 --tasks ${TASKS:-16384} --profile-run --no-e2e --no-secondary > ${out}.log 2>&1
