#!/bin/bash
# Round profile pack: launch list (share of the step) + ncu --set full of the three top kernels.
tag=${1:-r1}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 1 --profile-run --no-e2e --no-secondary > gpurun_out/launches_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_greedy|k_precompute|k_plan_cost" -s 3 -c 3 \
  -o gpurun_out/full_${tag} python bench.py --steps 1 --warmup 1 --profile-run --no-e2e --no-secondary > gpurun_out/full_${tag}.log 2>&1
