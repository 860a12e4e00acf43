#!/bin/bash
# Profile pack of the bench step (run under gpurun): bench line, ncu launch
# list of the step, ncu --set full of the top kernels (one launch each).
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; tail -1 gpurun_out/bench_r2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
    python bench.py --profile-run --steps 2 --warmup 1 --no-e2e --no-secondary --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_greedy_wgrp88|k_greedy_p2|k_greedy_replay|k_plan_cost_dmma|k_merge_order" \
    -s 60 -c 10 -o gpurun_out/full_r2 \
    python bench.py --profile-run --steps 1 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
