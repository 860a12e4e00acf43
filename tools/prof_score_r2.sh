#!/bin/bash
# ns_score_plans profile pack (run under gpurun): ncu --set full of one C3
# launch each of the tcgen05 pooling (k_pool_tc) and the comm MLP chain
# (k_plan_mlp_tc) at 2^20 plans (tools/bench_score.py order: C2 fp64, C2
# SIMT-pooled TF32X3, C2 TF32X3, C3 ...; 6 launches per mode).
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pool_tc" -s 6 -c 1 \
    -o gpurun_out/score_pool_r2 python tools/bench_score.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plan_mlp_tc" -s 36 -c 2 \
    -o gpurun_out/score_mlp_r2 python tools/bench_score.py > /dev/null 2>&1
