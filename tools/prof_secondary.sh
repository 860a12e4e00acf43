#!/bin/bash
# ncu --set full of one launch of each secondary kernel (run under gpurun)
ncu --set full --clock-control none --import-source on \
    -k regex:"k_plan_mlp_tc|k_pool_staged|k_pt_compute_grad|k_pt_comm_grad|k_pt_adam|k_bag_forward|k_bag_backward_sgd|k_pt_place|k_bag_hot_detect" \
    --launch-count 1 -o gpurun_out/full_r2sec python tools/prof_secondary.py > gpurun_out/prof_sec.log 2>&1
# one launch per kernel name: ncu's --launch-count applies per filter match, so re-run per kernel
for k in k_plan_mlp_tc k_pool_staged k_pt_compute_grad k_pt_comm_grad k_bag_forward k_bag_backward_sgd_hot k_bag_hot_detect; do
  ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/sec_$k python tools/prof_secondary.py > /dev/null 2>&1
done
ls gpurun_out
