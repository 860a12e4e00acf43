# ns_score_plans pooling on tcgen05: parity tests, throughput, ncu of the TF32X3 kernels (run under gpurun)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "tf32x3 or pool_tcgen05 or score or reading" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
timeout 300 python tools/bench_score.py > gpurun_out/bs2.log 2>&1
#timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plan_mlp_tc" -s 14 -c 1 -o gpurun_out/score_tc python tools/bench_score.py > gpurun_out/ncu_score.log 2>&1
