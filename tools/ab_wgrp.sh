#!/bin/bash
# A/B of k_greedy_wgrp88 build variants on the GPU box (run under gpurun):
#   tools/ab_wgrp.sh name1 "-DFOO=1" name2 "-DBAR=1" ...
# each variant: rebuild, the large-D bit-identity/oracle tests, C5 probe (128 tasks)
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  NS_NVCC_EXTRA="$defs" python -m paper_2305_01868_b200.build --force > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  echo "== $name ($defs)"
  timeout 600 python -m pytest -x -q tests/test_gpu_fullsize.py -k "grouped or batched or fixture" 2>&1 | grep -E "passed|failed|Error|assert" | head -5
  timeout 600 python tools/c5_probe.py ${TASKS:-128} 2>&1 | tail -1
done
python -m paper_2305_01868_b200.build --force > /dev/null 2>&1
