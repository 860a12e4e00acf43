#!/bin/bash
# A/B of single-task (latency) builds on the GPU box: tools/ab_wide.sh name "-DFOO" ...
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  NS_NVCC_EXTRA="$defs" python -m paper_2305_01868_b200.build --force > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  echo "== $name ($defs)"
  timeout 600 python -m pytest -x -q tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "wide or bit_identical or C5 or fixture" 2>&1 | grep -E "passed|failed|Error|assert" | head -5
  timeout 600 python tools/prof_latency.py C5 C4 2>&1 | tail -4
done
python -m paper_2305_01868_b200.build --force > /dev/null 2>&1
