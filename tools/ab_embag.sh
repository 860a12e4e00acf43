#!/bin/bash
# A/B of embedding-bag build variants (run under gpurun): tools/ab_embag.sh name "-DFOO" ...
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  NS_NVCC_EXTRA="$defs" python -m paper_2305_01868_b200.build --force > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  echo "== $name ($defs)"
  timeout 300 python -m pytest -q -x tests/test_gpu_embag.py 2>&1 | tail -1
  timeout 300 python tools/embag_probe.py 0 1.0 2>&1 | cut -c1-60
done
python -m paper_2305_01868_b200.build --force > /dev/null 2>&1
