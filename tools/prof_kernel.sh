#!/bin/bash
# ncu full capture (with source) of one launch of the kernels matching $1 in the bench workload
# usage: tools/prof_kernel.sh REGEX OUT [TASKS]
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${SKIP:-1} -c ${COUNT:-1} -o $2 \
  python bench.py --steps 1 --warmup 1 --tasks ${3:-16384} --profile-run --no-e2e --no-secondary > ${2}.log 2>&1
