# A/B timing of library builds under _variants/ (bench workload, device-resident step)
for v in ${VARIANTS:-b4 c}; do cp _variants/lib_$v.so paper_2305_01868_b200/libneuroshard.so; python bench.py --no-secondary --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['kernels_ms_per_step'])"; done
