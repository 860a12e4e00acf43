# A/B timing of ns_score_plans across library builds under _variants/
for v in ${VARIANTS:-g2 st}; do cp _variants/lib_$v.so paper_2305_01868_b200/libneuroshard.so; echo "== $v"; python tools/bench_score.py 2>/dev/null; done
