#!/bin/bash
# Build library variants (compile-time macros) into _variants/lib_<name>.so for tools/variants.sh.
# usage: tools/build_variants.sh name1 "-DFOO" name2 "-DBAR -DBAZ" ...
set -e
mkdir -p _variants
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  NS_NVCC_EXTRA="$defs" python -m paper_2305_01868_b200.build --force > /dev/null
  cp paper_2305_01868_b200/libneuroshard.so _variants/lib_$name.so
  grep -A4 "Compiling entry function .*k_greedy_dedupILi8ELi16" paper_2305_01868_b200/_build/k_search.cu.ptxas.txt | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr "\n" " " | sed "s/^/$name: /"
done
python -m paper_2305_01868_b200.build --force > /dev/null
