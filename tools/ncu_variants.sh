#!/bin/bash
# ncu --set full capture of the selected scheduler kernel for library variants:
#   bash tools/ncu_variants.sh <workload> <kernel-regex> <lib suffix|default>...
W=$1; K=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="SS_B200_LIB=paper_2506_12204_b200/_lib/libss_$v.so"; fi
  env $L timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -c 1 \
      -o gpurun_out/prof_${W}_$v -f python bench.py --workload $W --steps 1 --warmup 0 --no-e2e --no-cpu \
      > gpurun_out/ncu_${W}_$v.log 2>&1
  echo $v=$?
done
