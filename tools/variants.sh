# bench variants of the scheduler library: bash tools/variants.sh <workload> <lib suffixes...>
W=$1; shift
for v in "$@"; do
  SS_B200_LIB=paper_2506_12204_b200/_lib/libss_$v.so timeout 300 python bench.py --workload $W --steps 3 --warmup 1 --no-e2e --no-cpu > gpurun_out/var_${W}_$v.json 2>/dev/null; echo $v=$?
done
