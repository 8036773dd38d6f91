# e2e (host-buffer call) of library variants: bash tools/e2e_variants.sh <workload> <lib suffixes...>
W=$1; shift
for v in "$@"; do
  SS_B200_LIB=paper_2506_12204_b200/_lib/libss_$v.so timeout 600 python bench.py --workload $W --steps 3 --warmup 1 --no-cpu > gpurun_out/e2e_${W}_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_${W}_$v.json')); print('$W $v', round(d['ms_per_step'], 2), round(d['e2e']['ms_per_step'], 2))"
done
