for v in minb5 minb6 minb8; do
  SS_B200_LIB=paper_2506_12204_b200/_lib/libss_$v.so timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > gpurun_out/var_$v.json 2>/dev/null; echo $v=$?
done
