#!/bin/bash
# One GPU session's measurements of HEAD (run under gpurun):
#   gpurun -- 'bash tools/measure_round.sh <tag>'
# -> gpurun_out/m_<tag>/: bench lines of every workload (full default runs,
#    e2e + CPU baseline), the reference arm, issue-rate ncu profiles
#    (ncu_issue_<W>.json, read by bench.py's roofline), the launch list and one
#    ncu --set full capture of config B's and D's scheduler kernel, the
#    section timing of B and D (debug build, if present).
set -u
TAG=${1:-head}
O=gpurun_out/m_$TAG
mkdir -p $O
python tools/ncu_issue.py B D E A > $O/ncu_issue.log 2>&1; echo ncu_issue=$?
for W in A B D E; do cp gpurun_out/ncu_issue_$W.json profiles/ 2>/dev/null; cp gpurun_out/ncu_issue_$W.json $O/ 2>/dev/null; done
for W in B A C D E audit; do
  timeout 900 python bench.py --workload $W > $O/bench_$W.json 2> $O/bench_$W.err; echo bench_$W=$?
done
timeout 900 python bench.py --impl reference > $O/ref_arm_B.json 2> $O/ref_arm_B.err; echo ref_arm=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/ncu_launches_B.csv python bench.py --workload B --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
echo launches=$?
for WK in "B sched_kernelILi0ELi13E" "D sched_kernelILi0ELi1E"; do
  set -- $WK
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$2 -c 1 \
      -o $O/prof_$1 -f python bench.py --workload $1 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  echo full_$1=$?
done
if [ -f paper_2506_12204_b200/_lib/libss_dbgtime.so ]; then
  for W in B D; do python tools/section_timing.py $W > $O/section_timing_$W.txt 2>&1; done
fi
