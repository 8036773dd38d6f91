#!/bin/bash
# Profiles committed under profiles/<round>/ are made with this script (run under gpurun):
#   gpurun -- 'bash tools/profile.sh B r01 [kernel-regex]'
# 1) launch list of one bench run (cold-cache, serialised: compare shares)
# 2) one `ncu --set full` capture of the scheduler kernel (source-level stalls).
# Semantic runs launch two scheduler variants and the unselected one exits at
# once: the regex names the selected one by its mangled name, e.g.
# sched_kernelILi0ELi13E (semantic, digest, chunked, no eviction; config B/E), ILi0ELi5E (chunked, evicting; forced) or
# sched_kernelILi0ELi1E (semantic, digest, per-round; config D).
set -u
W=${1:-B}; R=${2:-r01}; K=${3:-sched_kernelILi0ELi13E}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/ncu_launches_${W}_${R}.csv \
    python bench.py --workload $W --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_run_${W}.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s 1 -c 1 \
    -o gpurun_out/prof_${W}_${R} -f \
    python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_run_${W}.log 2>&1
echo full=$?
