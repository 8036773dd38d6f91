timeout 900 bash tools/profile.sh D r02 sched_kernelILi0ELi1E > gpurun_out/profile_D.txt 2>&1; echo profile=$?
ncu -i gpurun_out/prof_D_r02.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/src_D_r02.csv 2>/dev/null; echo src=$?
ncu -i gpurun_out/prof_D_r02.ncu-rep --page source --csv > gpurun_out/srccuda_D_r02.csv 2>/dev/null; echo src2=$?
