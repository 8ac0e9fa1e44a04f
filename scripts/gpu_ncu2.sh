cd $GRAFT_REPO_ROOT
M2=gpurun_out/m3; mkdir -p $M2
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed"
ncu --set full --clock-control none --kernel-name-base demangled -k regex:"backward4_kernel<float, .bool.0, .bool.0" -s 1 -c 1 -o $M2/full_c3f_backward -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:contract_tc -s 1 -c 1 -o $M2/full_c3f_grads -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
for f in $M2/full_c3f_backward.ncu-rep $M2/full_c3f_grads.ncu-rep; do ncu -i $f --page raw --csv --metrics $M > ${f%.ncu-rep}.csv 2>/dev/null; done
