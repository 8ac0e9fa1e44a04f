# Round measurement (round 2): tests, bench lines for every config, launch
# list, ncu --set full captures of the dominant kernels, MUFU microbenchmark
# (outputs in gpurun_out/m2/; summaries are copied into profiles/ by hand).
set -x
M2=gpurun_out/m3
mkdir -p $M2
python -m pytest tests -m gpu -q > $M2/gputests.log 2>&1; tail -3 $M2/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $M2/smoke.log 2>&1; tail -1 $M2/smoke.log
python bench.py > $M2/bench_c3_default.json 2> $M2/bench_c3_default.err
python bench.py --impl reference > $M2/bench_reference.json 2> $M2/bench_reference.err
for c in c1 c2 c4 c5; do
  python bench.py --config $c --mode unfused --no-cpu-baseline > $M2/bench_${c}.json 2> $M2/bench_${c}.err
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $M2/mufu_rate scripts/micro/mufu_rate.cu && $M2/mufu_rate > $M2/mufu_r2.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $M2/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none -k regex:forward_tc -s 1 -c 1 -o $M2/full_c3f_forward -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
ncu --set full --clock-control none --kernel-name-base demangled -k regex:"backward4_kernel<float, .bool.0, .bool.0" -s 1 -c 1 -o $M2/full_c3f_backward -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:cost_gemm -s 1 -c 1 -o $M2/full_c3_costs -f python scripts/prof_step.py c3 unfused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:forward3 -s 1 -c 1 -o $M2/full_c3_forward -f python scripts/prof_step.py c3 unfused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:contract_tc -s 1 -c 1 -o $M2/full_c3f_grads -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg,sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed"
for f in $M2/full_*.ncu-rep; do ncu -i $f --page raw --csv --metrics $M > ${f%.ncu-rep}.csv 2>/dev/null; done
ls -la $M2
