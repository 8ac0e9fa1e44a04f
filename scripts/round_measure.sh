# Round measurement: tests, bench lines for every config, launch list and
# ncu --set full captures of the dominant kernels (outputs in gpurun_out/).

mkdir -p gpurun_out/m
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/m/bench_c2_default.json 2> gpurun_out/m/bench_c2_default.err
python bench.py --impl reference > gpurun_out/m/bench_reference.json 2> gpurun_out/m/bench_reference.err
python bench.py --config c1 --no-cpu-baseline > gpurun_out/m/bench_c1.json 2>&1
python bench.py --config c3 --no-cpu-baseline > gpurun_out/m/bench_c3_unfused.json 2>&1
python bench.py --config c3 --mode fused --single-mode --no-cpu-baseline > gpurun_out/m/bench_c3_fused.json 2>&1
python bench.py --config c4 --no-cpu-baseline > gpurun_out/m/bench_c4.json 2>&1
python bench.py --config c5 --no-cpu-baseline > gpurun_out/m/bench_c5.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed"
ncu --set full --clock-control none -k regex:backward4 -s 1 -c 1 -o gpurun_out/m/full_c2_backward -f python scripts/prof_step.py c2 unfused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:forward3 -s 1 -c 1 -o gpurun_out/m/full_c3_forward -f python scripts/prof_step.py c3 unfused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:forward_tc -s 1 -c 1 -o gpurun_out/m/full_c3f_forward -f python scripts/prof_step.py c3 fused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:contract_ordered -s 1 -c 1 -o gpurun_out/m/full_c4_grads -f python scripts/prof_step.py c4 unfused 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:cost_gemm -s 1 -c 1 -o gpurun_out/m/full_c3_costs -f python scripts/prof_step.py c3 unfused 2 > /dev/null 2>&1
for f in gpurun_out/m/full_*.ncu-rep; do ncu -i $f --page raw --csv --metrics $M > ${f%.ncu-rep}.csv 2>/dev/null; done
for f in gpurun_out/m/full_c3*.ncu-rep gpurun_out/m/full_c4*.ncu-rep; do rm -f $f; done
ls -la gpurun_out/m
