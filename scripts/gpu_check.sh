set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; tail -2 gpurun_out/b_default.err
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; done
python bench.py --config c3 --mode fused --no-cpu-baseline > gpurun_out/b_c3f.json 2>gpurun_out/b_c3f.err
python bench.py --config c5 --no-cpu-baseline > gpurun_out/b_c5.json 2>gpurun_out/b_c5.err
cat gpurun_out/b_*.json | cut -c1-600
