cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ct_t.log 2>&1
for c in c1 c2 c3 c4; do timeout 120 python scripts/ab_phases.py --config $c --modes unfused 2>&1 | tail -1 >> gpurun_out/ct_ab.log; done
for c in c1 c4; do SDTW_CONTRACT_SIMT=1 timeout 120 python scripts/ab_phases.py --config $c --modes unfused 2>&1 | tail -1 >> gpurun_out/ct_ab.log; done
timeout 300 python bench.py --config c5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300 >> gpurun_out/ct_ab.log
SDTW_CONTRACT_SIMT=1 timeout 300 python bench.py --config c5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300 >> gpurun_out/ct_ab.log
