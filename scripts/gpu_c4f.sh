cd $GRAFT_REPO_ROOT
for c in c4 c1; do timeout 200 python scripts/ab_phases.py --config $c --modes fused 2>&1 | tail -1 >> gpurun_out/c4f_ab.log; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/c4f_t.log 2>&1
