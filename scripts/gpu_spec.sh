cd $GRAFT_REPO_ROOT
for r in -100 0 1 2 3; do for c in c1 c2 c3; do SDTW_BWD_SPEC_RIGHT=$r timeout 120 python scripts/ab_phases.py --config $c --modes unfused 2>&1 | tail -1 | sed "s/^/spec=$r /" >> gpurun_out/spec.log; done; done
