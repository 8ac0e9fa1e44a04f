cd $GRAFT_REPO_ROOT
for w in 2 3; do for c in c2 c3; do SDTW_BWD_WIN=$w timeout 120 python scripts/ab_phases.py --config $c --modes fused,unfused 2>&1 | tail -1 | sed "s/^/win=$w /" >> gpurun_out/win.log; done; done
