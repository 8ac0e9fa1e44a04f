python -m pytest tests -m gpu -q 2>&1 | tail -2
for c in c1 c2 c3; do python scripts/prof_step.py $c fused 4 2>&1 | tail -1; done
