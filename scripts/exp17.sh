python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c1 c2 c4; do python scripts/prof_step.py $c unfused 4 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$c grads', round(d['grads'],4))"; done
