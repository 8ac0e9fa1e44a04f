for lib in main scripts/lib_early2.so scripts/lib_early3.so scripts/lib_late2.so; do
  if [ $lib != main ]; then export SDTW_LIB=$GRAFT_REPO_ROOT/$lib; else unset SDTW_LIB; fi
  echo "== $lib"
  for c in c2 c4; do python scripts/prof_step.py $c unfused 4 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$c grads', round(d['grads'],4))"; done
done
