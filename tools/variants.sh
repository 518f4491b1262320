cd ${GRAFT_REPO_ROOT:-.}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
time timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
for n in 100000; do
  echo "== M156 bicgstab $n"; REPS=3 timeout 300 python tools/prof_block.py $n 2>&1 | tail -1
  echo "== M156 bicg $n"; REPS=3 timeout 300 python tools/prof_block.py $n bicg 2>&1 | tail -1
  echo "== M312 bicgstab $n"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py $n 2>&1 | tail -1
  echo "== M312 bicg $n"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py $n bicg 2>&1 | tail -1
done
