cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for n in 100 1000 2000 100000; do
  echo "== M156 bicgstab $n cells"; REPS=3 timeout 200 python tools/prof_block.py $n 2>&1 | tail -1
done
echo "== M156 bicg 100 cells"; REPS=3 timeout 200 python tools/prof_block.py 100 bicg 2>&1 | tail -1
