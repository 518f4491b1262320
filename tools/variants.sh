cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "BC_YRD_WEIGHT=2"; do
  echo "== M156 bicgstab $v"; env $v REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== M156 bicg $v"; env $v REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
done
for v in "" "BC_COPY1_SHIFT=0"; do
  echo "== M312 bicgstab $v"; env $v SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== M312 bicg $v"; env $v SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
done
