cd ${GRAFT_REPO_ROOT:-.}
for v in "" "BC_YST_WEIGHT=3" "BC_YST_WEIGHT=4" "BC_ANNEAL_ITERS=600000" "BC_YRD_WEIGHT=2 BC_YST_WEIGHT=3"; do
  echo "== M156 bicgstab $v"; env $v REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== M156 bicg $v"; env $v REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
done
