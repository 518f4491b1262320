cd ${GRAFT_REPO_ROOT:-.}
for v in "" "BC_TMEM_TEAM=2"; do
echo "== M156 bicg $v"; env $v REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
echo "== M312 bicgstab $v"; env $v SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
echo "== M312 bicg $v"; env $v SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
done
