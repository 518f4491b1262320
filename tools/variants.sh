cd ${GRAFT_REPO_ROOT:-.}
for v in "" "BC_TMEM_WARPS=12"; do
echo "== M156 bicgstab $v"; env $v REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
done
