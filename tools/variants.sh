cd ${GRAFT_REPO_ROOT:-.}
echo "== M156 bicgstab"; REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
echo "== M156 bicg"; REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
echo "== M312 bicgstab"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
