cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo "== M156 bicgstab"; REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
echo "== M312 bicgstab"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
echo "== M156 bicgstab 1000"; REPS=3 timeout 300 python tools/prof_block.py 1000 2>&1 | tail -1
