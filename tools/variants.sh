cd ${GRAFT_REPO_ROOT:-.}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "== M312 bicgstab"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
echo "== M156 bicgstab"; REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
timeout 900 python tools/compare_strategies.py 20000 156 2>&1 | grep "block-cells(N)" | head -4
