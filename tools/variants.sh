cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\|^$" | tail -4
timeout 900 python tools/compare_strategies.py 20000 156 2>&1 | grep "block-cells(N)" | head -1
echo "== M312 bicgstab"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
