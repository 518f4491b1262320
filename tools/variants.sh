cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\|^$" | tail -8
REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
timeout 900 python tools/compare_strategies.py 100000 156 > /dev/null 2>&1; cp gpurun_out/strategies_m156.json gpurun_out/strategies_m156_v4.json
timeout 900 python tools/compare_strategies.py 100000 312 > /dev/null 2>&1; cp gpurun_out/strategies_m312.json gpurun_out/strategies_m312_v4.json
