# Kernel variant timing on the GPU box: python tools/prof_block.py under env overrides.
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in ""; do
  echo "== M156 $v"; env $v REPS=2 timeout 120 python tools/prof_block.py 100000 2>&1 | tail -1
done
for v in "" "BC_TMEM_STREAMS=1" "BC_GATHER_COPIES=1" "BC_KERNEL=v1"; do
  echo "== M312 $v"; env $v SPECIES=312 REPS=2 timeout 200 python tools/prof_block.py 100000 2>&1 | tail -1
done
