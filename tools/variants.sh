# GPU tests + kernel timings on the GPU box.
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in "" "BC_TMEM_TEAM=1"; do
  echo "== M312 bicgstab $v"; env $v SPECIES=312 REPS=2 timeout 200 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== M312 bicg $v"; env $v SPECIES=312 REPS=1 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
  echo "== M156 bicg $v"; env $v REPS=2 timeout 200 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
done
for v in "" "BC_TMEM_TEAM=2" "BC_TMEM_TEAM=4"; do
  echo "== M156 bicgstab $v"; env $v REPS=2 timeout 200 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== M156 bicgstab 100 cells $v"; env $v REPS=3 timeout 200 python tools/prof_block.py 100 2>&1 | tail -1
  echo "== M156 bicgstab 2000 cells $v"; env $v REPS=3 timeout 200 python tools/prof_block.py 2000 2>&1 | tail -1
done
