cd ${GRAFT_REPO_ROOT:-.}
for lib in base pp; do
  if [ $lib = pp ]; then cp gpurun_alt/libbc_pp.so paper_2405_17363_b200/libbc_b200.so; fi
  echo "== $lib M156 bicgstab"; REPS=3 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
  echo "== $lib M156 bicg"; REPS=2 timeout 300 python tools/prof_block.py 100000 bicg 2>&1 | tail -1
  echo "== $lib M312 bicgstab"; SPECIES=312 REPS=2 timeout 300 python tools/prof_block.py 100000 2>&1 | tail -1
done
