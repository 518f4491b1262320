#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every device kernel
# path at small shapes (tools/sanitize_cases.py); run under gpurun.  Summaries
# into gpurun_out/sanitize_<tool>.txt.
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  out=gpurun_out/sanitize_$tool.txt
  : > $out
  for c in tmem_bicgstab tmem_bicg tmem_team2 tmem_team4_coupled latency_bicgstab latency_bicg v1_bicg v1_bicgstab \
           multi_cells thread_per_cell lu_blockdiag lu_dense; do
    echo "== $tool $c" >> $out
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py $c >> $out 2>&1
    echo "rc=$?" >> $out
  done
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|==.*rc=\|bitwise" gpurun_out/sanitize_*.txt | tail -80
