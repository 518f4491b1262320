#!/bin/bash
# Kernel time of 1000 P-regime Jacobi-BiCGSTAB iterations vs batch size and
# team width (BC_TMEM_TEAM): one cell alone per SM vs 16 per SM.  Run under gpurun.
cd "$(dirname "$0")/.."
for team in 1 2 4; do for c in 148 592 1184 2368 4736; do
  r=$(BC_TMEM_TEAM=$team timeout 300 python bench.py --cells $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])")
  echo "team=$team cells=$c $r"
done; done
