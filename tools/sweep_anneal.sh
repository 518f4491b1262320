#!/bin/bash
# Schedule-annealing objective weights and length vs bench throughput (run
# under gpurun): BC_YST_WEIGHT / BC_YRD_WEIGHT / BC_PUB_WEIGHT / BC_ANNEAL_ITERS.
cd "$(dirname "$0")/.."
for cfg in "3 1 1 200000" "3 2 1 200000" "4 2 1 200000" "2 2 1 200000" "3 1 1 600000" "3 2 2 200000"; do
  set -- $cfg
  r=$(BC_YST_WEIGHT=$1 BC_YRD_WEIGHT=$2 BC_PUB_WEIGHT=$3 BC_ANNEAL_ITERS=$4 timeout 600 python bench.py --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline --no-parity --no-companion --no-dropin 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['roofline']['binding']['model_wavefronts_per_group_iteration'], round(d['roofline']['binding']['frac_model'],3))")
  echo "yst=$1 yrd=$2 pub=$3 iters=$4 -> $r"
done
