#!/bin/bash
# Every BASELINE.json config on one B200 (run under gpurun); JSON lines into
# gpurun_out/configs_<tag>.jsonl, the strategy tables into
# gpurun_out/strategies_m{156,312}.json.  Copy into profiles/ afterwards.
cd "$(dirname "$0")/.."
TAG=${1:-round1}
OUT=gpurun_out/configs_$TAG.jsonl
: > $OUT
run() { timeout 900 python bench.py "$@" 2>>gpurun_out/configs_$TAG.err | tail -1 >> $OUT; }
run                                                     # configs[2]/headline: 100k M156, Block-cells(1), BiCGSTAB
run --cells 10000 --steps 100                           # configs[1]: 10k cells vs CPU 1 thread / all cores
run --cells 100 --steps 600                    # configs[0]: the reference's CPU workload size
run --cells 1000000 --steps 3 --no-cpu-baseline         # configs[3]: one 1M-cell shard (8 GPUs: 125k each)
run --species 312 --steps 5 --no-cpu-baseline           # configs[4]: scaled mechanism
run --algo bicg --steps 5 --no-cpu-baseline             # the reference algorithm on the same workload
run --regime C --steps 10 --no-cpu-baseline             # converging regime (early exit, imbalance)
timeout 900 python tools/compare_strategies.py 100000 156 > /dev/null 2>>gpurun_out/configs_$TAG.err
timeout 900 python tools/compare_strategies.py 100000 312 > /dev/null 2>>gpurun_out/configs_$TAG.err
wc -l $OUT
