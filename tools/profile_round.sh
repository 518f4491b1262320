#!/bin/bash
# Run on the GPU box (gpurun): bench line, ncu launch list of the same bench
# command, one ncu --set full capture of the hot kernel on the bench workload.
# Outputs under gpurun_out/; summaries are copied into profiles/ afterwards.
cd "$(dirname "$0")/.."
TAG=${1:-round1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:block_cells_tmem -c 1 \
    -o gpurun_out/prof_$TAG python tools/prof_block.py 100000 > gpurun_out/prof_$TAG.log 2>&1
ls -la gpurun_out/ | tail -20
