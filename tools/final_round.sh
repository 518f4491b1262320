#!/bin/bash
# The round's evidence in one GPU session (run under gpurun): the GPU test
# suite, smoke, the driver-shaped bench and reference arm, every BASELINE
# config, the strategy tables, the ncu profile of the hot kernel, the N=2 path
# under torchrun (ranks sharing the box's GPU: a path test, not a scaling
# number), the sanitizers and a fuzz run.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
TAG=${1:-round2d}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_$TAG.log 2>&1; tail -2 gpurun_out/gputest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_reference_$TAG.json 2>&1
bash tools/round_configs.sh $TAG
bash tools/profile_round.sh $TAG
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
    bench.py --gpus 2 --cells 20000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_$TAG.json 2> gpurun_out/bench_n2_$TAG.err
# small batches (latency kernel phase profile + sweep) and the Block-cells(N)
# launch list (LU fallback share of the step)
[ -x tools/latprof.bin ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 --extended-lambda \
    -DBC_LAT_PROFILE -I paper_2405_17363_b200/csrc -I include -o tools/latprof.bin tools/latprof.cu \
    paper_2405_17363_b200/csrc/bc_latency_plan.cpp paper_2405_17363_b200/csrc/bc_plan.cpp -L paper_2405_17363_b200 \
    -lbc_workload -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2405_17363_b200'
./tools/latprof.bin > gpurun_out/latprof_$TAG.txt 2>&1
CELLS=1,10,100,148,1000,10000 timeout 600 python tools/latency_sweep.py > gpurun_out/latsweep_$TAG.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bcN_$TAG.csv \
    python bench.py --strategy block-cells-N --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity --no-companion --no-dropin > /dev/null 2>&1
# (compute-sanitizer runs are closed on this GPU pool since round 2e: profiles/round2_sanitize_*.txt are the last)
timeout 900 python tools/fuzz_gpu.py 600 43 > gpurun_out/fuzz_$TAG.txt 2>&1; tail -1 gpurun_out/fuzz_$TAG.txt
ls gpurun_out | wc -l
