# shared-memory LU (bc_lu_sm.cuh): bitwise tests, Block-cells(N) bench with parity, kernel times
B="python bench.py --strategy block-cells-N --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-companion --no-dropin"
P='import json,sys; d=json.loads(sys.stdin.read()); p=d.get("parity") or {}; print(round(d["value"]), round(d["ms_per_step"],1), p.get("mismatched_cells"), p.get("cells_checked"))'
timeout 900 python -m pytest tests/test_lu_blockdiag.py -q -x -m gpu > gpurun_out/lu_sm_tests.log 2>&1; tail -2 gpurun_out/lu_sm_tests.log
echo "new:"; timeout 600 $B 2>gpurun_out/lu_sm_bench.err | tail -1 | python -c "$P"
K=N timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_sm_launches.csv \
    python tools/prof_block.py 20000 > gpurun_out/lu_sm_launch.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lu_sm_launches.csv')) if len(r)>14 and r[0].isdigit()]
agg={}
for r in rows:
    k=r[4].split('(')[0][:60]; agg.setdefault(k,[0,0]); agg[k][0]+=1; agg[k][1]+=float(r[14])
for k,(c,t) in agg.items(): print(f"{k:60s} n={c} total_ms={t/1e6:.2f}")
PY
if [ -n "$FULL" ]; then timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_devset.py -q -x -m gpu > gpurun_out/lu_sm_tests2.log 2>&1; tail -2 gpurun_out/lu_sm_tests2.log; fi
