# launch list + one full capture of the shared-memory LU kernels (Block-cells(N), M156, P regime)
K=N ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_sm_launches.csv \
    python tools/prof_block.py 20000 > gpurun_out/lu_sm_launch.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lu_sm_launches.csv')) if len(r)>14 and r[0].isdigit()]
agg={}
for r in rows:
    k=r[4].split('(')[0][:60]; agg.setdefault(k,[0,0]); agg[k][0]+=1; agg[k][1]+=float(r[14])
for k,(c,t) in agg.items(): print(f"{k:60s} n={c} total_ms={t/1e6:.2f}")
PY
K=N ncu --set full --clock-control none --import-source on -k regex:lu_sm_factor -c 1 -o gpurun_out/lu_sm_factor \
    python tools/prof_block.py 20000 > gpurun_out/lu_sm_full.log 2>&1
tail -1 gpurun_out/lu_sm_full.log
