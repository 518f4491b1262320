# GPU tests + e2e bench on the GPU box.
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/e2e_probe.py
for v in "" "BC_PIPE_CHUNKS=8" "BC_PIPE_CHUNKS=64"; do
env $v timeout 400 python bench.py --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v value',d['value'],'e2e',d['e2e']['value'], d['e2e']['ms_per_step'])"
done
