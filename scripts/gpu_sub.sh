# K3 with GNNA_K3_SUB consecutive tiles per CTA (1 = one tile, the r02 default)
set -x
GNNA_K3_SUB=2 timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -1
for rep in 1 2; do
for sb in 1 2 4; do
for agg in sum gcn; do
GNNA_K3_SUB=$sb timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu --agg $agg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 $agg sub $sb', round(d['ms_per_step']*1000,2))"
done
GNNA_K3_SUB=$sb timeout 600 python bench.py --workload c4 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 sum sub $sb', round(d['ms_per_step']*1000,2))"
done
done
