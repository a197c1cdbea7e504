# default upc cap 32 vs uncapped (GNNA_K3_UPC_MAX=0): full GPU tests + C3 / C4 / C5 K3 + train step
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -1  # (default cap)
for u in 32 0 32 0; do
for w in c3 c4; do
for agg in sum gin; do
GNNA_K3_UPC_MAX=$u timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu --agg $agg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w $agg upc_max=$u', round(d['ms_per_step']*1000,2))"
done
done
GNNA_K3_UPC_MAX=$u timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 sum upc_max=$u', round(d['ms_per_step'],3))"
GNNA_K3_UPC_MAX=$u timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3train upc_max=$u', round(d['ms_per_step'],4))"
done
