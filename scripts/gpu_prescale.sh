# GCN gather form: per-source weights applied by a row pre-scale pass + plain K3 (default) vs per-edge weights (GNNA_PRESCALE=0);
# the caller's L2 window on x follows to the scaled copy (C5's hub rows)
set -x
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "gcn or weight or c3 or configs or fanout or layers or model" 2>&1 | tail -1
for rep in 1 2; do
for pre in 1 0; do
GNNA_PRESCALE=$pre timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu --agg gcn 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 gcn prescale $pre', round(d['ms_per_step']*1000,2), d.get('parity'))"
GNNA_PRESCALE=$pre timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras --no-ncu --agg gcn 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 gcn prescale $pre', round(d['ms_per_step'],3), d.get('parity'))"
done
done
