# C3 K3 with narrower teams (GNNA_K3_TEAM_MAX: TEAM 2 x KMAX 2, TEAM 1 x KMAX 4) vs the default TEAM 4
set -x
for rep in 1 2; do
for tm in 0 2 1; do
GNNA_K3_TEAM_MAX=$tm timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('team_max $tm', d['ms_per_step'], d.get('parity',{}).get('max_rel_err') if isinstance(d.get('parity'),dict) else d.get('parity'))"
GNNA_K3_TEAM_MAX=$tm timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu --agg gcn 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gcn team_max $tm', d['ms_per_step'])"
done
done
