# K3 narrow-team unroll / register-cap variants at the 32-unit (128-thread) CTAs
set -x
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_s4m5.so $V/libgnna_s6m5.so $V/libgnna_s5m4.so; do
GNNA_LIB=$lib timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 sum $(basename $lib)', round(d['ms_per_step']*1000,2))"
GNNA_LIB=$lib timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3train $(basename $lib)', round(d['ms_per_step'],4))"
done
done
