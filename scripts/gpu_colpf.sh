# K3: L2 prefetch of the column-index span of the tile pf/2 ahead vs none (variants/libgnna_nocolpf.so)
set -x
timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_c3_parity_gpu.py -q -x 2>&1 | tail -1
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_nocolpf.so; do
for w in c3 c4; do
GNNA_LIB=$lib timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w sum $(basename $lib)', round(d['ms_per_step']*1000,2))"
done
GNNA_LIB=$lib timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 sum $(basename $lib)', round(d['ms_per_step'],3))"
GNNA_LIB=$lib timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3train $(basename $lib)', round(d['ms_per_step'],4))"
done
done
