# K3: L2 prefetch of the flush's x[v] row at unit start (EPI_SELF forms) vs none (variants/libgnna_noselfpf.so)
set -x
timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_c3_parity_gpu.py -q -x 2>&1 | tail -1
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_noselfpf.so; do
for agg in sum gin; do
GNNA_LIB=$lib timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras --no-ncu --agg $agg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 $agg $(basename $lib)', round(d['ms_per_step']*1000,2))"
GNNA_LIB=$lib timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras --no-ncu --agg $agg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 $agg $(basename $lib)', round(d['ms_per_step'],3))"
done
done
done
