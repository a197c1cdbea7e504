# partial-sum reducer for few outputs x many chunks (8 x 128 slices per block) vs the 32 x 32 one
set -x
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x 2>&1 | tail -1
for n in 1 0; do
GNNA_REDUCE_NARROW=$n timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_reduce -s 2 -c 1 python scripts/dense_one.py 2>&1 | grep -E "k_reduce|duration" | sed "s/^/narrow=$n /"
done
for rep in 1 2; do
for n in 1 0; do
GNNA_REDUCE_NARROW=$n timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3train narrow=$n', round(d['ms_per_step'],4))"
done
done
