# k6_gemm_tc_tma with A_hi in TMEM (both MMAs TS; default where it fits) vs A_hi from shared memory (GNNA_TC_AT=0)
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -1
for at in 1 0 1 0; do
for shape in "410236 96 16" "410236 16 22" "1000000 64 64" "1000000 32 32"; do
GNNA_TC_AT=$at timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 python scripts/gemm_one.py $shape 3 2>&1 | grep -E "duration|rror" | sed "s/^/$at $shape /"
done
done
for at in 1 0; do
GNNA_TC_AT=$at timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
