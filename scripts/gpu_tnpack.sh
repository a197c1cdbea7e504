# packed [B_hi | B_lo] slice for q <= 16 (default) vs separate B_lo slice (GNNA_TN_PACK=0)
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -2
for pk in 1 0 1 0; do
GNNA_TN_PACK=$pk timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration"
GNNA_TN_PACK=$pk timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
