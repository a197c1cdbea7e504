# k6_gemm_tn_tc: 128-row blocks where three stages fit (default) vs 64 (GNNA_TN_BK=64)
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py tests/test_sharded_gpu.py -q -x --timeout 600 2>&1 | tail -1
for bk in 128 64 128 64; do
GNNA_TN_BK=$bk timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration|rror"
GNNA_TN_BK=$bk timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
