# A/B of k6_gemm_tn_tc with the ring refilled by a producer warp (GNNA_TN_PROD=1)
set -x
GNNA_TN_PROD=1 timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py -q -x --timeout 600 2>&1 | tail -2
for prod in 0 1 0 1; do
GNNA_TN_PROD=$prod timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration"
done
for prod in 0 1 0 1; do
GNNA_TN_PROD=$prod timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-200
done
