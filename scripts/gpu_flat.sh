# y = z2 W2 (16 -> 22): tcgen05 TMA (default) vs k6_gemm_flat on FFMA2 (GNNA_GEMM_FLAT=1)
set -x
GNNA_GEMM_FLAT=1 timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py -q -x --timeout 600 2>&1 | tail -1
for f in 0 1 0 1; do
if [ $f = 1 ]; then export GNNA_GEMM_FLAT=1; else unset GNNA_GEMM_FLAT; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm -s 2 -c 1 python scripts/gemm_one.py 410236 16 22 3 2>&1 | grep -E "k6_gemm|duration|rror"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm -s 2 -c 1 python scripts/gemm_one.py 410236 22 16 3 2>&1 | grep -E "duration|rror"
done
