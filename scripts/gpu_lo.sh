# truncated-lo converters (default) vs round-to-nearest lo (variants/libgnna_lorna.so)
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -2
V=paper_2006_06608_b200/variants
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_lorna.so paper_2006_06608_b200/libgnna.so $V/libgnna_lorna.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration"
GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 2>&1 | grep -E "duration"
GNNA_LIB=$lib timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
