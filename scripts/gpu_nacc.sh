# k6_gemm_tn_tc: NACC independent TMEM accumulators (default 8 for q <= 16) vs 1 / 2
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -2
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_nacc1.so $V/libgnna_nacc2.so $V/libgnna_tndbg1.so $V/libgnna_tndbg2.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration"
done
done
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
