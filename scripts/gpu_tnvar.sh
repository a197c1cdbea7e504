# A/B of k6_gemm_tn_tc block size / ring depth variants (libs built by `make variants`)
set -x
V=paper_2006_06608_b200/variants
for lib in $V/libgnna_tnbk32.so $V/libgnna_tnbk32s8.so $V/libgnna_tnlob6.so; do
GNNA_LIB=$lib timeout 900 python -m pytest tests/test_gemm_tc_gpu.py -q -x --timeout 600 2>&1 | tail -1
done
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_tnbk32.so $V/libgnna_tnbk32s8.so $V/libgnna_tnlob6.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration"
done
done
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_tnbk32.so $V/libgnna_tnbk32s8.so $V/libgnna_tnlob6.so; do
GNNA_LIB=$lib timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
