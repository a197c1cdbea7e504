set -x
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in $V/libgnna_nacc1.so $V/libgnna_tndbg3.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration|rror"
done
done
