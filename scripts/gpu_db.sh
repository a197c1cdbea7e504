# k6_dense_bwd tile rows / ring depth variants (make variants VNAMES="db64s6 db128s3")
set -x
V=paper_2006_06608_b200/variants
for lib in $V/libgnna_db64s6.so $V/libgnna_db128s3.so; do
GNNA_LIB=$lib timeout 600 python -m pytest tests/test_layers_gpu.py -q -x -k dense 2>&1 | tail -1
done
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_db64s6.so $V/libgnna_db128s3.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k6_dense_bwd -s 2 -c 1 python scripts/dense_one.py 2>&1 | grep -E "duration|warps_active"
done
done
