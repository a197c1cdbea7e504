# k6_dense_bwd: dz with W in registers (default) vs W in shared memory (variants/libgnna_dbsmemw.so)
set -x
timeout 600 python -m pytest tests/test_layers_gpu.py tests/test_model_gpu.py -q -x -k "dense or gcn2 or train" 2>&1 | tail -1
V=paper_2006_06608_b200/variants
for rep in 1 2; do
for lib in paper_2006_06608_b200/libgnna.so $V/libgnna_dbsmemw.so; do
echo $lib; GNNA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_dense_bwd -s 2 -c 1 python scripts/dense_one.py 2>&1 | grep -E "duration"
done
done
