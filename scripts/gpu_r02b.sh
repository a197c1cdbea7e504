# dense backward fusion + train step; same-box A/B of the previous libgnna (HEAD~1) vs this one
set -x
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_model_gpu.py tests/test_c3_parity_gpu.py -q -x --timeout 600 2>&1 | tail -3
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 > gpurun_out/c3train_r02b.json 2>/dev/null; cut -c1-600 gpurun_out/c3train_r02b.json
GNNA_DENSE_BWD=0 timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_r02b_launches.csv python bench.py --workload c3train --steps 3 --warmup 3 --no-graph > /dev/null 2>&1; echo ncu $?
for i in 1 2; do
GNNA_LIB=paper_2006_06608_b200/variants/libgnna_prev.so timeout 300 python scripts/k3p_ab.py prev >> gpurun_out/prev_ab.jsonl 2>&1
timeout 300 python scripts/k3p_ab.py cur >> gpurun_out/prev_ab.jsonl 2>&1
done
cat gpurun_out/prev_ab.jsonl
