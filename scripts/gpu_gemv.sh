set -x
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_c3_parity_gpu.py tests/test_sharded_gpu.py -q -x --timeout 600 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c90-200
GNNA_FUSED_UPDATE=0 timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c90-200
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_r02g_launches.csv python bench.py --workload c3train --steps 3 --warmup 3 --no-graph > /dev/null 2>&1; echo ncu $?
