set -x
timeout 900 python -m pytest tests/test_layers_gpu.py -q -x --timeout 600 -k dense 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_r02c_launches.csv python bench.py --workload c3train --steps 3 --warmup 3 --no-graph > /dev/null 2>&1; echo ncu $?
