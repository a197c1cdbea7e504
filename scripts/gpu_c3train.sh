timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_model_gpu.py -q -x --timeout 600 2>&1 | tail -2
timeout 600 python bench.py --workload c3train --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/c3train.json
cut -c1-300 gpurun_out/c3train.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3train.csv python bench.py --workload c3train --steps 2 --warmup 1 > /dev/null 2>&1
