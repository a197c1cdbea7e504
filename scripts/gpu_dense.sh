set -x
timeout 900 python -m pytest tests/test_layers_gpu.py -q -x --timeout 600 -k dense 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k6_dense_bwd -s 2 -c 1 python scripts/dense_one.py 2>&1 | grep -E "duration|warps_active|dram__bytes" 
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_launches.csv python bench.py --workload c3train --steps 2 --warmup 3 --no-ncu > /dev/null 2>&1; echo launches $?
