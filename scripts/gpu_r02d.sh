set -x
timeout 900 python -m pytest tests/test_layers_gpu.py -q -x --timeout 600 -k dense 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k6_dense_bwd -s 2 -c 1 -o /tmp/db python scripts/dense_one.py > /dev/null 2>&1; echo ncu $?
ncu -i /tmp/db.ncu-rep --page raw --csv > gpurun_out/dense_bwd_raw.csv 2>/dev/null
ncu -i /tmp/db.ncu-rep --page source --csv > gpurun_out/dense_bwd_source.csv 2>/dev/null
