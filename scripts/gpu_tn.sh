set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py -q -x --timeout 600 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 python scripts/gemm_one.py 410236 96 16 3 tn 2>&1 | grep -E "duration|warps_active|dram__bytes|tensor"
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 2>/dev/null | cut -c90-200
