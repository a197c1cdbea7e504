# A/B of the dW partial reduction: k_reduce_partials (default) vs the sequential reducers (GNNA_TN_SEQ_REDUCE=1).
R=${1:-r01q}
timeout 600 python -m pytest tests/test_gemm_tc_gpu.py tests/test_layers_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -1
for v in "" 1; do
  env ${v:+GNNA_TN_SEQ_REDUCE=1} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_red${v}_launches_$R.csv python bench.py --workload c3train --steps 2 --warmup 3 > /dev/null 2>&1
  for i in 1 2; do env ${v:+GNNA_TN_SEQ_REDUCE=1} timeout 600 python bench.py --workload c3train --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; print('seq=$v', json.load(sys.stdin)['ms_per_step'])"; done
done
