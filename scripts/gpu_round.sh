set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
cat gpurun_out/bench_c5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_aggregate -s 2 -c 1 -o gpurun_out/k3_c5 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 $?
tail -5 gpurun_out/ncu_full.log
