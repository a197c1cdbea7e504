# full validation: smoke, GPU tests, default bench + reference arm, launch list of the default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; tail -2 gpurun_out/bench_$1.err | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$1.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras --no-ncu > /dev/null 2>&1; echo ncu $?
