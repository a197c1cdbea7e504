# r02a: GPU tests (incl. the new full-size C3 parity), then the default bench with its in-run ncu probe.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; tail -5 gpurun_out/bench_r02a.err
cut -c1-3000 gpurun_out/bench_r02a.json
