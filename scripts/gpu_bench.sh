# the default bench (as the driver runs it), then the reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; tail -3 gpurun_out/bench_$1.err | cut -c1-300; grep -E "Elapsed|Maximum resident" gpurun_out/bench_$1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$1.json 2>&1; tail -c 600 gpurun_out/bench_ref_$1.json
