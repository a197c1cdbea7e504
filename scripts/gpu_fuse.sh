# fused carry combine (no K3b) + K3A for fp64: full GPU suite, C3/C4 A/B, C5 bench line
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -4
timeout 300 python scripts/k3p_ab.py fused > gpurun_out/fuse_ab.jsonl 2>&1
GNNA_K3A=2 timeout 300 python scripts/k3p_ab.py fused_k3a_all >> gpurun_out/fuse_ab.jsonl 2>&1
cat gpurun_out/fuse_ab.jsonl
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu > gpurun_out/bench_fuse.json 2> gpurun_out/bench_fuse.err; tail -3 gpurun_out/bench_fuse.err
cut -c1-1500 gpurun_out/bench_fuse.json
