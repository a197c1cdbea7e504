# GPU parity tests + smoke (run under gpurun)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -30
