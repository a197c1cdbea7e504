# GPU parity tests + smoke (run under gpurun); extra args go to pytest
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 "$@" 2>&1 | tail -40
