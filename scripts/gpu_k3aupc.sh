# K3A (fp64 narrow rows) with 16 units per CTA (GNNA_K3A_UPC=16, 128 threads) vs 32 (256)
set -x
GNNA_K3A_UPC=16 timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_configs_gpu.py tests/test_c3_parity_gpu.py -q -x 2>&1 | tail -1
timeout 300 python scripts/sanitize.py 2>&1 | tail -1
for rep in 1 2; do
for u in "" 16 8; do
GNNA_K3A_UPC=$u timeout 300 python scripts/upc_ab.py 2>&1 | grep float64 | sed "s/^/k3a_upc=$u /"
done
done
