# tensor-core GEMM A/B: TMA-fed (default) vs register-fed vs SIMT, C3 training shapes
timeout 200 python scripts/gemm_ab.py 2>&1 | tail -4
echo "--- GNNA_GEMM_TC_LD"; GNNA_GEMM_TC_LD=1 timeout 200 python scripts/gemm_ab.py 2>&1 | tail -4
echo "--- GNNA_GEMM_SIMT"; GNNA_GEMM_SIMT=1 timeout 200 python scripts/gemm_ab.py 2>&1 | tail -4
