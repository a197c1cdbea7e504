# k6_gemm_tn_small CTAs-per-SM sweep on the C3 dW2 shape (Z^T dY: 410236 x 16, 410236 x 22), ncu device times.
for c in ${CTAS:-2 3 4 6 8}; do
  GNNA_TN_SMALL_CTAS=$c timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k6_gemm_tn_small|k_reduce" python scripts/gemm_one.py 410236 16 22 3 tn 2>/dev/null | grep -E "gpu__time" | awk -F'","' -v c=$c '{print "ctas=" c, $5, $NF}' | tail -2
done
