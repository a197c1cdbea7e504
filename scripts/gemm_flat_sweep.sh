# k6_gemm_flat CTAs-per-SM sweep on the C3 dZ shape (410236 x 22 . 22 x 16), ncu device times, + one --set full capture.
R=${1:-r01p}
for c in ${CTAS:-1 2 3 4 5}; do
  GNNA_FLAT_CTAS=$c timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k6_gemm_flat python scripts/gemm_one.py 410236 22 16 3 2>/dev/null | grep -E "gpu__time|dram__bytes" | tail -3 | sed "s/^/ctas=$c /"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k6_gemm_flat -s 1 -c 1 -o /tmp/flat_$R python scripts/gemm_one.py 410236 22 16 3 > /dev/null 2>&1; echo ncu $?
ncu -i /tmp/flat_$R.ncu-rep --page raw --csv > gpurun_out/gemm_flat_${R}_raw.csv 2>/dev/null
