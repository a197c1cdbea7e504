set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k6_gemm_tn_tc -s 2 -c 1 -o gpurun_out/tn_prod -f python scripts/gemm_one.py 410236 96 16 3 tn > /dev/null 2>&1
ncu -i gpurun_out/tn_prod.ncu-rep --page raw --csv > gpurun_out/tn_prod_raw.csv
ncu -i gpurun_out/tn_prod.ncu-rep --page source --csv --print-source sass > gpurun_out/tn_prod_source.csv
ls -la gpurun_out
