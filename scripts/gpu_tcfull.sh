set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 -o gpurun_out/tc_y -f python scripts/gemm_one.py 410236 16 22 3 > /dev/null 2>&1
ncu -i gpurun_out/tc_y.ncu-rep --page raw --csv > gpurun_out/tc_y_raw.csv
ncu -i gpurun_out/tc_y.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_y_source.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 -o gpurun_out/tc_x -f python scripts/gemm_one.py 410236 96 16 3 > /dev/null 2>&1
ncu -i gpurun_out/tc_x.ncu-rep --page raw --csv > gpurun_out/tc_x_raw.csv
ncu -i gpurun_out/tc_x.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_x_source.csv
