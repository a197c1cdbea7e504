set -x
for k in k3p_aggregate k3_aggregate; do
  if [ $k = k3_aggregate ]; then export GNNA_K3P=0; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/$k python scripts/k3p_one.py c3 > /dev/null 2>&1; echo ncu $?
  ncu -i /tmp/$k.ncu-rep --page raw --csv > gpurun_out/${k}_c3_raw.csv 2>/dev/null
  ncu -i /tmp/$k.ncu-rep --page source --csv > gpurun_out/${k}_c3_source.csv 2>/dev/null
  ncu -i /tmp/$k.ncu-rep --page details --csv > gpurun_out/${k}_c3_details.csv 2>/dev/null
done
ls -la gpurun_out
