# drop-in hub layout on a shuffled C5-shape graph (fp64): K3 time vs the number of hot rows copied to the tail
for k in 49152 500000 1000000 2500000; do
  GNNSIM_HUB_ROWS=$k timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k3_aggregate --csv --log-file gpurun_out/dropin_rows_$k.csv tests/cpp/bin/dropin_check bench 10000000 100000000 128 1 > gpurun_out/dropin_rows_$k.json 2>&1
  echo "k=$k $(grep -o 'hub_edges[^,]*' gpurun_out/dropin_rows_$k.json | head -1)"; grep k3_aggregate gpurun_out/dropin_rows_$k.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
done
