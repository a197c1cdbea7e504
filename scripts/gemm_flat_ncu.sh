# Device time per launch of the narrow GEMMs inside the C3 train step, flat vs tcgen05 (GNNA_GEMM_NOFLAT=1).
R=${1:-r01p}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_flat_launches_$R.csv python bench.py --workload c3train --steps 2 --warmup 3 > /dev/null 2>&1; echo $?
GNNA_GEMM_NOFLAT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3train_noflat_launches_$R.csv python bench.py --workload c3train --steps 2 --warmup 3 > /dev/null 2>&1; echo $?
