# Round measurement: tests, bench (C5 default), launch list, ncu --set full of K3 (C5 and C3), sweep.
# ncu reports are reduced to CSV on the box (gpurun_out/ must stay < 64 MiB).
set -x
R=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -3 gpurun_out/bench_$R.err
cat gpurun_out/bench_$R.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 $?
for w in c5 c3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_aggregate -s 2 -c 1 -o /tmp/k3_${w}_$R python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu_$w $?
  ncu -i /tmp/k3_${w}_$R.ncu-rep --page raw --csv > gpurun_out/k3_${w}_${R}_raw.csv 2>/dev/null
  ncu -i /tmp/k3_${w}_$R.ncu-rep --page source --csv > gpurun_out/k3_${w}_${R}_source.csv 2>/dev/null
done
for w in c1 c2 c3 c4; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1; done > gpurun_out/sweep_$R.jsonl
timeout 600 python bench.py --workload c3 --agg gcn --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 > gpurun_out/c3gcn_$R.json
timeout 600 python bench.py --workload c3train --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/c3train_$R.json
timeout 300 python scripts/gemm_ab.py > gpurun_out/gemm_ab_$R.jsonl 2>&1
GNNA_GEMM_SIMT=1 timeout 300 python scripts/gemm_ab.py > gpurun_out/gemm_ab_simt_$R.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k6_gemm_tc -s 2 -c 1 -o /tmp/gemm_tc_$R python scripts/gemm_one.py 410236 96 16 3 > /dev/null 2>&1; echo ncu_gemm $?
ncu -i /tmp/gemm_tc_$R.ncu-rep --page raw --csv > gpurun_out/gemm_tc_${R}_raw.csv 2>/dev/null
du -sh gpurun_out
