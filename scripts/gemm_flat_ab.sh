# A/B of k6_gemm_flat (narrow k, n <= 32) vs the tcgen05 path (GNNA_GEMM_NOFLAT=1):
# gemm tests, skinny GEMM timings and the C3 train step both ways.
R=${1:-r01o}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "gemm or layer or model or smoke" 2>&1 | tail -3
timeout 300 python scripts/gemm_ab.py > gpurun_out/gemm_ab_flat_$R.jsonl 2>&1
GNNA_GEMM_NOFLAT=1 timeout 300 python scripts/gemm_ab.py > gpurun_out/gemm_ab_noflat_$R.jsonl 2>&1
for i in 1 2; do
  timeout 600 python bench.py --workload c3train --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/c3train_flat_${R}_$i.json
  GNNA_GEMM_NOFLAT=1 timeout 600 python bench.py --workload c3train --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/c3train_noflat_${R}_$i.json
done
cat gpurun_out/gemm_ab_flat_$R.jsonl gpurun_out/gemm_ab_noflat_$R.jsonl
for f in gpurun_out/c3train_*flat_${R}_*.json; do echo $f; python -c "import json,sys; print(json.load(open('$f'))['ms_per_step'])"; done
for c in 3 5 6 8; do GNNA_FLAT_CTAS=$c timeout 300 python scripts/gemm_ab.py 2>&1 | sed -n 2,3p | sed "s/^/ctas=$c /"; done
