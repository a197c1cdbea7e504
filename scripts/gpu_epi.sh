# X.W epilogue store loop unrolled x4 (staging loads overlap) -- timing of the C3 products
set -x
timeout 900 python -m pytest tests/test_gemm_tc_gpu.py -q -x --timeout 600 2>&1 | tail -1
for rep in 1 2; do
for shape in "410236 96 16" "410236 16 22" "410236 128 64"; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 python scripts/gemm_one.py $shape 3 2>&1 | grep -E "duration|rror" | sed "s/^/$shape /"
done
done
timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
