# k6_gemm_tc_tma_split (4 converter warps, 2 x 4 epilogue warps, MMA and producer warps) vs the two-group kernel
set -x
for sp in 1 0; do
GNNA_TC_SPLIT=$sp timeout 900 python -m pytest tests/test_gemm_tc_gpu.py -q -x --timeout 600 2>&1 | tail -1
done
for rep in 1 2; do
for sp in 1 0; do
for shape in "410236 96 16" "410236 16 22" "410236 128 64" "1000000 64 64" "1000000 32 32"; do
GNNA_TC_SPLIT=$sp timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k6_gemm_tc_tma -s 2 -c 1 python scripts/gemm_one.py $shape 3 2>&1 | grep -E "duration|rror" | sed "s/^/$sp $shape /"
done
done
done
for sp in 1 0; do
GNNA_TC_SPLIT=$sp timeout 600 python bench.py --workload c3train --steps 30 --warmup 5 --no-ncu 2>/dev/null | cut -c90-160
done
