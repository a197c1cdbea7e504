# quick per-workload bench lines (no e2e / cpu legs)
for w in c1 c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1
done
