for w in c3 c4 c5; do for a in sum gcn gin; do
  timeout 600 python bench.py --workload $w --agg $a --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1
done; done
