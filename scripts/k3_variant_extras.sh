# C3 sum/gcn/gcn_gather/gin and C5 per K3 variant via bench.py's extras.
for v in default "$@" default; do
  if [ $v = default ]; then L=""; else L=paper_2006_06608_b200/variants/libgnna_$v.so; fi
  GNNA_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r={'variant': '$v', 'c5_ms': round(d['ms_per_step'],3)}
for e in d['extra_workloads']:
    if 'aggregation' in e and e['workload'].startswith('C3'): r['c3_'+e['aggregation']] = round(e['kernel_ms']*1e3,1)
print(json.dumps(r))"
done
