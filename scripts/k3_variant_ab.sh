# K3 small-team (d <= 28 fp32) occupancy/unroll variants on C3 (k3_ab.py,
# all three aggregation flavours via bench extras is too slow; sum only), the
# default library first and last.  Usage: bash scripts/k3_variant_ab.sh v1 v2 ...
for v in default "$@" default; do
  if [ $v = default ]; then L=""; else L=paper_2006_06608_b200/variants/libgnna_$v.so; fi
  c3=$(GNNA_LIB=$L timeout 300 python scripts/k3_ab.py --workloads c3 --params b200 --reps 20 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms'])")
  echo "{\"variant\": \"$v\", \"c3_ms\": $c3}"
done
