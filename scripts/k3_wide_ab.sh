# K3 wide-team (d >= 32 fp32) variants on C5 (bench default config), default first and last.
for v in default "$@" default; do
  if [ $v = default ]; then L=""; else L=paper_2006_06608_b200/variants/libgnna_$v.so; fi
  c5=$(GNNA_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms_per_step'],3))")
  echo "{\"variant\": \"$v\", \"c5_ms\": $c5}"
done
