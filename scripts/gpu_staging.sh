# staged pageable copies: tests, then drop-in per-call times A/B on one box (GNNA_STAGING=0: the driver's staging)
# (a parallel MADV_POPULATE_WRITE pre-fault of the output was measured here too and made the call slower)
set -x
timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_dropin.py -q -x --timeout 600 2>&1 | tail -1
for rep in 1 2; do
for w in c3 c4; do
for v in "1" "0"; do
set -- $v
GNNA_STAGING=$1 timeout 600 ./tests/cpp/bin/dropin_check config $w 7 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w staging=$1', d['warm_call_ms_median'])"
done
done
done
