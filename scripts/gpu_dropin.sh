# drop-in: the reference's suites + our C++ caller check; the shuffled C5-shape fp64 bench, kernel times by ncu
set -x
timeout 1500 python -m pytest tests/test_dropin.py -q -x --timeout 1200 2>&1 | tail -3
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k3_aggregate --csv --log-file gpurun_out/dropin_c5_k3.csv tests/cpp/bin/dropin_check bench 10000000 100000000 128 2 > gpurun_out/dropin_c5_bench.json 2> gpurun_out/dropin_c5_bench.err; echo rc $?
cat gpurun_out/dropin_c5_bench.json; tail -3 gpurun_out/dropin_c5_bench.err
grep -c k3_aggregate gpurun_out/dropin_c5_k3.csv
