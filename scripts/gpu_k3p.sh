# K3P correctness + A/B against the plain K3 and the build variants
set -x
timeout 900 python -m pytest tests/test_aggregate_gpu.py tests/test_c3_parity_gpu.py tests/test_model_gpu.py tests/test_fanout_gpu.py -q -x --timeout 600 2>&1 | tail -5
GNNA_K3P=0 timeout 300 python scripts/k3p_ab.py plainK3 > gpurun_out/k3p_ab2.jsonl 2>&1
timeout 300 python scripts/k3p_ab.py k3p_default >> gpurun_out/k3p_ab2.jsonl 2>&1
for v in p2u8 p3u6 p3u8 p4u4 p4u2 p3s2; do GNNA_LIB=paper_2006_06608_b200/variants/libgnna_$v.so timeout 300 python scripts/k3p_ab.py $v >> gpurun_out/k3p_ab2.jsonl 2>&1; done
grep -v c4 gpurun_out/k3p_ab2.jsonl
