# K3S (CTA-level prefetch of metadata + indices) A/B on C3/C4, correctness via k3p_ab's parity check
python scripts/k3p_ab.py k3 2>&1 | grep -v c4
GNNA_K3S=2 python scripts/k3p_ab.py k3s_m4 2>&1 | grep -v c4
for v in s3 s2; do GNNA_K3S=2 GNNA_LIB=paper_2006_06608_b200/variants/libgnna_$v.so python scripts/k3p_ab.py k3s_$v 2>&1 | grep -v c4; done
