for r in 1 2; do
GNNA_LIB=paper_2006_06608_b200/variants/libgnna_old.so timeout 900 python scripts/k3_ab.py --workloads c5,c4,c3 --params b200 --reps 20 --tag old 2>&1 | grep '^{'
timeout 900 python scripts/k3_ab.py --workloads c5,c4,c3 --params b200 --reps 20 --tag new 2>&1 | grep '^{'
done
