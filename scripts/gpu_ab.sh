for v in u4mb4 u4mb5 u4mb6 u2mb8 u6mb4 u8mb4; do
  L=paper_2006_06608_b200/variants/libgnna_$v.so
  GNNA_LIB=$L timeout 900 python scripts/k3_ab.py --workloads c5,c4,c3 --params auto --reps 20 --tag $v 2>&1 | grep '^{'
done
