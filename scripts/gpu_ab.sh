for v in default b16 b16mb4 b16u6mb4 b8mb4; do
  if [ $v = default ]; then L=""; else L=paper_2006_06608_b200/variants/libgnna_$v.so; fi
  GNNA_LIB=$L timeout 900 python scripts/k3_ab.py --workloads c3,c4 --params b200 --reps 20 --tag $v 2>&1 | grep '^{'
done
