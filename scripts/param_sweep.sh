# gs x dw x tpb sweep of K3 (BASELINE config C4 asks for it); C3 and C5 too
P=""
for g in 1 4 16 64 256 1024 4096; do for d in 4 8 16 32; do for t in 32 128 512 1024; do P="$P,$g/$d/$t"; done; done; done
P=${P#,}
timeout 1500 python scripts/k3_ab.py --workloads c4,c3 --params $P --reps 10 --tag sweep 2>&1 | grep '^{'
P5=""
for g in 16 64 256 1024 4096; do for t in 128 512; do P5="$P5,$g/32/$t"; done; done
timeout 900 python scripts/k3_ab.py --workloads c5 --params ${P5#,} --reps 5 --tag sweep 2>&1 | grep '^{'
