# ncu --set full of the tensor-core GEMM (and the SIMT kernel for contrast) on one shape
set -x
M=${1:-410236}; K=${2:-96}; N=${3:-16}; TAG=${4:-gemm}
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k6_gemm_tc -s 2 -c 1 -o gpurun_out/${TAG}_tc -f python scripts/gemm_one.py $M $K $N 3 > gpurun_out/${TAG}_tc.log 2>&1
timeout 300 env GNNA_GEMM_SIMT=1 ncu --set full --clock-control none -k regex:k6_gemm -s 2 -c 1 -o gpurun_out/${TAG}_simt -f python scripts/gemm_one.py $M $K $N 3 > gpurun_out/${TAG}_simt.log 2>&1
for f in ${TAG}_tc ${TAG}_simt; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null; ncu -i gpurun_out/$f.ncu-rep --page source --csv > gpurun_out/$f.source.csv 2>/dev/null; done
ls -la gpurun_out | tail
