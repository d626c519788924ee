# ncu --set full of the C2 step's four conv/carry kernels (run after the plain command exits 0)
set -e
TAG=${1:-r1}
mkdir -p gpurun_out
CMD2="python scripts/quick_perf.py ${2:-1e6,5e5,1024}"
$CMD2 > gpurun_out/plain_qp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_carry" -s 4 -c 4 -o gpurun_out/prof_${TAG} $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
