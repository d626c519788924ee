# ncu --set full (with source) of one kernel of bench's C2 batch (after a clean plain run).
set -e
mkdir -p gpurun_out
K=${1:-k_row}
TAG=${2:-r2}
W=${3:-C2}
python scripts/ncu_counts.py run $W > gpurun_out/full_plain_$W.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o gpurun_out/full_${K}_${W}_${TAG} python scripts/ncu_counts.py run $W > gpurun_out/full_${K}_${TAG}.log 2>&1
echo done
