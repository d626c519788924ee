# ncu counters for bench.py's roofline: C2, C5, C4 batches (one ncu tool, three runs).
set -e
mkdir -p gpurun_out
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_counts; print(ncu_counts.METRICS)")
for W in ${WORKLOADS:-C2 C5 C4 C3 C1}; do
  python scripts/ncu_counts.py run $W > gpurun_out/ncu_counts_plain_$W.log 2>&1
  ncu --metrics $M --clock-control none -k regex:"k_" --csv \
      --log-file gpurun_out/ncu_counts_$W.csv python scripts/ncu_counts.py run $W \
      > gpurun_out/ncu_counts_$W.log 2>&1
done
echo done
