# four-step split sweep: every feasible lgC per size (PAB_LGC override), one process each
mkdir -p gpurun_out
SIZES=${SIZES:-"1e6,5e5,1024 2e6,1e6,512 4e6,2e6,256 1e7,2e6,64 2e7,1e7,48 4e7,2e7,24 6e7,3e7,16 8e7,4e7,12 1e8,5e7,8 1.2e8,6e7,8"}
for lgc in 0 6 7 8 9 10 11 12; do
  if [ $lgc = 0 ]; then unset PAB_LGC; else export PAB_LGC=$lgc; fi
  timeout 300 python scripts/quick_perf.py $SIZES 2>/dev/null | sed "s/^{/{\"lgc_force\": $lgc, /"
done > gpurun_out/split_sweep.jsonl
echo done
