set -e
mkdir -p gpurun_out
python scripts/quick_perf.py 1e6,5e5,1024 > gpurun_out/qp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_carry" -s 1 -c 1 -o gpurun_out/prof_wide python scripts/quick_perf.py 1e6,5e5,1024 > gpurun_out/ncu_wide.log 2>&1
echo done
