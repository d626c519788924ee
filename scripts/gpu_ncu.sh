set -e
cd paper_1910_04429_b200/csrc && make -s 2>&1 | grep -i error || true; cd ../..
make -s -C oracle
mkdir -p gpurun_out
TAG=${1:-r1}
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python scripts/quick_perf.py 1e6,5e5,1024"
$CMD2 > gpurun_out/plain_qp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_carry" -s 6 -c 4 -o gpurun_out/prof_${TAG} $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
