# Round evidence: GPU tests, bench (both arms), launch list of the bench command.
# (The --set full capture is a separate call: scripts/gpu_ncu_full.sh; one ncu per call.)
set -e
TAG=${1:-r1}
make -s -C oracle
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 900 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_${TAG}.log
/tmp/int_peak > gpurun_out/int_peak_${TAG}.json 2>/dev/null || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int_peak scripts/int_peak.cu && /tmp/int_peak > gpurun_out/int_peak_${TAG}.json)
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --config C5 --steps 20 --no-cpu > gpurun_out/bench_C5_${TAG}.json 2> gpurun_out/bench_C5_${TAG}.err
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
