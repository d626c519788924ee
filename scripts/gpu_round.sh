# One evidence pass: the GPU tests, bench (both arms), then the ncu counters of bench's batches.
set -e
TAG=${1:-r2}
make -s -C oracle
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 1500 python -m pytest tests -q -s -m gpu --timeout 600 > gpurun_out/pytest_gpu_${TAG}.full 2>&1 || true
grep -E "passed|failed|ratio spread|compress criterion|round:" gpurun_out/pytest_gpu_${TAG}.full > gpurun_out/pytest_gpu_${TAG}.log || true
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --config C3 --steps 20 --warmup 5 --no-extra > gpurun_out/bench_C3_${TAG}.json 2> gpurun_out/bench_C3_${TAG}.err
bash scripts/gpu_ncu_counts.sh > gpurun_out/ncu_counts_${TAG}.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo done
cat gpurun_out/pytest_gpu_${TAG}.log
