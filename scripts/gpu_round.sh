# One evidence pass: bench (both arms), then the ncu counters of bench's batches.
set -e
TAG=${1:-r2}
make -s -C oracle
mkdir -p gpurun_out
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
bash scripts/gpu_ncu_counts.sh > gpurun_out/ncu_counts_${TAG}.log 2>&1
echo done
