set -e
cd paper_1910_04429_b200/csrc && make -s 2>&1 | grep -i error || true; cd ../..
make -s -C oracle
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int_peak scripts/int_peak.cu
mkdir -p gpurun_out
/tmp/int_peak | tee gpurun_out/int_peak.json
timeout 900 python bench.py ${BENCH_ARGS:-} 2>&1 | tee gpurun_out/bench.log
