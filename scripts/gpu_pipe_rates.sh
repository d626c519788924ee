# Builds and runs scripts/pipe_rates.cu on the GPU box; result -> gpurun_out/pipe_rates.json
set -e
mkdir -p gpurun_out /tmp/pr
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pr/pipe_rates scripts/pipe_rates.cu
/tmp/pr/pipe_rates | tee gpurun_out/pipe_rates.json
