set -e
cd paper_1910_04429_b200/csrc && make -s 2>&1 | grep -i error || true; cd ../..
make -s -C oracle
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 300 ${PYTEST_ARGS:-} 2>&1 | tee gpurun_out/pytest_gpu.log | tail -30
