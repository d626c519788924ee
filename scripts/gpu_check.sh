set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd paper_1910_04429_b200/csrc && make -s 2>&1 | tail -3; cd ../..
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30
