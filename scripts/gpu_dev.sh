# dev loop: parity tests then quick perf (library is prebuilt here and shipped)
set -e
make -s -C oracle
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_dev.log 2>&1 || true; tail -3 gpurun_out/pytest_dev.log
timeout 300 python scripts/quick_perf.py ${QP_ARGS:-}
