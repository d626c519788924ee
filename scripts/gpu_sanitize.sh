# one compute-sanitizer tool per gpurun call: bash scripts/gpu_sanitize.sh memcheck|racecheck|synccheck
set -e
T=${1:-memcheck}
mkdir -p gpurun_out
make -s -C oracle
python scripts/sanitize_small.py > gpurun_out/sanitize_plain_$T.log 2>&1
timeout 2400 compute-sanitizer --tool $T --error-exitcode 9 --log-file gpurun_out/sanitize_$T.log \
    python scripts/sanitize_small.py > gpurun_out/sanitize_${T}_stdout.log 2>&1
echo "sanitizer $T exit $?"
tail -5 gpurun_out/sanitize_$T.log
