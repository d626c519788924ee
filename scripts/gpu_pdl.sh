# A/B of programmatic dependent launch (PAB_PDL=0/1) + parity (development aid)
set -e
mkdir -p gpurun_out
CASES="1e6,5e5,1 1e6,5e5,16 1e6,5e5,1024 1e7,2e6,64 1e8,5e7,1 1e8,5e7,16"
for rep in 1 2; do
  for v in 0 1; do
    echo "== PAB_PDL=$v rep $rep"
    PAB_PDL=$v python scripts/quick_perf.py $CASES
  done
done 2>&1 | tee gpurun_out/pdl_ab.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['batch'], d['ms_per_batch'], d['kernels_ms'])
    else: print(l.strip())
"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_split.py tests/test_gpu_guards.py -q -x -m gpu 2>&1 | tail -3
