# ncu --set full on one kernel of quick_perf: $1 = tag, $2 = kernel regex, $3 = quick_perf case
set -e
mkdir -p gpurun_out
CMD="python scripts/quick_perf.py $3"
$CMD > gpurun_out/plain_one.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${SKIP:-0} -c ${COUNT:-3} -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_one.log 2>&1
echo done
