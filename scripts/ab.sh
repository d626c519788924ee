# A/B of library builds: bash scripts/ab.sh name1 name2 ... (paper_1910_04429_b200/_lib/libpa_b200_<name>.so;
# "cur" = libpa_b200.so), each timed on the same cases, interleaved twice.
mkdir -p gpurun_out
CASES=${CASES:-"1e6,5e5,1024 1e8,5e7,16"}
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = cur ]; then L=paper_1910_04429_b200/_lib/libpa_b200.so; else L=paper_1910_04429_b200/_lib/libpa_b200_$v.so; fi
    echo "== $v rep $rep"
    PAB_LIB=$L python scripts/quick_perf.py $CASES
  done
done
