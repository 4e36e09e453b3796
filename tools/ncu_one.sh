#!/bin/bash
# ncu evidence for one round, summarised on the box (reports exceed gpurun's
# copy-back limit). Each capture runs only after the same command exited 0
# without ncu (B200_PROFILING.md).
#   bash tools/ncu_one.sh list <tag>                launch list of bench.py (shares, not absolutes)
#   bash tools/ncu_one.sh <kernel-regex> <tag>      --set full of the first launch in the timed region
# BENCH_ARGS (default "--steps 2 --warmup 3 --no-cpu-baseline --no-parity-pass") selects the workload,
# e.g. BENCH_ARGS="--mode parity ..." for the PARITY kernels.
set -u
OUT=gpurun_out
K=$1; TAG=$2
ARGS=${BENCH_ARGS:-"--steps 2 --warmup 3 --no-cpu-baseline --no-parity-pass"}
python bench.py $ARGS > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
if [ "$K" = "list" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py $ARGS > $OUT/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
  python tools/summarize_launches.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches.md
  exit 0
fi
DOCP_PROFILE_RANGE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:$K -c 1 -o $OUT/${TAG} -f python bench.py $ARGS > $OUT/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py $OUT/${TAG}.ncu-rep > $OUT/${TAG}_table.md
python tools/ncu_summary.py --traffic $OUT/${TAG}.ncu-rep > $OUT/${TAG}_traffic.json
ncu -i $OUT/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${TAG}_src.csv
python tools/ncu_lines.py $OUT/${TAG}_src.csv 60 > $OUT/${TAG}_lines.txt
ncu -i $OUT/${TAG}.ncu-rep --page raw --csv > $OUT/${TAG}_raw.csv
rm -f $OUT/${TAG}.ncu-rep $OUT/${TAG}_src.csv
