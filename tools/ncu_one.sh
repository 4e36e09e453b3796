#!/bin/bash
# One ncu --set full capture of kernel $1 (first launch in bench.py's timed
# region), summarised on the box: counters table, DRAM traffic, per-line stalls.
# usage: bash tools/ncu_one.sh <kernel-regex> <tag>
set -u
OUT=gpurun_out
K=$1; TAG=$2
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
DOCP_PROFILE_RANGE=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:$K -c 1 -o $OUT/${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py $OUT/${TAG}.ncu-rep > $OUT/${TAG}_table.md
ncu -i $OUT/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${TAG}_src.csv
python tools/ncu_lines.py $OUT/${TAG}_src.csv 60 > $OUT/${TAG}_lines.txt
ncu -i $OUT/${TAG}.ncu-rep --page raw --csv > $OUT/${TAG}_raw.csv
rm -f $OUT/${TAG}.ncu-rep $OUT/${TAG}_src.csv
