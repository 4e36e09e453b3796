set -u
OUT=gpurun_out
[ -n "${SKIP_PLAIN:-}" ] || { python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }; }
tail -1 $OUT/plain.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r1h_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_list.log 2>&1; echo "list rc=$?"
export DOCP_PROFILE_RANGE=1
for k in pcg_kernel_h8s assemble_kernel_t step_kernel kkt_kernel gamma_kernel recover_kernel vjp_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -c 1 \
     -o $OUT/r1h_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# summarise on the box (the reports themselves exceed gpurun's copy-back limit)
python tools/ncu_summary.py $OUT/r1h_*.ncu-rep > $OUT/r1h_ncu_table.md
python tools/ncu_summary.py --traffic $OUT/r1h_pcg_kernel_h8s.ncu-rep > $OUT/r1h_pcg_traffic.json
for k in pcg_kernel_h8s assemble_kernel_t; do
  ncu -i $OUT/r1h_$k.ncu-rep --page raw --csv > $OUT/r1h_${k}_raw.csv
  ncu -i $OUT/r1h_$k.ncu-rep --page source --csv --print-source cuda,sass > $OUT/r1h_${k}_src.csv
  python tools/ncu_lines.py $OUT/r1h_${k}_src.csv 40 > $OUT/r1h_${k}_lines.txt
done
ls -la $OUT; rm -f $OUT/*.ncu-rep $OUT/r1h_*_src.csv
