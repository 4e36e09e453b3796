#!/bin/bash
# ncu captures for profiles/ (run on the GPU box from the repo root). The
# plain run must exit 0 first; each kernel is then captured once with
# --set full, restricted to the bench's timed epochs (DOCP_PROFILE_RANGE):
# the first launch of each kernel inside the timed region.
set -u
OUT=gpurun_out
TAG=${TAG:-r1}
KERNELS=${KERNELS:-"pcg_kernel_h8 assemble_kernel_t step_kernel kkt_kernel il_loss_kernel il_sum_kernel init_solve_kernel gamma_kernel recover_kernel vjp_kernel"}
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
export DOCP_PROFILE_RANGE=1
for k in $KERNELS; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -c 1 \
     -o $OUT/${TAG}_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
