#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
#   1. the default bench line (the driver's command), then
#   2. the ncu launch list of the same bench (per-launch gpu__time_duration), then
#   3. ncu --set full captures of the dominant kernel (GMRES MGS pass), the Ax
#      kernel and the dssum kernel at the bench's size.
# Outputs land in gpurun_out/ (summaries copied to profiles/ by hand).
set -u
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:mgs2_kernel -s 40 -c 4 \
  -o gpurun_out/mgs_full --force-overwrite \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_mgs.log 2>&1
echo "mgs capture rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:ax_helm8s -c 2 \
  -o gpurun_out/ax_full --force-overwrite \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ax.log 2>&1
echo "ax capture rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:dssum_blk -s 8 -c 2 \
  -o gpurun_out/dssum_full --force-overwrite \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dssum.log 2>&1
echo "dssum capture rc=$?"
