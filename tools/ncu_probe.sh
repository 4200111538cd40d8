#!/bin/bash
# ncu --set full captures of the hot kernels at the given box sizes
# (tools/kernel_probe.py), exported on the GPU box to gzipped raw CSV pages and
# a JSON summary so gpurun_out/ stays far below its 64 MiB copy-back limit:
#   tools/ncu_probe.sh 32 48 64
set -u
mkdir -p gpurun_out
for ne in "$@"; do
  rep=/tmp/r2_ncu_$ne
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"mgs2|ax8t|dssum_blk" -c 14 -o $rep --force-overwrite \
    python tools/kernel_probe.py $ne > gpurun_out/ncu_probe_$ne.log 2>&1
  echo "ncu probe $ne rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv 2>/dev/null | gzip -9 > gpurun_out/r2_ncu_raw_$ne.csv.gz
  python tools/ncu_summary.py gpurun_out/r2_ncu_summary_$ne.json $rep.ncu-rep > /dev/null 2>&1
  # keep the report itself only when it is small
  sz=$(stat -c %s $rep.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 15000000 ]; then cp $rep.ncu-rep gpurun_out/; fi
done
