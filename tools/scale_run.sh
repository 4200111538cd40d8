#!/bin/bash
# Strong-scaling series of bench.py on the visible GPUs: N = 1, 2, 4 (, 8).
# usage: tools/scale_run.sh "1 2 4" [bench args...]
NS="$1"; shift
for n in $NS; do
  if [ "$n" = "1" ]; then
    timeout 1200 python bench.py --gpus 1 --no-cpu-baseline "$@" 2>/dev/null | tail -1
  else
    timeout 1200 torchrun --standalone --nproc-per-node "$n" bench.py --gpus "$n" "$@" 2>/dev/null | tail -1
  fi
done
