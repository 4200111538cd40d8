#!/bin/bash
# Strong-scaling series of bench.py on the visible GPUs: N = 1, 2, 4 (, 8).
# usage: tools/scale_run.sh "1 2 4" [bench args...]
NS="$1"; shift
port=29600
for n in $NS; do
  if [ "$n" = "1" ]; then
    timeout 1200 python bench.py --gpus 1 --no-cpu-baseline "$@" 2>/dev/null | tail -1
  else
    port=$((port + 1))
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus "$n" "$@" 2>/dev/null | tail -1
  fi
done
