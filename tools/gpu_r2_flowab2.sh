#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
for args in "--rows 24576" "--rows 36000" "--rows 4096 --D 35" "--rows 196608"; do
  echo "== flow $args" >> ${O}_flow.log
  FLOW_ARGS="$args" timeout -s KILL 900 python tools/ab_variants.py run flow >> ${O}_flow.log 2>&1
done
echo done
