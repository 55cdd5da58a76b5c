#!/bin/bash
# fixed-cost model of the flow chain call: rows sweep x {fused+stats, fused no stats, forward only}
# usage: tools/gpu_flow_small.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
for r in 4 1024 4096 12288 24576 49152 98304 196608; do
  for v in "" "--no-stats" "--fwd"; do
    timeout -s KILL 120 python tools/prof_flow.py --rows $r --iters 40 $v >> ${O}_sweep.jsonl 2>>${O}_sweep.err
  done
done
echo done
