#!/bin/bash
# L2 eviction-policy A/B of the TMA log-prob kernel (sustained bench, burst, bwd, base clock),
# the flow kernel (24,576 / 196,608 steps) and the fp32 row kernel
set -u
bash tools/gpu_ab.sh $1 bench fused bwd fused32
FLOW_ARGS="--rows 24576" bash tools/gpu_ab.sh ${1}_f24k flow
bash tools/gpu_ab.sh ${1}_f196k flow
echo done
