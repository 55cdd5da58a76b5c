#!/bin/bash
# ceiling of the fused kernel's memory structure: ring-only diagnostic build vs the product vs
# torch's copy of the same bytes (interleaved)
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
for i in 1 2 3; do
  timeout -s KILL 120 python tools/prof_fused.py --mode copy --iters 12 >> ${O}_copy.jsonl 2>&1
done
bash tools/gpu_ab.sh $1 fused bwd bench
for i in 1 2 3; do
  timeout -s KILL 120 python tools/prof_fused.py --mode copy --iters 12 >> ${O}_copy.jsonl 2>&1
done
echo done
