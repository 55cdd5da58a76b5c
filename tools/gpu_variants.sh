#!/bin/bash
# fused-kernel timing with each NEXT-2 loss knob (tools/prof_fused.py --variant)
mkdir -p gpurun_out
O=gpurun_out/$1
for v in none dual kl ent all none; do timeout -s KILL 200 python tools/prof_fused.py --mode fused --iters 20 --variant $v >> ${O}_variants.log 2>&1; done
