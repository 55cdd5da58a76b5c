#!/bin/bash
# batcher timings (3 runs) incl. the event + launch floor of a one-element kernel
mkdir -p gpurun_out
for i in 1 2 3; do timeout -s KILL 300 python tools/prof_batcher.py --iters 30 >> gpurun_out/$1_batcher.jsonl 2>>gpurun_out/$1_batcher.err; done
echo done
