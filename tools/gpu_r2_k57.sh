#!/bin/bash
# ncu --set full of the forward (K5) and external-backward (K7) kernels, after a clean run
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 120 python tools/prof_fused.py --mode fwd --iters 2 > ${O}_plain.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1 -o ${O}_fwd python tools/prof_fused.py --mode fwd --iters 1 > ${O}_ncu_fwd.log 2>&1
timeout -s KILL 120 python tools/prof_fused.py --mode bwd --iters 2 >> ${O}_plain.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 2 -c 1 -o ${O}_bwd python tools/prof_fused.py --mode bwd --iters 1 > ${O}_ncu_bwd.log 2>&1
echo done
