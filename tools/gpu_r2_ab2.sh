#!/bin/bash
# A/B of the built variants (fused only) + one ncu --set full of the current fused kernel
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "== fused" >> ${O}_ab.log
timeout -s KILL 900 python tools/ab_variants.py run fused >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1 -o ${O}_fused python tools/prof_fused.py --mode fused --iters 1 > ${O}_ncu_full.log 2>&1; echo "rc=$?" >> ${O}_ncu_full.log
timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:lp_tma_kernel -s 1 -c 1 --csv python tools/prof_fused.py --mode fused --iters 1 > ${O}_base_fused.csv 2>&1
echo done
