#!/bin/bash
# one profiler per gpurun call: ncu --set full of one fused launch (after it ran clean)
mkdir -p gpurun_out
O=gpurun_out/$1
MODE=${2:-fused}
# kernels before the captured one: fused/fwd skip the forward that builds logp_behav; bwd
# also skips the forward that produces lse
SKIP=1; [ "$MODE" = "bwd" ] && SKIP=2
timeout -s KILL 120 python tools/prof_fused.py --mode $MODE --iters 1 > ${O}_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s $SKIP -c 1 -o ${O}_${MODE} python tools/prof_fused.py --mode $MODE --iters 1 > ${O}_ncu2.log 2>&1
echo "rc=$?"
