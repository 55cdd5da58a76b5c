#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 120 python tools/prof_flow.py --iters 3 > ${O}_fplain.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:flow_ -s 3 -c 1 -o ${O}_flow24k python tools/prof_flow.py --iters 3 > ${O}_fncu.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,launch__waves_per_multiprocessor -k regex:batch_poll -c 30 --csv python tools/prof_batcher.py --iters 5 > ${O}_bpoll.csv 2>&1
echo done
