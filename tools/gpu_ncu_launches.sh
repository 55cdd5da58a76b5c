#!/bin/bash
# one profiler per gpurun call: the ncu launch list of a short bench (after it ran clean)
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_bench_small.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_ncu1.log 2>&1
echo "rc=$?"
