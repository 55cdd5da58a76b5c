#!/bin/bash
# ncu captures of the dominant kernels (one profiler process at a time, after a clean run):
#   <tag>_fused.ncu-rep : --set full --import-source, clocks free (source-level counts)
#   <tag>_base_*.csv    : duration + DRAM bytes at the locked BASE clock (--clock-control base)
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 120 python tools/prof_fused.py --mode fused --iters 3 > ${O}_plain.log 2>&1; echo "plain rc=$?" >> ${O}_plain.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1 -o ${O}_fused python tools/prof_fused.py --mode fused --iters 1 > ${O}_ncu_full.log 2>&1; echo "rc=$?" >> ${O}_ncu_full.log
for m in fused fwd; do
  timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum -k regex:lp_tma_kernel -s 1 -c 3 --csv python tools/prof_fused.py --mode $m --iters 3 > ${O}_base_$m.csv 2>&1; echo "rc=$?" >> ${O}_base_$m.csv
  timeout -s KILL 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum -k regex:lp_tma_kernel -s 1 -c 3 --csv python tools/prof_fused.py --mode $m --iters 3 > ${O}_none_$m.csv 2>&1; echo "rc=$?" >> ${O}_none_$m.csv
done
echo done
