#!/bin/bash
# round-2 evidence, one GPU: bench line, reference arm, kernel timings, ncu launch list, ncu
# --set full of the fused kernel, base-clock captures, flow and batcher timings + captures.
# Each profiler runs after its command ran clean. usage: tools/gpu_r2_final1.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout -s KILL 900 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_ref.jsonl 2>&1
for m in fused fwd bwd; do timeout -s KILL 120 python tools/prof_fused.py --mode $m --iters 20 >> ${O}_prof.log 2>&1; done
for m in fused fwd; do timeout -s KILL 120 python tools/prof_fused.py --mode $m --f32 --rows 32768 --iters 20 >> ${O}_prof_f32.log 2>&1; done
timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_bench_small.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1 -o ${O}_fused python tools/prof_fused.py --mode fused --iters 1 > ${O}_ncu2.log 2>&1
for m in fused fwd; do
  timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum -k regex:lp_tma_kernel -s 1 -c 1 --csv python tools/prof_fused.py --mode $m --iters 1 > ${O}_base_$m.csv 2>&1
done
for a in "" "--learned --f32" "--rows 196608" "--rows 196608 --learned --f32" "--rows 4096 --D 35"; do timeout -s KILL 120 python tools/prof_flow.py $a >> ${O}_fprof.log 2>&1; done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:flow_ -s 3 -c 1 -o ${O}_flow python tools/prof_flow.py --rows 196608 --iters 3 > ${O}_fncu.log 2>&1
timeout -s KILL 300 python tools/prof_batcher.py > ${O}_bprof.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:batch_poll_kernel -s 8 -c 1 -o ${O}_bpoll python tools/prof_batcher.py --iters 5 > ${O}_bncu2.log 2>&1
echo done
