#!/bin/bash
# NEXT-4 evidence: flow parity, timings at pi_0 shapes, one ncu --set full capture
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 300 python -m pytest tests/test_parity_flow.py -q --timeout 300 > ${O}_fpytest.log 2>&1; echo "rc=$?" >> ${O}_fpytest.log
for a in "" "--learned --f32" "--rows 196608" "--rows 196608 --learned --f32" "--rows 4096 --D 35"; do timeout -s KILL 120 python tools/prof_flow.py $a >> ${O}_fprof.log 2>&1; done
timeout -s KILL 120 python tools/prof_flow.py --rows 196608 --iters 3 > ${O}_fplain.log 2>&1 && \
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:flow_ -s 3 -c 1 -o ${O}_flow python tools/prof_flow.py --rows 196608 --iters 3 > ${O}_fncu.log 2>&1
echo done
