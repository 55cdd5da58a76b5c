#!/bin/bash
# NEXT-3 evidence: batcher parity, timing, then ONE ncu --set full capture of a firing poll
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 300 python -m pytest tests/test_parity_batcher.py -q --timeout 300 > ${O}_bpytest.log 2>&1; echo "rc=$?" >> ${O}_bpytest.log
timeout -s KILL 300 python tools/prof_batcher.py > ${O}_bprof.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:batch_poll_kernel -s 8 -c 1 -o ${O}_bpoll python tools/prof_batcher.py --iters 5 > ${O}_bncu2.log 2>&1
echo done
