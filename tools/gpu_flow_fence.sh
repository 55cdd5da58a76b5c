#!/bin/bash
# fence-writers A/B of the statistics tail (flow small/large, fused bench) + parity of the build
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests/test_parity_flow.py tests/test_parity_logprob.py tests/test_parity_next2.py tests/test_multigpu.py -m gpu -q -x > ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
FLOW_ARGS="--rows 24576" bash tools/gpu_ab.sh ${1}_24k flow
FLOW_ARGS="--rows 4096" bash tools/gpu_ab.sh ${1}_4k flow
bash tools/gpu_ab.sh ${1}_196k flow bench
for r in 4096 24576 196608; do
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:flow_ -s 3 -c 1 --csv python tools/prof_flow.py --rows $r --iters 1 2>&1 | grep -E '^"[0-9]' >> ${O}_ncu.csv
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:flow_ -s 3 -c 1 --csv python tools/prof_flow.py --rows $r --iters 1 --no-stats 2>&1 | grep -E '^"[0-9]' >> ${O}_ncu.csv
done
echo done
