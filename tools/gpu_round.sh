#!/bin/bash
# full GPU round without profilers: pytest -m gpu, smoke, kernel timings, bench (default).
# The ncu captures run as their own gpurun calls (one profiler per call):
#   tools/gpu_ncu_launches.sh <tag>   ncu launch list of bench.py --steps 2 --warmup 1
#   tools/gpu_ncu_full.sh <tag>       ncu --set full of one fused launch
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
for m in fused fwd bwd; do timeout -s KILL 120 python tools/prof_fused.py --mode $m --iters 20 >> ${O}_prof.log 2>&1; done
timeout -s KILL 600 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_ref.log 2>&1; echo "ref rc=$?" >> ${O}_ref.log
echo done
