#!/bin/bash
# full GPU round: pytest -m gpu, smoke, bench (default), ncu launch list of the bench, ncu --set full of the fused kernel
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
for m in fused fwd bwd; do timeout -s KILL 120 python tools/prof_fused.py --mode $m --iters 20 >> ${O}_prof.log 2>&1; done
timeout -s KILL 600 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
if [ "${2:-}" != "noncu" ]; then
timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_bench_small.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > ${O}_ncu1.log 2>&1
timeout -s KILL 120 python tools/prof_fused.py --mode fused --iters 1 > ${O}_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1 -o ${O}_fused python tools/prof_fused.py --mode fused --iters 1 > ${O}_ncu2.log 2>&1
fi
echo done
