#!/bin/bash
# quick GPU check: logprob parity tests + kernel timings + bench
mkdir -p gpurun_out
O=gpurun_out/$1
export RLVLA_DEBUG=1
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 -x ${2:-} > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
for m in fused fwd bwd; do timeout -s KILL 200 python tools/prof_fused.py --mode $m --iters 20 >> ${O}_prof.log 2>&1; done
timeout -s KILL 400 python bench.py --no-cpu-baseline > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
