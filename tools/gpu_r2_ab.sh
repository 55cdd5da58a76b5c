#!/bin/bash
# A/B of the built variants (tools/ab_variants.py build) + logprob parity + base-clock ncu.
# usage: tools/gpu_r2_ab.sh <tag> [modes...]
set -u
mkdir -p gpurun_out
O=gpurun_out/$1; shift
MODES=${@:-fused fwd bwd}
timeout -s KILL 900 python -m pytest tests/test_parity_logprob.py tests/test_parity_next2.py tests/test_fullsize.py tests/test_guard_regions.py tests/test_parity_path.py -q -x --timeout 600 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
for m in $MODES; do
  echo "== $m" >> ${O}_ab.log
  timeout -s KILL 900 python tools/ab_variants.py run $m >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
done
for m in fused fwd; do
  timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum -k regex:lp_tma_kernel -s 1 -c 2 --csv python tools/prof_fused.py --mode $m --iters 2 > ${O}_base_$m.csv 2>&1; echo "rc=$?" >> ${O}_base_$m.csv
done
echo done
