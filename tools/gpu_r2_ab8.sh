#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests/test_parity_logprob.py tests/test_fullsize.py -q --timeout 600 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
for m in bench fused fwd bwd; do
  echo "== $m" >> ${O}_ab.log
  timeout -s KILL 1500 python tools/ab_variants.py run $m >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
done
for v in base nopf; do
  echo "== $v" >> ${O}_base.log
  RLVLA_LIB=paper_2602_05765_b200/variants/$v.so timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:lp_ -s 1 -c 1 --csv python tools/prof_fused.py --mode fused --iters 1 2>&1 | grep -E '^"[0-9]' >> ${O}_base.log
done
echo done
